"""Summarise scripts/ab.sh output: per (variant, case) the median and max of
the repetition values over all rounds."""
import json
import sys
from collections import defaultdict

import numpy as np

res = defaultdict(list)
clk = defaultdict(list)
key = None
for ln in open(sys.argv[1]):
    if ln.startswith("# "):
        key = tuple(x.strip() for x in ln[2:].split("|"))
    elif ln.startswith("{") and key:
        d = json.loads(ln)
        res[key] += d["repetitions"]["ms"] and [d["repetitions"]["value_median"], d["repetitions"]["value_max"]]
        clk[key].append(d["clocks"].get("sm_mhz"))
for (v, c), vals in sorted(res.items(), key=lambda kv: (kv[0][1], kv[0][0])):
    med = vals[0::2]
    mx = vals[1::2]
    print(f"{c:40s} {v:10s} median-of-medians {np.median(med):7.1f}  best {max(mx):7.1f}  runs {len(med)}  "
          f"clk {clk[(v, c)]}")
