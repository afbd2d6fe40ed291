#!/usr/bin/env python
"""One line per bench.py JSON line of a log with '# <args>' headers."""
import json
import sys

case = None
for ln in open(sys.argv[1]):
    if ln.startswith("# "):
        case = ln[2:].strip()
    elif ln.startswith("{"):
        d = json.loads(ln)
        r = d.get("repetitions", {})
        print(f"{case:42s} {d['value']:7.1f} (min {r.get('value_min', 0):.1f} max {r.get('value_max', 0):.1f}) "
              f"frac {d['roofline']['frac']:.3f} {d['roofline']['kernel']} {d['clocks'].get('sm_mhz')} "
              f"zc {d['config'].get('zchunks')} ctas {d['config'].get('ctas')}")
    elif "rror" in ln:
        print(case, ln.strip()[:200])
