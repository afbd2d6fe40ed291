#!/usr/bin/env python
"""Key metrics, stall samples and the instruction mix of one kernel in an
ncu --set full capture (run here, no GPU):  python scripts/ncu_brief.py X.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__block_size"]
for n in want:
    if n in h:
        print(f"{n:58s} {v[h.index(n)]:>16s} {u[h.index(n)]}")
st = [(n[len("smsp__pcsamp_warps_issue_stalled_"):], int(float(v[i] or 0))) for i, n in enumerate(h)
      if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
print("stall samples:", ", ".join(f"{k} {c}" for k, c in sorted(st, key=lambda t: -t[1]) if c))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
k = next(i for i, r in enumerate(srows) if "Address" in r)
hdr, data = srows[k], srows[k + 1:]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
c = collections.Counter()
tot = 0
for r in data:
    if len(r) <= iex:
        continue
    n = int(r[iex] or 0)
    ops = [o for o in r[isrc].split() if not o.startswith("@")]
    c[ops[0].split(".")[0] if ops else "?"] += n
    tot += n
print("instruction mix (warp instr):", tot)
print("  " + ", ".join(f"{m} {n / tot * 100:.1f}%" for m, n in c.most_common(18)))
