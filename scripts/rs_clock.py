"""Per-warp timing of one rs2d launch (FD_RS_CLOCK debug build, gpurun):
   FD_LIB=paper_2311_05038_b200/libfd_clk.so python scripts/rs_clock.py C2 2 > log; python scripts/rs_clock.py --summary log"""
import sys

if sys.argv[1] == "--summary":
    import collections
    import statistics as st
    rows = [tuple(int(x) for x in ln.split()[1:]) for ln in open(sys.argv[2]) if ln.startswith("RSCLK")]
    hi, lo = max(r[5] for r in rows), min(r[5] for r in rows)
    last = [r for r in rows if r[5] > (hi + lo) / 2] or rows      # the second launch
    t0 = min(r[5] for r in last)
    q = lambda v: " ".join(f"{p}:{v[min(len(v) - 1, int(len(v) * p / 100))]:.1f}" for p in (0, 10, 50, 90, 100))
    print("warps", len(last))
    print("warp end (us)        ", q(sorted((r[6] - t0) / 1e3 for r in last)))
    print("static-run end (us)  ", q(sorted((r[9] - t0) / 1e3 for r in last if r[9] > 0)))
    print("runs per warp", dict(collections.Counter(r[7] for r in last)))
    print("rows per warp        ", q(sorted(float(r[8]) for r in last)))
    for r in sorted(last, key=lambda r: -r[6])[:8]:
        print(f"  slowest: sm {r[0]:3d} unit {r[1]:4d} warp {r[2]} rows [{r[3]}, {r[4]}) end {(r[6] - t0) / 1e3:.1f}"
              f" runs {r[7]} rows {r[8]}")
    sys.exit(0)
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2311_05038_b200 as fd
from workloads import config
wl = config(sys.argv[1], order=int(sys.argv[2]))
with fd.Simulation(wl.vel(), wl.h, wl.dt, wl.order, options={fd.FD_OPT_GRAPH: 0}) as sim:
    for s in wl.sources:
        sim.add_source(s.idx, s.f, s.t0, s.amp)
    sim.set_receivers(wl.receivers)
    sim.step(4)
