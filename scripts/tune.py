#!/usr/bin/env python
"""Sweep the compiled tile configurations and z-chunk counts of the fused
kernels on one GPU (run under gpurun):

    python scripts/tune.py C3:2 C3:8 C2:2 C2:8 [--steps 100]

Prints one JSON line per (workload, tile, zchunks) with Gpts/s, and the best.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--zchunks", default="0")
    ap.add_argument("--tsteps", type=int, default=1)
    args = ap.parse_args()
    import torch
    import paper_2311_05038_b200 as fd
    from paper_2311_05038_b200 import fd as fdm
    from workloads import config
    stream = torch.cuda.Stream()
    for spec in args.specs:
        name, order = spec.split(":")
        wl = config(name, order=int(order))
        vel = wl.vel()
        best = None
        for tile in range(64):
            for zc in [int(z) for z in args.zchunks.split(",")]:
                try:
                    opts = {fd.FD_OPT_ZCHUNKS: zc, fd.FD_OPT_ASYNC: 1}
                    if args.tsteps == 2:
                        opts.update({fd.FD_OPT_TSTEPS: 2, fdm.FD_OPT_TB2TILE: tile})
                    else:
                        opts[fd.FD_OPT_TILE] = tile
                    sim = fd.Simulation(vel, wl.h, wl.dt, wl.order, stream=stream.cuda_stream, options=opts)
                except fdm.FDError as e:
                    if "tile" in e.detail:
                        continue
                    raise
                for s in wl.sources:
                    sim.add_source(s.idx, s.f, s.t0, s.amp)
                sim.set_receivers(wl.receivers)
                try:
                    sim.step(6)
                except fdm.FDError as e:
                    sim.close()
                    if e.status in (-5, -7) and "temporal" in e.detail:   # tb2 tile for another order
                        continue
                    raise
                sim.reserve(args.steps)
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sim.step(args.steps)
                e1.record(stream)
                e1.synchronize()
                ms = e0.elapsed_time(e1) / args.steps
                info = sim.info()
                sim.close()
                g = wl.npts / (ms / 1e3) / 1e9
                rec = {"workload": name, "order": wl.order, "tile": tile, "tsteps": args.tsteps, "tx": info["tile_x"],
                       "ty": info["tile_y"], "ny": info["rows_per_thread"], "zchunks": info["zchunks"],
                       "ctas": info["ctas"], "threads": info["threads_per_cta"], "smem": info["smem_bytes"],
                       "ms": ms, "gpts": g, "frac_16B_6549": g * 16 / 6549.4}
                print(json.dumps(rec), flush=True)
                if best is None or g > best["gpts"]:
                    best = rec
        print("BEST", json.dumps(best), flush=True)


if __name__ == "__main__":
    main()
