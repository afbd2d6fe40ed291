#!/usr/bin/env python
"""Small-grid sweep: one cluster launch per fd_step call (FD_OPT_RESIDENT) vs
the tiled kernels replayed from CUDA graphs (run under gpurun):

    python scripts/resident_sweep.py [steps]

Prints one JSON record per (grid, order, path) with us/step from CUDA events
around fd_step(steps) on the context stream (after a warm-up call).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2311_05038_b200 as fd
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    stream = torch.cuda.Stream()
    grids = [(64, 64), (128, 128), (256, 256), (384, 384), (512, 512), (32, 32, 32), (40, 40, 40), (48, 48, 48)]
    paths = [("tiled", {fd.FD_OPT_RESIDENT: 1}), ("cluster8", {fd.FD_OPT_RESIDENT: 2, fd.FD_OPT_CLUSTER: 8}),
             ("cluster16", {fd.FD_OPT_RESIDENT: 2, fd.FD_OPT_CLUSTER: 16})]
    for dims in grids:
        vel = np.full(dims, 2000.0, np.float32)
        for order in (2, 8):
            for name, opts in paths:
                try:
                    with fd.Simulation(vel, 10.0, 1e-3, order, stream=stream.cuda_stream,
                                       options={**opts, fd.FD_OPT_ASYNC: 1}) as sim:
                        sim.add_source(tuple(d // 2 for d in dims), 25.0, 0.04)
                        sim.set_receivers([tuple([d // 3 for d in dims])])
                        sim.reserve(2 * steps + 16)
                        sim.step(16)
                        stream.synchronize()
                        a = torch.cuda.Event(enable_timing=True)
                        b = torch.cuda.Event(enable_timing=True)
                        a.record(stream)
                        sim.step(steps)
                        b.record(stream)
                        b.synchronize()
                        us = a.elapsed_time(b) * 1e3 / steps
                        info = sim.info()
                except fd.FDError as e:
                    print(json.dumps({"dims": dims, "order": order, "path": name, "error": e.detail}), flush=True)
                    continue
                npts = int(np.prod(dims))
                print(json.dumps({"dims": dims, "order": order, "path": name, "us_per_step": us,
                                  "gpts": npts / us / 1e3, "cluster_ctas": info["cluster_ctas"],
                                  "threads": info["threads_per_cta"], "smem": info["smem_bytes"]}), flush=True)


if __name__ == "__main__":
    main()
