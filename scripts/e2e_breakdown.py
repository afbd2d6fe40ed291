#!/usr/bin/env python
"""Where the end-to-end time goes (run under gpurun):

    python scripts/e2e_breakdown.py C3 2 [steps]

Times fd_create, the first fd_step (setup: buffers, tables, graph capture),
the remaining steps, fd_get_traces, fd_get_wavefield and fd_destroy with
pinned host buffers (FD_TORCH_ALLOC=1: device memory from torch's caching
allocator, as bench.py).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2311_05038_b200 as fd
    from workloads import config
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    order = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
    if os.environ.get("FD_TORCH_ALLOC") == "1":
        from paper_2311_05038_b200 import fd as fdm
        fdm.fd_set_allocator_torch()      # as bench.py: torch's caching allocator
    wl = config(name, order=order)
    vel = wl.vel()
    vp = torch.empty(vel.shape, dtype=torch.float32, pin_memory=True).numpy()
    vp[...] = vel
    out = torch.empty(vel.shape, dtype=torch.float32, pin_memory=True).numpy()
    torch.cuda.synchronize()
    for rep in range(2):
        t = [time.perf_counter()]
        sim = fd.Simulation(vp, wl.h, wl.dt, wl.order)
        for s in wl.sources:
            sim.add_source(s.idx, s.f, s.t0, s.amp)
        sim.set_receivers(wl.receivers)
        t.append(time.perf_counter())
        sim.step(16)
        t.append(time.perf_counter())
        sim.step(steps - 16)
        t.append(time.perf_counter())
        T = sim.traces()
        t.append(time.perf_counter())
        sim.wavefield(out=out)
        t.append(time.perf_counter())
        sim.close()
        t.append(time.perf_counter())
        names = ["create", "first 16 steps (setup)", f"{steps - 16} steps", "traces", "wavefield", "destroy"]
        print(f"rep {rep}: total {t[-1] - t[0]:.4f} s  " +
              "  ".join(f"{n} {b - a:.4f}" for n, a, b in zip(names, t[:-1], t[1:])), flush=True)


if __name__ == "__main__":
    main()
