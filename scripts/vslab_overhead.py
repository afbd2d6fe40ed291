#!/usr/bin/env python
"""Cost of the z-slab decomposition on one GPU (run under gpurun):

    python scripts/vslab_overhead.py C3 2 [steps]

Times fd_step over K steps (CUDA events on the context stream, inputs
resident) with FD_OPT_VSLABS = 1, 2, 4, 8 for single steps (overlapped
boundary/interior schedule + device-copy halos) and for temporal blocking
(exchange of 3r planes per face after each two-step launch).  Virtual slabs
run the schedule of NCCL ranks with the transfer replaced by a device copy, so
the gap to one slab is the decomposition's own overhead (smaller launches, halo
copies, serialisation) -- the part of multi-GPU weak-scaling loss that does
not depend on NVLink.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2311_05038_b200 as fd
    from workloads import config
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    order = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
    wl = config(name, order=order)
    vel = wl.vel()
    stream = torch.cuda.Stream()
    for ts in ((1, 2) if (wl.ndim == 2 or order <= 4) else (1,)):
        for nv in (1, 2, 4, 8):
            opts = {fd.FD_OPT_TSTEPS: ts, fd.FD_OPT_VSLABS: nv, fd.FD_OPT_ASYNC: 1}
            with fd.Simulation(vel, wl.h, wl.dt, wl.order, stream=stream.cuda_stream, options=opts) as sim:
                for s in wl.sources:
                    sim.add_source(s.idx, s.f, s.t0, s.amp)
                sim.set_receivers(wl.receivers)
                sim.reserve(steps + 20)
                sim.step(20)
                stream.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                sim.step(steps)
                b.record(stream)
                b.synchronize()
                ms = a.elapsed_time(b)
            rec = {"workload": name, "order": order, "tsteps": ts, "vslabs": nv,
                   "gpts": wl.npts * steps / (ms / 1e3) / 1e9, "ms_per_step": ms / steps}
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
