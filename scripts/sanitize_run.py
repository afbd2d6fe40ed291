#!/usr/bin/env python
"""Tiny runs of every kernel path for compute-sanitizer:

    compute-sanitizer --tool memcheck  python scripts/sanitize_run.py
    compute-sanitizer --tool racecheck python scripts/sanitize_run.py
    compute-sanitizer --tool synccheck python scripts/sanitize_run.py
    compute-sanitizer --tool initcheck python scripts/sanitize_run.py

Covers the fused 3D and 2D kernels (r = 1 and 4, ragged sizes, several
z-chunks), virtual slabs with the overlapped schedule, CUDA-graph replay, the
naive and unfused reference paths, the two-steps-per-launch kernels
(3D and 2D, one slab and virtual slabs), the peer-push and sponge variants,
the per-plane-K (KZ) variants and the cluster-resident kernel.  With
FD_TB2D_LINEAR=1 the 2D two-step launches use linear units (r2).  r3: the
register-streamed 2D defaults (rs2d, S = 3, 4; the 2D single-slab default
policy), with few warps (long runs, work stealing).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2311_05038_b200 as fd
    rng = np.random.default_rng(0)
    cases = [((19, 21, 37), 2), ((23, 18, 41), 8), ((40, 75), 2), ((45, 70), 8), ((50, 90), 4)]
    for dims, order in cases:
        vel = rng.uniform(1500, 2500, dims).astype(np.float32)
        tb = [{fd.FD_OPT_TSTEPS: 2}, {fd.FD_OPT_TSTEPS: 2, fd.FD_OPT_ZCHUNKS: 3},
              {fd.FD_OPT_TSTEPS: 2, fd.FD_OPT_VSLABS: 3}] \
            if (len(dims) == 2 or order <= 4) else [{fd.FD_OPT_TSTEPS: 2}]
        if len(dims) == 2 and order <= 4:          # S steps per launch (rs2d, r3; fd_tbs.cuh)
            tb += [{fd.FD_OPT_TSTEPS: 3}, {fd.FD_OPT_TSTEPS: 3, fd.FD_OPT_ZCHUNKS: 3}]
            if order == 2:
                tb += [{fd.FD_OPT_TSTEPS: 4}]
        if len(dims) == 2 and order <= 4:          # rs2d defaults with a few warps (long runs, stealing)
            tb += [{fd.FD_OPT_ZCHUNKS: 1}, {fd.FD_OPT_TSTEPS: 4 if order == 2 else 3, fd.FD_OPT_ZCHUNKS: 2}]
        # per-plane K (KZ variants) needs a layered model: the first half of
        # the planes at one velocity, the rest at another
        kz = [{fd.FD_OPT_KPLANE: 1, "layered": True}, {fd.FD_OPT_KPLANE: 1, fd.FD_OPT_TSTEPS: 1, "layered": True},
              {fd.FD_OPT_KPLANE: 1, fd.FD_OPT_VSLABS: 2, fd.FD_OPT_TRANSPORT: 1, "layered": True}]
        for opts in [{}, {fd.FD_OPT_ZCHUNKS: 3}, {fd.FD_OPT_VSLABS: 2}, {fd.FD_OPT_KERNEL: 1},
                     {fd.FD_OPT_KERNEL: 3}, {fd.FD_OPT_GRAPH: 0}, {fd.FD_OPT_TSTEPS: 1},
                     {fd.FD_OPT_VSLABS: 2, fd.FD_OPT_TRANSPORT: 1}, {"sponge": True}] + tb + kz:
            # these small grids would take the cluster-resident path by default:
            # off here, on in its own case below
            opts = {fd.FD_OPT_RESIDENT: 1, **opts}
            layered, sponge = opts.pop("layered", False), opts.pop("sponge", False)
            v = vel
            if layered:
                v = np.full(dims, 1800.0, np.float32)
                v[dims[0] // 2:] = 2300.0
            with fd.Simulation(v, 10.0, 5e-4, order, options=opts) as sim:
                if sponge:
                    sim.set_sponge(4, 0.05)
                sim.add_source(tuple(d // 2 for d in dims), 25.0, 0.02)
                sim.set_receivers([tuple(d // 3 for d in dims), tuple(d - 1 for d in dims)])
                sim.step(20)
                P = sim.wavefield()
                T = sim.traces()
                assert np.all(np.isfinite(P)) and np.all(np.isfinite(T))
            print("ok", dims, order, opts, "layered" if layered else "", "sponge" if sponge else "", flush=True)
        # whole fd_step calls in one cluster launch (DSMEM halo pushes)
        for ncl in (0, 4):
            with fd.Simulation(vel, 10.0, 5e-4, order,
                               options={fd.FD_OPT_RESIDENT: 2, fd.FD_OPT_CLUSTER: ncl}) as sim:
                sim.add_source(tuple(d // 2 for d in dims), 25.0, 0.02)
                sim.set_receivers([tuple(d // 3 for d in dims), tuple(d - 1 for d in dims)])
                sim.step(7)
                sim.step(13)
                assert np.all(np.isfinite(sim.wavefield())) and np.all(np.isfinite(sim.traces()))
            print("ok", dims, order, "resident", ncl, flush=True)


if __name__ == "__main__":
    main()
