"""Worker of tests/test_gpu_peer.py (launched by torch.distributed.run).

Each rank owns a z-slab of the grid on cuda:0 (all ranks share the one GPU of
this run) and steps it with FD_OPT_TRANSPORT=1: the boundary launches store
their planes into the neighbours' halos through CUDA IPC mappings, with flag
sync.  Rank 0 writes the assembled wavefields and traces to argv[1].
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [  # dims, order, fd_step call lengths, sponge frame (width, alpha) or None
    ((40, 30, 70), 2, (1, 2, 17, 6), None),        # two steps per launch (2r-plane boundary regions)
    ((37, 26, 45), 8, (3, 12), None),              # single steps, r = 4
    ((90, 140), 4, (5, 20), None),                 # 2D two-step
    ((42, 30, 60), 2, (3, 30), (6, 0.07)),         # sponge frame (global-z factors on every rank)
]


def main():
    import torch.distributed as dist
    dist.init_process_group("gloo")
    import paper_2311_05038_b200 as fd
    from paper_2311_05038_b200 import dist as fdd
    rank, world = dist.get_rank(), dist.get_world_size()
    out = {}
    for ci, (dims, order, seq, sponge) in enumerate(CASES):
        vel = np.random.default_rng(ci).uniform(1500, 2500, dims).astype(np.float32)
        z0, z1 = fdd.partition(dims[0], world, rank)
        rest = tuple(d // 2 for d in dims[1:])
        f1 = fdd.partition(dims[0], world, 1)[0]
        src = [((f1,) + rest, 25.0, 0.02, 1.0), ((f1 - 1,) + rest, 15.0, 0.03, -0.5)]
        recs = [(f1 - 1,) + rest, (f1,) + rest, (dims[0] - 3,) + rest]
        sim = fdd.create(vel[z0:z1], dims, 10.0, 5e-4, order, device=0, transport="peer",
                         options={fd.FD_OPT_RESIDENT: 1}, sponge=sponge)
        for s in src:
            sim.add_source(*s)
        sim.set_receivers(recs)
        for n in seq:
            sim.step(n)
        P = fdd.gather_wavefield(sim.wavefield())
        Pp = fdd.gather_wavefield(sim.wavefield(fd.FD_FIELD_PREV))
        T = fdd.assemble_traces(sim.traces())
        info = sim.info()
        fdd.close(sim)
        if rank == 0:
            out[f"P{ci}"], out[f"Pp{ci}"], out[f"T{ci}"] = P, Pp, T
            out[f"spl{ci}"] = info["steps_per_launch"]
    if rank == 0:
        np.savez(sys.argv[1], **out)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
