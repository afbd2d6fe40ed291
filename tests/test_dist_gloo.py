"""Multi-process (world_size 2, gloo, CPU) tests of the slab harness host logic:
NCCL-id bootstrap, partition agreement, trace assembly and wavefield gather
(paper_2311_05038_b200/dist.py), checked against the global oracle run, which
the slab decomposition must reproduce bitwise."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2311_05038_b200 import dist as fdd
        from workloads import velocity

        # 1. bootstrap: rank 0's id reaches every rank
        uid = fdd.bootstrap_nccl_id(make_id=lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        # 2. partition agrees with the oracle's and tiles [0, nz)
        nz = 37
        spans = [fdd.partition(nz, world, q) for q in range(world)]
        assert spans == [oracle.partition(nz, world, q) for q in range(world)]
        z0, z1 = spans[rank]
        # 3. per-rank view of a global oracle run: owned planes + owned trace rows
        dims = (nz, 12, 14)
        vel = velocity("RANDOM", dims)
        src = [((spans[0][1] - 1, 6, 7), 25.0, 0.02, 1.0)]
        recs = [(2, 3, 4), (spans[0][1], 6, 8), (nz - 3, 5, 5)]
        P, _, T = oracle.run(vel, 10.0, 1e-3, 4, 25, src, recs)
        Pl, _, Tl = oracle.run(vel, 10.0, 1e-3, 4, 25, src, recs, nranks=world)
        assert np.array_equal(P, Pl) and np.array_equal(T, Tl)
        own = np.array([z0 <= r[0] < z1 for r in recs])
        T_local = np.where(own[:, None], T, 0.0).astype(np.float32)
        T_all = fdd.assemble_traces(T_local)
        assert np.array_equal(T_all, T.astype(np.float32))
        W = fdd.gather_wavefield(P[z0:z1].astype(np.float32))
        if rank == 0:
            assert np.array_equal(W, P.astype(np.float32))
        else:
            assert W is None
        # 4. timings reduce to the slowest rank; guard flag
        assert fdd.max_over_ranks(1.0 + rank) == float(world)
        assert fdd.all_ok(True) and not fdd.all_ok(rank == 0)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_slab_harness_world2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
