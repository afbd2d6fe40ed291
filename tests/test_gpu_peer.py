"""Peer transport (FD_OPT_TRANSPORT=1): halo planes stored by the
step kernels straight into the neighbouring slab's buffers.

* virtual slabs (one process): bitwise equal to one slab, single steps and
  two steps per launch, 2D and 3D, and within relative L2 1e-4 of the fp64
  oracle run in its own z-slab mode (oracle.run(nranks=...), memcpy halos);
* two processes on the one GPU of this run (torch.distributed.run, gloo for the
  plumbing, CUDA IPC mappings + flag sync for the data path -- the multi-rank
  code path without NCCL): bitwise equal to one process, and the assembled
  fields and traces within relative L2 1e-4 of the oracle (the sponge case
  against the oracle's Cerjan run).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from test_gpu_parity import TOL, _rand_vel, rel_l2, run_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fd():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from __graft_entry__ import build_lib
    build_lib()
    import paper_2311_05038_b200 as m
    return m


@pytest.fixture(scope="module")
def oracle():
    import oracle as o
    o.build()
    return o


@pytest.mark.parametrize("dims,order", [((40, 30, 70), 2), ((41, 29, 66), 4), ((45, 26, 50), 8),
                                        ((96, 300), 2), ((70, 140), 8)])
@pytest.mark.parametrize("nslabs", [2, 3])
@pytest.mark.parametrize("tsteps", [1, 2])
def test_peer_virtual_slabs_bitwise(fd, oracle, dims, order, nslabs, tsteps):
    if tsteps == 2 and len(dims) == 3 and order > 4:
        pytest.skip("3D two-step r >= 3: tuning-only configurations (no peer-push variant compiled)")
    vel = _rand_vel(dims, seed=73)
    r = order // 2
    nz = dims[0]
    from paper_2311_05038_b200.dist import partition
    f1 = partition(nz, nslabs, 1)[0]
    rest = tuple(d // 2 for d in dims[1:])
    src = [((f1,) + rest, 25.0, 0.02, 1.0), ((f1 - r,) + rest, 15.0, 0.03, -0.4)]
    recs = [(f1 - 1,) + rest, (f1,) + rest, (f1 + 2 * r - 1,) + rest, (nz - 3,) + rest]
    ref = run_gpu(fd, vel, 10.0, 5e-4, order, 33, src, recs, options={fd.FD_OPT_TSTEPS: 1})
    for graph in (1, 0):
        got = run_gpu(fd, vel, 10.0, 5e-4, order, 33, src, recs,
                      options={fd.FD_OPT_VSLABS: nslabs, fd.FD_OPT_TRANSPORT: 1, fd.FD_OPT_TSTEPS: tsteps,
                               fd.FD_OPT_GRAPH: graph})
        for a, b in zip(got[:3], ref[:3]):
            assert np.array_equal(a, b), (nslabs, tsteps, graph)
    # the oracle's own slab mode (memcpy halos, bitwise its global run)
    Po, Ppo, To = oracle.run(vel, 10.0, 5e-4, order, 33, src, recs, nranks=nslabs, nthreads=4)
    assert rel_l2(got[0], Po) <= TOL and rel_l2(got[1], Ppo) <= TOL and rel_l2(got[2], To) <= TOL


@pytest.mark.parametrize("resident", [1, 0])
def test_peer_transport_needs_slabs(fd, resident):
    """FD_OPT_TRANSPORT=1 on a single-slab context fails at the first step --
    also where the auto policy would pick the cluster-resident path (a small
    grid, FD_OPT_RESIDENT left at auto: ADVICE r1)."""
    vel = _rand_vel((20, 20, 20), seed=1)
    with pytest.raises(fd.FDError) as e:
        with fd.Simulation(vel, 10.0, 1e-3, 2, options={fd.FD_OPT_TRANSPORT: 1, fd.FD_OPT_RESIDENT: resident}) as sim:
            sim.step(1)
    assert e.value.status == fd.FD_ERR_STATE


@pytest.mark.parametrize("nranks", [2, 3])
def test_peer_two_processes_one_gpu_bitwise(fd, oracle, tmp_path, nranks):
    import importlib.util
    spec = importlib.util.spec_from_file_location("peer_worker", os.path.join(ROOT, "tests", "peer_worker.py"))
    worker = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(worker)
    out = str(tmp_path / "peer.npz")
    port = 29600 + nranks + (os.getpid() % 200)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "peer_worker.py"),
           out]
    env = {**os.environ, "PYTHONPATH": ROOT}
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    got = np.load(out)
    for ci, (dims, order, seq, sponge) in enumerate(worker.CASES):
        vel = np.random.default_rng(ci).uniform(1500, 2500, dims).astype(np.float32)
        rest = tuple(d // 2 for d in dims[1:])
        from paper_2311_05038_b200.dist import partition
        f1 = partition(dims[0], nranks, 1)[0]
        src = [((f1,) + rest, 25.0, 0.02, 1.0), ((f1 - 1,) + rest, 15.0, 0.03, -0.5)]
        recs = [(f1 - 1,) + rest, (f1,) + rest, (dims[0] - 3,) + rest]
        with fd.Simulation(vel, 10.0, 5e-4, order, options={fd.FD_OPT_RESIDENT: 1, fd.FD_OPT_TSTEPS: 1}) as sim:
            if sponge:
                sim.set_sponge(*sponge)
            for s in src:
                sim.add_source(*s)
            sim.set_receivers(recs)
            for n in seq:
                sim.step(n)
            ref = (sim.wavefield(), sim.wavefield(fd.FD_FIELD_PREV), sim.traces())
        assert np.array_equal(got[f"P{ci}"], ref[0]), ci
        assert np.array_equal(got[f"Pp{ci}"], ref[1]), ci
        assert np.array_equal(got[f"T{ci}"], ref[2]), ci
        # the multi-rank result against the fp64 oracle (slab mode; Cerjan frame for the sponge case)
        steps = sum(seq)
        if sponge:
            Po, Ppo, To = oracle.run(vel, 10.0, 5e-4, order, steps, src, recs, sponge=sponge, nthreads=4)
        else:
            Po, Ppo, To = oracle.run(vel, 10.0, 5e-4, order, steps, src, recs, nranks=nranks, nthreads=4)
        for a, b in ((got[f"P{ci}"], Po), (got[f"Pp{ci}"], Ppo), (got[f"T{ci}"], To)):
            assert rel_l2(a, b) <= TOL, (ci, rel_l2(a, b))


@pytest.mark.parametrize("strong", [False, True])
def test_bench_two_ranks_peer_transport_shared_gpu(fd, strong):
    """bench.py's N>1 path end to end (torchrun, barriers, max over ranks, e2e,
    one JSON line from rank 0) with the peer transport, both ranks on the one
    GPU of this run (FD_BENCH_SHARE_GPU test hook; not a scaling number):
    weak (N stacked copies) and --strong (the grid split across the ranks,
    with the sponge frame, which the peer transport needs at creation)."""
    import json
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(29800 + os.getpid() % 100 + (1 if strong else 0)),
           os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "20", "--warmup", "3", "--config", "C1", "--transport", "peer",
           "--no-cpu-baseline"] + (["--strong", "--sponge", "8"] if strong else [])
    env = {**os.environ, "FD_BENCH_SHARE_GPU": "1", "PYTHONPATH": ROOT}
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["traces_finite"]
    assert d["config"]["global_grid"][0] == (1 if strong else 2) * d["config"]["grid"][0]
    assert d["scaling"] == ("strong" if strong else "weak")
    assert d["roofline"]["points_per_launch"] == (d["config"]["grid"][0] // (2 if strong else 1)) * d["config"]["grid"][1]
    assert "peer" in d["config"]["parallelism"] and d["config"]["shared_gpu"]


def test_nccl_init_failure_poisons_the_context(fd, tmp_path):
    """SURVEY T5 (NCCL error propagation): rank 1 of a two-rank context given a
    unique id whose bootstrap root does not exist -- ncclCommInitRank fails at
    the first fd_step, which returns FD_ERR_NCCL; the context is poisoned
    (later calls FD_ERR_STATE) and fd_destroy still succeeds.  Run in a child
    process (NCCL retries the connection for a few seconds)."""
    code = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1])\n"
        "import paper_2311_05038_b200 as fd\n"
        "vel = np.full((40, 64), 2000.0, np.float32)\n"
        "ctx = fd.fd_create_dist(vel, (80, 64), 10.0, 1e-3, 2, 1, 2, 0, bytes(128), True)\n"
        "try:\n    fd.fd_step(ctx, 1)\n    print('NOERROR')\n"
        "except fd.FDError as e:\n    print('STEP', e.status)\n"
        "try:\n    fd.fd_step(ctx, 1)\nexcept fd.FDError as e:\n    print('AGAIN', e.status)\n"
        "fd.fd_destroy(ctx)\nprint('DESTROYED')\n")
    env = {**os.environ, "NCCL_SOCKET_IFNAME": "lo", "NCCL_DEBUG": "WARN"}
    res = subprocess.run([sys.executable, "-c", code, ROOT], env=env, capture_output=True, text=True, timeout=300)
    out = res.stdout
    assert f"STEP {fd.FD_ERR_NCCL}" in out, out + res.stderr[-2000:]
    assert f"AGAIN {fd.FD_ERR_STATE}" in out and "DESTROYED" in out, out


def test_virtual_slabs_over_nccl_bitwise(fd, oracle, tmp_path):
    """The NCCL send/recv exchange on one GPU: with FD_VSLAB_NCCL=1 virtual
    slabs move their halos with ncclSend/ncclRecv pairs over a one-rank
    communicator (self peer) in one group per exchange -- the NCCL calls of
    the multi-rank path, on the comm stream of the overlapped schedule and
    captured into the CUDA graphs.  Bitwise equal to one slab; the oracle
    within 1e-4; the communicator is live (fd_get_info comm_nranks == 1)."""
    cases = [((40, 30, 70), 2, 2, 2), ((45, 26, 50), 8, 3, 1), ((96, 300), 4, 3, 2), ((70, 140), 8, 2, 1),
             ((60, 29, 66), 2, 3, 1)]
    code = ("import sys, numpy as np; sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[2])\n"
            "import test_gpu_parity as t, paper_2311_05038_b200 as fd\n"
            f"cases = {cases!r}\n"
            "out = {}\n"
            "for i, (dims, order, ns, ts) in enumerate(cases):\n"
            "    vel = t._rand_vel(dims, seed=73)\n"
            "    nz = dims[0]; rest = tuple(d // 2 for d in dims[1:])\n"
            "    src = [((nz // 2,) + rest, 25.0, 0.02, 1.0), ((nz // 3,) + rest, 15.0, 0.03, -0.4)]\n"
            "    recs = [(nz // 2 - 1,) + rest, (nz // 3 + 1,) + rest, (nz - 3,) + rest]\n"
            "    for g in (1, 0):\n"
            "        r = t.run_gpu(fd, vel, 10.0, 5e-4, order, 37, src, recs,\n"
            "                      options={fd.FD_OPT_VSLABS: ns, fd.FD_OPT_TSTEPS: ts, fd.FD_OPT_GRAPH: g})\n"
            "        out[f'P{i}_{g}'], out[f'Pp{i}_{g}'], out[f'T{i}_{g}'] = r[0], r[1], r[2]\n"
            "        out[f'c{i}_{g}'] = r[3]['comm_nranks']; out[f'gs{i}_{g}'] = r[3]['graph_steps']\n"
            "np.savez(sys.argv[3], **out)\n")
    here = os.path.dirname(os.path.abspath(__file__))
    res = subprocess.run([sys.executable, "-c", code, ROOT, here, str(tmp_path / "vn.npz")],
                         env={**os.environ, "FD_VSLAB_NCCL": "1", "NCCL_DEBUG": "WARN"}, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    got = np.load(tmp_path / "vn.npz")
    for i, (dims, order, ns, ts) in enumerate(cases):
        vel = _rand_vel(dims, seed=73)
        nz = dims[0]
        rest = tuple(d // 2 for d in dims[1:])
        src = [((nz // 2,) + rest, 25.0, 0.02, 1.0), ((nz // 3,) + rest, 15.0, 0.03, -0.4)]
        recs = [(nz // 2 - 1,) + rest, (nz // 3 + 1,) + rest, (nz - 3,) + rest]
        ref = run_gpu(fd, vel, 10.0, 5e-4, order, 37, src, recs, options={fd.FD_OPT_TSTEPS: 1})
        for g in (1, 0):
            assert int(got[f"c{i}_{g}"]) == 1, (i, g)
            assert (int(got[f"gs{i}_{g}"]) > 0) == (g == 1), (i, g)
            for k, a in zip("P Pp T".split(), ref[:3]):
                assert np.array_equal(got[f"{k}{i}_{g}"], a), (i, g, k)
        Po, _, To = oracle.run(vel, 10.0, 5e-4, order, 37, src, recs, nthreads=4)
        assert rel_l2(ref[0], Po) <= TOL and rel_l2(ref[2], To) <= TOL
