"""Full-length parity on the BASELINE configurations (north star: "relative L2
<= 1e-4 after the configured number of steps"; SURVEY 4.2 T3, 8(d) "parity
metric (same run)").

Each test runs the workload exactly as bench.py does (default options: the
launch configuration that is timed) for the configured step count, copies the
CUR and PREV fields and the whole trace matrix out, and compares them with the
fp64 oracle run on the same seeded inputs (the paper's five-step procedure,
P:131-137).  Margins are printed and, with FD_PARITY_LOG=<file>, appended as
JSON lines.

C4 (1024^3, 500 steps) is beyond the oracle's budget on the full grid; it runs
the longest light-cone window the oracle affords on the cone's sub-grid (the
exact-zero property outside the cone holds at any size).

Oracle cost on a 16-thread host: C1 < 1 s, C2 ~1-3 min per order, C3 ~4 min,
C4 windows ~30 s each.
"""
import json
import os
import time

import numpy as np
import pytest

from test_gpu_parity import TOL, rel_l2

pytestmark = pytest.mark.gpu


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


def _log(rec: dict):
    print(json.dumps(rec))
    path = os.environ.get("FD_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(rec) + "\n")


def _gpu_run(fd, wl, vel):
    with fd.Simulation(vel, wl.h, wl.dt, wl.order) as sim:
        for s in wl.sources:
            sim.add_source(s.idx, s.f, s.t0, s.amp)
        sim.set_receivers(wl.receivers)
        sim.step(wl.steps)
        return sim.wavefield(), sim.wavefield(fd.FD_FIELD_PREV), sim.traces(), sim.info()


@pytest.mark.parametrize("name,order", [("C1", 2), ("C1", 8), ("C2", 2), ("C2", 4), ("C2", 6), ("C2", 8), ("C3", 2), ("C3", 8)])
def test_full_length_parity(fd, oracle, name, order):
    from workloads import config
    wl = config(name, order=order)
    vel = wl.vel()
    t0 = time.perf_counter()
    P, Pp, T, info = _gpu_run(fd, wl, vel)
    t_gpu = time.perf_counter() - t0
    src = [(s.idx, s.f, s.t0, s.amp) for s in wl.sources]
    t0 = time.perf_counter()
    Po, Ppo, To = oracle.run(vel, wl.h, wl.dt, wl.order, wl.steps, src, wl.receivers,
                             nthreads=oracle.max_threads())
    t_or = time.perf_counter() - t0
    eP, ePp, eT = rel_l2(P, Po), rel_l2(Pp, Ppo), rel_l2(T, To)
    _log({"test": "full_length", "workload": name, "order": order, "steps": wl.steps, "grid": list(wl.dims),
          "relL2_cur": eP, "relL2_prev": ePp, "relL2_traces": eT,
          "steps_per_launch": info["steps_per_launch"], "kernel_launches": info["kernel_launches"],
          "gpu_s": round(t_gpu, 2), "oracle_s": round(t_or, 1), "oracle_threads": oracle.max_threads()})
    assert info["steps_done"] == wl.steps
    assert T.shape == (len(wl.receivers), wl.steps)
    assert np.linalg.norm(To) > 0 and np.linalg.norm(Po) > 0     # the wave reached the receivers
    assert eP <= TOL and ePp <= TOL and eT <= TOL, (eP, ePp, eT)


@pytest.mark.parametrize("order,k", [(2, 240), (8, 60)])
def test_c4_longest_light_cone_window(fd, oracle, order, k):
    """C4 (1024^3 HET3D, the strong-scaling grid) for k steps in the bench's
    launch configuration; the oracle on the sub-grid holding the discrete light
    cone (radius r k, meeting the real z face 32 planes above the source); the
    GPU field exactly 0 outside it."""
    from test_gpu_parity import _cone_case
    from workloads import config
    t0 = time.perf_counter()
    info = _cone_case(fd, oracle, config("C4", order=order), k)
    _log({"test": "c4_light_cone", "workload": "C4", "order": order, "steps": k,
          "relL2_cone_box": info["relL2_box"], "relL2_traces": info["relL2_traces"],
          "steps_per_launch": info["steps_per_launch"], "seconds": round(time.perf_counter() - t0, 1)})
