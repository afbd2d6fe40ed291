"""Absorbing sponge frame on the GPU (fd_set_sponge):
parity with the fp64 oracle (oracle_run_sponge, pinned in test_oracle_pins)
and bitwise agreement of every kernel variant with the frame on."""
import numpy as np
import pytest

from test_gpu_parity import TOL, _rand_vel, rel_l2

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


def run(fd, vel, order, steps, src, recs, nb, alpha, options=None, P0=None, Pm1=None, seq=None):
    with fd.Simulation(vel, 10.0, 5e-4, order, options=options) as sim:
        sim.set_sponge(nb, alpha)
        if P0 is not None:
            sim.set_wavefield(fd.FD_FIELD_CUR, P0)
            sim.set_wavefield(fd.FD_FIELD_PREV, Pm1)
        for s in src:
            sim.add_source(*s)
        sim.set_receivers(recs)
        for n in (seq or (steps,)):
            sim.step(n)
        return sim.wavefield(), sim.wavefield(fd.FD_FIELD_PREV), sim.traces(), sim.info()


CASES = [((60, 90), 2, 8, 0.05), ((61, 100), 8, 10, 0.04), ((34, 30, 40), 2, 6, 0.08),
         ((33, 28, 44), 4, 5, 0.1), ((30, 32, 36), 8, 7, 0.06)]


@pytest.mark.parametrize("dims,order,nb,alpha", CASES)
def test_sponge_parity_vs_oracle(fd, oracle, dims, order, nb, alpha):
    vel = _rand_vel(dims, seed=81)
    rest = tuple(d // 2 for d in dims[1:])
    src = [((dims[0] // 2,) + rest, 25.0, 0.02, 1.0), ((2,) + tuple(d // 3 for d in dims[1:]), 18.0, 0.03, 0.5)]
    recs = [((dims[0] // 2 + 3,) + rest), ((1,) + rest), ((dims[0] - 2,) + tuple(d - 3 for d in dims[1:]))]
    rng = np.random.default_rng(83)
    P0 = rng.standard_normal(dims).astype(np.float32) * 1e-2
    Pm1 = rng.standard_normal(dims).astype(np.float32) * 1e-2
    steps = 60
    P, Pp, T, _ = run(fd, vel, order, steps, src, recs, nb, alpha, P0=P0, Pm1=Pm1)
    Po, Ppo, To = oracle.run(vel, 10.0, 5e-4, order, steps, src, recs, P0=P0, Pm1=Pm1, sponge=(nb, alpha),
                             nthreads=4)
    assert rel_l2(P, Po) <= TOL and rel_l2(Pp, Ppo) <= TOL and rel_l2(T, To) <= TOL
    # the frame really damps: the oracle without it differs
    Pb, _, _ = oracle.run(vel, 10.0, 5e-4, order, steps, src, recs, P0=P0, Pm1=Pm1, nthreads=4)
    assert rel_l2(Pb, Po) > 100 * TOL


@pytest.mark.parametrize("dims,order", [((40, 36, 70), 2), ((37, 30, 45), 4), ((35, 28, 40), 8), ((90, 140), 2),
                                        ((75, 130), 4), ((64, 96), 8)])
def test_sponge_all_kernels_bitwise(fd, dims, order):
    """With the frame on, the two-step kernels, the cluster-resident kernel,
    virtual slabs (copies and peer pushes), the naive and the unfused paths all
    equal the single-step tiled kernel bit for bit."""
    vel = _rand_vel(dims, seed=85)
    rest = tuple(d // 2 for d in dims[1:])
    src = [((dims[0] // 2,) + rest, 25.0, 0.02, 1.0), ((3,) + rest, 12.0, 0.03, -0.4)]
    recs = [((dims[0] // 2 + 1,) + rest), ((2,) + rest), ((dims[0] - 4,) + rest)]
    seq = (1, 2, 19, 6)
    nb, alpha = 6, 0.07
    ref = run(fd, vel, order, 0, src, recs, nb, alpha, seq=seq,
              options={fd.FD_OPT_TSTEPS: 1, fd.FD_OPT_RESIDENT: 1})
    variants = [{fd.FD_OPT_KERNEL: 1, fd.FD_OPT_RESIDENT: 1}, {fd.FD_OPT_KERNEL: 3, fd.FD_OPT_RESIDENT: 1},
                {fd.FD_OPT_VSLABS: 3, fd.FD_OPT_TSTEPS: 1}, {fd.FD_OPT_VSLABS: 2, fd.FD_OPT_TRANSPORT: 1},
                {fd.FD_OPT_RESIDENT: 2}]
    if len(dims) == 2 or order <= 4:
        variants += [{fd.FD_OPT_TSTEPS: 2, fd.FD_OPT_RESIDENT: 1},
                     {fd.FD_OPT_TSTEPS: 2, fd.FD_OPT_VSLABS: 3, fd.FD_OPT_TRANSPORT: 1}]
    n = 0
    for opts in variants:
        try:
            got = run(fd, vel, order, 0, src, recs, nb, alpha, seq=seq, options=opts)
        except fd.FDError as e:
            assert e.status == fd.FD_ERR_STATE and opts.get(fd.FD_OPT_RESIDENT) == 2, (opts, e)
            continue
        n += 1
        for a, b in zip(got[:3], ref[:3]):
            assert np.array_equal(a, b), opts
    assert n >= len(variants) - 1


def test_sponge_inactive_until_the_wave_arrives(fd):
    """Before the wave (and the zero initial field) reaches the frame, G = 1
    wherever the field is nonzero: bitwise the band-rule run."""
    dims = (81, 81)
    vel = np.full(dims, 2000.0, np.float32)
    src = [((40, 40), 25.0, 0.0, 1.0)]
    recs = [(40, 45)]
    for k in (5, 12):     # light cone radius r k = 12 < 40 - 20 cells to the frame
        a = run(fd, vel, 2, k, src, recs, 20, 0.015)
        with fd.Simulation(vel, 10.0, 5e-4, 2) as sim:
            sim.add_source(*src[0])
            sim.set_receivers(recs)
            sim.step(k)
            b = (sim.wavefield(), sim.wavefield(fd.FD_FIELD_PREV), sim.traces())
        for x, y in zip(a[:3], b):
            assert np.array_equal(x, y)


def test_sponge_arguments(fd):
    vel = _rand_vel((20, 20), seed=1)
    with fd.Simulation(vel, 10.0, 1e-3, 2) as sim:
        with pytest.raises(fd.FDError) as e:
            sim.set_sponge(-1, 0.01)
        assert e.value.status == fd.FD_ERR_ARG
        with pytest.raises(fd.FDError):
            sim.set_sponge(3, float("nan"))
        sim.step(1)
        with pytest.raises(fd.FDError) as e:
            sim.set_sponge(3, 0.01)
        assert e.value.status == fd.FD_ERR_STATE
