"""Per-plane K (FD_OPT_KPLANE; SURVEY 8(f) N4 "reduced-byte K").

When K = fl32((v dt/h)^2/scale) is constant on every plane of the slow axis
(layered and homogeneous models), the tiled kernels' KZ variants read K per
plane from a table of the same fp32 values instead of streaming the K field.
The result must be bitwise the K-field run for every kernel (single step, two
steps per launch, virtual slabs with copies and with peer pushes, the sponge
frame), within the 1e-4 gate of the fp64 oracle, and the device check must
refuse (fall back to the K field) as soon as one point of one plane differs.
"""
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


def layered(dims, layers=8):
    """LAYERED-style model with `layers` equal layers along the slow axis."""
    from workloads import velocity
    v = velocity("LAYERED", dims)
    if layers != 8:
        gz = np.arange(dims[0]).reshape((-1,) + (1,) * (len(dims) - 1))
        v = (1500.0 + 3000.0 * np.minimum(gz * layers // dims[0], layers - 1) / (layers - 1)
             + np.zeros(dims)).astype(np.float32)
    return v


def run(fd, vel, order, seq, src, recs, options=None, sponge=None, P0=None, Pm1=None, dt=5e-4):
    with fd.Simulation(vel, 10.0, dt, order, options=options) as sim:
        if sponge:
            sim.set_sponge(*sponge)
        if P0 is not None:
            sim.set_wavefield(fd.FD_FIELD_CUR, P0)
            sim.set_wavefield(fd.FD_FIELD_PREV, Pm1)
        for s in src:
            sim.add_source(*s)
        sim.set_receivers(recs)
        for n in seq:
            sim.step(n)
        return sim.wavefield(), sim.wavefield(fd.FD_FIELD_PREV), sim.traces(), sim.info()


def _case(dims):
    rest = tuple(d // 2 for d in dims[1:])
    src = [((dims[0] // 2,) + rest, 25.0, 0.02, 1.0), ((2,) + tuple(d // 3 for d in dims[1:]), 18.0, 0.03, -0.5)]
    recs = [((dims[0] // 2 + 3,) + rest), ((1,) + rest), ((dims[0] - 2,) + tuple(d - 3 for d in dims[1:]))]
    return src, recs


def _assert_same(a, b, what):
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y), what


# (dims, order): 3D and 2D, every order; sizes span several tiles with ragged tails
CASES = [((70, 40, 150), 2), ((53, 35, 70), 4), ((45, 26, 50), 6), ((41, 30, 66), 8),
         ((130, 300), 2), ((97, 200), 4), ((90, 140), 6), ((75, 130), 8)]


@pytest.mark.parametrize("dims,order", CASES)
def test_kplane_bitwise_every_kernel(fd, dims, order):
    vel = layered(dims)
    src, recs = _case(dims)
    seq = (1, 2, 37, 6)
    base = {fd.FD_OPT_RESIDENT: 1}
    modes = [{fd.FD_OPT_TSTEPS: 1}, {fd.FD_OPT_VSLABS: 3, fd.FD_OPT_TSTEPS: 1},
             {fd.FD_OPT_VSLABS: 2, fd.FD_OPT_TRANSPORT: 1, fd.FD_OPT_TSTEPS: 1}]
    if len(dims) == 2 or order <= 4:
        modes += [{fd.FD_OPT_TSTEPS: 2}, {fd.FD_OPT_TSTEPS: 2, fd.FD_OPT_VSLABS: 3},
                  {fd.FD_OPT_TSTEPS: 2, fd.FD_OPT_VSLABS: 2, fd.FD_OPT_TRANSPORT: 1}]
    ref = run(fd, vel, order, seq, src, recs, options={**base, fd.FD_OPT_TSTEPS: 1})
    assert ref[3]["kplane"] == 0
    for m in modes:
        got = run(fd, vel, order, seq, src, recs, options={**base, **m, fd.FD_OPT_KPLANE: 1})
        assert got[3]["kplane"] == 1, m
        _assert_same(got, ref, m)


@pytest.mark.parametrize("dims,order", [((44, 30, 70), 2), ((40, 28, 50), 8), ((100, 160), 2), ((80, 120), 8)])
def test_kplane_sponge_bitwise(fd, dims, order):
    """The SP|KZ variants: sponge frame with per-plane K equals the sponge run
    with the K field."""
    vel = layered(dims)
    src, recs = _case(dims)
    seq = (3, 30)
    for ts in ((1, 2) if (len(dims) == 2 or order <= 4) else (1,)):
        opts = {fd.FD_OPT_RESIDENT: 1, fd.FD_OPT_TSTEPS: ts}
        ref = run(fd, vel, order, seq, src, recs, options=opts, sponge=(6, 0.07))
        got = run(fd, vel, order, seq, src, recs, options={**opts, fd.FD_OPT_KPLANE: 1}, sponge=(6, 0.07))
        assert got[3]["kplane"] == 1
        _assert_same(got, ref, ts)


@pytest.mark.parametrize("dims,order", [((48, 40, 72), 2), ((40, 33, 50), 8), ((120, 200), 2), ((96, 150), 4)])
def test_kplane_parity_vs_oracle(fd, oracle, dims, order):
    vel = layered(dims, layers=5)
    src, recs = _case(dims)
    rng = np.random.default_rng(91)
    P0 = rng.standard_normal(dims).astype(np.float32) * 1e-2
    Pm1 = rng.standard_normal(dims).astype(np.float32) * 1e-2
    steps = 80
    P, Pp, T, info = run(fd, vel, order, (steps,), src, recs, options={fd.FD_OPT_KPLANE: 1, fd.FD_OPT_RESIDENT: 1},
                         P0=P0, Pm1=Pm1)
    assert info["kplane"] == 1
    Po, Ppo, To = oracle.run(vel, 10.0, 5e-4, order, steps, src, recs, P0=P0, Pm1=Pm1, nthreads=4)
    assert rel_l2(P, Po) <= TOL and rel_l2(Pp, Ppo) <= TOL and rel_l2(T, To) <= TOL


@pytest.mark.parametrize("dims", [(30, 26, 40), (60, 90)])
def test_kplane_detection(fd, dims):
    """One point of one plane off by one ulp: the check falls back to the K
    field (kplane 0); homogeneous models qualify; results stay bitwise."""
    src, recs = _case(dims)
    opts = {fd.FD_OPT_KPLANE: 1, fd.FD_OPT_RESIDENT: 1, fd.FD_OPT_TSTEPS: 1}
    vel = layered(dims)
    idx = (dims[0] - 1,) + tuple(d - 1 for d in dims[1:])    # last in-grid point (pitch padding follows)
    vel[idx] = np.nextafter(vel[idx], np.float32(np.inf))
    got = run(fd, vel, 2, (9,), src, recs, options=opts)
    ref = run(fd, vel, 2, (9,), src, recs, options={fd.FD_OPT_RESIDENT: 1, fd.FD_OPT_TSTEPS: 1})
    assert got[3]["kplane"] == 0
    _assert_same(got, ref, "fallback")
    homo = np.full(dims, 2000.0, np.float32)
    assert run(fd, homo, 2, (3,), src, recs, options=opts)[3]["kplane"] == 1
    # velocity varying along a fast axis only is not plane-constant
    alongx = np.broadcast_to(np.linspace(1500, 2500, dims[-1], dtype=np.float32), dims).copy()
    assert run(fd, alongx, 2, (3,), src, recs, options=opts)[3]["kplane"] == 0


@pytest.mark.parametrize("cfg,order", [("C2", 2), ("C2", 8), ("C3", 2), ("C3", 8)])
def test_kplane_full_size_bench_config(fd, cfg, order):
    """C2 (4096^2, LAYERED) and C3 (512^3, HOMO) in the launch configuration
    bench.py --kplane times: bitwise equal to the K-field run over 40 steps."""
    from workloads import config
    w = config(cfg, order)
    vel = w.vel()
    src = [(s.idx, s.f, s.t0, s.amp) for s in w.sources]
    recs = w.receivers
    a = run(fd, vel, order, (40,), src, recs, dt=w.dt)
    b = run(fd, vel, order, (40,), src, recs, dt=w.dt, options={fd.FD_OPT_KPLANE: 1})
    assert a[3]["kplane"] == 0 and b[3]["kplane"] == 1
    _assert_same(a, b, cfg)
    assert np.abs(a[0]).max() > 0


def test_kplane_with_pinned_tuning_tile_keeps_the_k_field(fd):
    """A pinned tuning-only tile (no KZ variants compiled) does not fail: the
    request is ignored (kplane 0) and the run is bitwise the default one."""
    from paper_2311_05038_b200 import fd as fdm
    dims = (40, 36, 70)
    vel = layered(dims)
    src, recs = _case(dims)
    base = {fd.FD_OPT_RESIDENT: 1, fd.FD_OPT_TSTEPS: 1}
    ref = run(fd, vel, 2, (5, 6), src, recs, options=base)
    n = 0
    for tile in range(6):                      # the 3D r=1 entries: one full, five tuning-only
        try:
            got = run(fd, vel, 2, (5, 6), src, recs, options={**base, fd.FD_OPT_TILE: tile, fd.FD_OPT_KPLANE: 1})
        except fdm.FDError as e:
            assert e.status == fd.FD_ERR_ARG, e   # not an r=1 3D tile
            continue
        n += 1
        _assert_same(got, ref, tile)
        assert got[3]["kplane"] in (0, 1)
    assert n >= 2
