"""GPU parity of the register-streamed 2D multi-step kernel (rs2d_step_kernel,
fd_rs2d.cuh) through the C ABI.

Each compiled rs2d configuration (S = 2, 3, 4 steps per pass) must equal
single steps bit for bit and the fp64 oracle within 1e-4 (P:131-137 test
procedure; Listing 3's run() body P:154-161 applied S times per pass) on the
cases its strip / event logic has to get right:
  * strips straddling the right edge (nx not a multiple of the 120 / 112 own
    columns), a grid narrower than one strip;
  * receivers: a full receiver line (more than 32 per strip: several ballot
    rounds per row), a receiver column (an event block every few rows), on
    strip faces and in the band;
  * sources: several in one strip at distant rows (the conservative event
    interval), on the halo quads of a neighbouring strip, in the band, two on
    one point;
  * fd_step lengths that are not multiples of S, graphs on / off, z-chunk
    counts (warp runs of a few rows up to whole columns).
"""
import numpy as np
import pytest

from test_gpu_parity import TOL, _rand_vel, fd, oracle, rel_l2, tiled  # noqa: F401 (fixtures)

pytestmark = pytest.mark.gpu


def _rs2d_tiles(fd, order, S):
    """Indices of the rs2d configurations for (order, S) in the temporal-blocking table."""
    from paper_2311_05038_b200 import fd as fdm
    vel = _rand_vel((40, 64), seed=1)
    out = []
    for tile in range(64):
        try:
            with fd.Simulation(vel, 10.0, 5e-4, order,
                               options=tiled(fd, {fd.FD_OPT_TSTEPS: S, fdm.FD_OPT_TB2TILE: tile})) as sim:
                sim.step(S)
                info = sim.info()
        except fdm.FDError:
            continue
        if info["tb_kind"] == 1 and info["steps_per_launch"] == S:
            out.append(tile)
    return out


def _events(dims, order):
    nz, nx = dims
    r = order // 2
    src = [((nz // 2, nx // 2), 25.0, 0.02, 1.0),
           ((nz // 5, 64), 18.0, 0.03, -0.6),               # same strip as the next, distant rows
           ((4 * nz // 5, 70), 15.0, 0.025, 0.5),
           ((nz // 3, 120), 20.0, 0.02, 0.4),               # first column of strip 1 (halo of strip 0)
           ((nz // 3 + 7, 119), 22.0, 0.03, -0.3),          # last column of strip 0
           ((nz // 2, nx // 2), 12.0, 0.04, 0.3),           # second source on one point
           ((r - 1, 33), 20.0, 0.025, 0.2)]                 # in the band
    line = [(nz // 4, x) for x in range(nx)]                 # a full receiver line
    column = [(z, 121) for z in range(0, nz, 3)]             # a receiver every third row
    extra = [(nz // 2, nx // 2), (nz // 3, 120), (nz - 1, nx - 1), (0, 0)]
    src = [sd for sd in src if sd[0][0] < nz and sd[0][1] < nx]
    recs = [rc for rc in line + column + extra if rc[0] < nz and rc[1] < nx]
    return src, recs


@pytest.mark.parametrize("dims,order,S", [((150, 517), 2, 2), ((131, 250), 4, 2), ((97, 361), 6, 2), ((103, 330), 6, 3),
                                          ((90, 245), 8, 2), ((123, 517), 2, 3), ((101, 300), 2, 4),
                                          ((117, 400), 4, 3), ((90, 250), 4, 4), ((70, 90), 2, 2),
                                          ((64, 100), 4, 4)])
def test_rs2d_bitwise_and_oracle(fd, oracle, dims, order, S):
    from paper_2311_05038_b200 import fd as fdm
    tiles = _rs2d_tiles(fd, order, S)
    assert tiles, (order, S)
    vel = _rand_vel(dims, seed=211)
    h, dt = 10.0, 0.5e-3
    src, recs = _events(dims, order)
    seq = (1, 5, 2 * S + 1, 16 + S, 3)
    P0 = np.random.default_rng(5).standard_normal(dims).astype(np.float32) * 1e-3

    def run(options):
        with fd.Simulation(vel, h, dt, order, options=tiled(fd, options)) as sim:
            sim.set_wavefield(fd.FD_FIELD_CUR, P0)
            for sdef in src:
                sim.add_source(*sdef)
            sim.set_receivers(recs)
            for n in seq:
                sim.step(n)
            return sim.wavefield(), sim.wavefield(fd.FD_FIELD_PREV), sim.traces(), sim.info()

    ref = run({fd.FD_OPT_TSTEPS: 1})
    for tile in tiles:
        for zc in (0, 1, 5):
            for graph in (1, 0):
                got = run({fd.FD_OPT_TSTEPS: S, fdm.FD_OPT_TB2TILE: tile, fd.FD_OPT_ZCHUNKS: zc,
                           fd.FD_OPT_GRAPH: graph})
                assert got[3]["tb_kind"] == 1 and got[3]["steps_per_launch"] == S
                for a, b in zip(got[:3], ref[:3]):
                    assert np.array_equal(a, b), (tile, zc, graph)
    Po, Ppo, To = oracle.run(vel, h, dt, order, sum(seq), src, recs, P0=P0, nthreads=4)
    assert rel_l2(ref[0], Po) <= TOL and rel_l2(ref[1], Ppo) <= TOL and rel_l2(ref[2], To) <= TOL


@pytest.mark.parametrize("order", [2, 4])
def test_rs2d_virtual_slabs_and_sponge(fd, oracle, order):
    """Two steps per pass on z-slabs (halo exchange of 2r / r planes) and with
    the absorbing frame: bitwise equal to single steps on one slab."""
    from paper_2311_05038_b200 import fd as fdm
    dims = (160, 389)
    vel = _rand_vel(dims, seed=17)
    src, recs = _events(dims, order)
    for sponge in (None, (12, 0.02)):
        def run(options):
            with fd.Simulation(vel, 10.0, 5e-4, order, options=tiled(fd, options)) as sim:
                if sponge:
                    sim.set_sponge(*sponge)
                for sdef in src:
                    sim.add_source(*sdef)
                sim.set_receivers(recs)
                sim.step(37)
                return sim.wavefield(), sim.wavefield(fd.FD_FIELD_PREV), sim.traces(), sim.info()
        ref = run({fd.FD_OPT_TSTEPS: 1})
        for tile in _rs2d_tiles(fd, order, 2):
            for ns in (1, 3):
                try:
                    got = run({fd.FD_OPT_TSTEPS: 2, fdm.FD_OPT_TB2TILE: tile, fd.FD_OPT_VSLABS: ns})
                except fdm.FDError as e:          # a tuning-only tile: no sponge variant
                    assert e.status in (-1, -5, -7), e
                    continue
                assert got[3]["tb_kind"] == 1
                for a, b in zip(got[:3], ref[:3]):
                    assert np.array_equal(a, b), (tile, ns, sponge)


@pytest.mark.parametrize("order,S", [(2, 4), (4, 3), (6, 3)])
def test_rs2d_is_the_2d_default(fd, order, S):
    """Auto policy: 2D orders 2 / 4 / 6 on one slab with the band rule run four /
    three / three steps per pass in the register-streamed kernel; slabs and
    the sponge frame keep two steps per pass (order 6: single steps)."""
    vel = _rand_vel((300, 700), seed=3)
    with fd.Simulation(vel, 10.0, 5e-4, order, options=tiled(fd)) as sim:
        sim.step(8)
        info = sim.info()
    assert info["tb_kind"] == 1 and info["steps_per_launch"] == S, info
    with fd.Simulation(vel, 10.0, 5e-4, order, options=tiled(fd, {fd.FD_OPT_VSLABS: 2})) as sim:
        sim.step(8)
        assert sim.info()["steps_per_launch"] == (2 if order <= 4 else 1)
    with fd.Simulation(vel, 10.0, 5e-4, order, options=tiled(fd)) as sim:
        sim.set_sponge(10, 0.02)
        sim.step(8)
        assert sim.info()["steps_per_launch"] == (2 if order <= 4 else 1)
