"""fd_create on a GPU: the model is uploaded once and validated on the device
(velocity_to_K_kernel: finite and > 0, the max for the CFL check of R#8);
the error classes and the reported first invalid index are those of the host
check the CPU tests exercise (tests/test_abi.py), and K is bitwise the host
formula (every parity test depends on it)."""
import numpy as np
import pytest

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


@pytest.mark.parametrize("dims", [(37, 45, 70), (90, 300)])
@pytest.mark.parametrize("bad", [np.nan, -1.0, 0.0, np.inf])
def test_invalid_velocity_reports_first_index(fd, dims, bad):
    vel = np.full(dims, 2000.0, np.float32)
    flat = vel.reshape(-1)
    i1, i2 = flat.size // 3 + 7, flat.size - 5
    flat[i2] = bad
    flat[i1] = bad
    with pytest.raises(fd.FDError) as e:
        fd.Simulation(vel, 10.0, 1e-3, 2)
    assert e.value.status == fd.FD_ERR_ARG
    assert f"velocity[{i1}]" in e.value.detail


@pytest.mark.parametrize("dims,order", [((40, 40, 40), 2), ((100, 120), 8)])
def test_cfl_checked_on_device_max(fd, dims, order):
    import oracle
    oracle.build()
    h = 10.0
    vel = np.full(dims, 2000.0, np.float32)
    vel.reshape(-1)[vel.size // 2 + 3] = 4000.0            # the max decides
    lim = oracle.cfl_max(len(dims), order)
    ok_dt = 0.99 * lim * h / 4000.0
    bad_dt = 1.01 * lim * h / 4000.0
    with fd.Simulation(vel, h, ok_dt, order) as sim:
        sim.step(2)
    with pytest.raises(fd.FDError) as e:
        fd.Simulation(vel, h, bad_dt, order)
    assert e.value.status == fd.FD_ERR_UNSTABLE
    with fd.Simulation(vel, h, bad_dt, order, fd.FD_FLAG_ALLOW_UNSTABLE) as sim:
        sim.step(1)
