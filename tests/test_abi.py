"""C-ABI contract tests that need no GPU: the library loads, exports every
symbol include/fd.h declares, and validates host metadata before any device
work (error taxonomy of DESIGN.md section 2)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fd():
    from __graft_entry__ import build_lib
    build_lib()
    import paper_2311_05038_b200 as m
    return m


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "fd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    names = _declared_functions()
    for must in ("fd_create", "fd_add_source", "fd_set_receivers", "fd_step", "fd_get_wavefield",
                 "fd_get_traces", "fd_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(fd):
    lib = ctypes.CDLL(str(fd.fd.LIB_PATH))
    missing = [n for n in _declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(fd.fd.EXPORTED) == _declared_functions()


def test_strerror_and_partition(fd):
    for code in range(-7, 1):
        assert fd.lib.fd_strerror(code)
    spans = [fd.fd_partition(1024, 8, q) for q in range(8)]
    assert spans[0] == (0, 128) and spans[-1] == (896, 1024)
    assert [fd.fd_partition(10, 3, q) for q in range(3)] == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(fd.FDError) as e:
        fd.fd_partition(2, 3, 0)
    assert e.value.status == -1


def test_destroy_null_ok(fd):
    assert fd.lib.fd_destroy(None) == 0


@pytest.mark.parametrize("case,status", [
    ("ndim", -1), ("order", -1), ("small", -1), ("h", -1), ("dt", -1), ("vel0", -1), ("velnan", -1),
    ("cfl", -3),
])
def test_create_validation(fd, case, status):
    dims = (20, 24)
    vel = np.full(dims, 2000.0, np.float32)
    h, dt, order = 10.0, 1e-3, 4
    if case == "order":
        order = 5
    elif case == "small":
        vel = np.full((4, 24), 2000.0, np.float32)
    elif case == "h":
        h = 0.0
    elif case == "dt":
        dt = -1.0
    elif case == "vel0":
        vel[3, 4] = 0.0
    elif case == "velnan":
        vel[3, 4] = np.nan
    elif case == "cfl":
        dt = 1e-2
    if case == "ndim":
        v = vel.reshape(1, 1, 1, *dims)
        dims4 = np.asarray(v.shape, np.int64)
        ctx = ctypes.c_void_p()
        st = fd.lib.fd_create(ctypes.byref(ctx), 4, dims4.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), h, dt,
                              order, v.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 0)
        assert st == status and not ctx.value
        return
    with pytest.raises(fd.FDError) as e:
        fd.fd_create(vel, h, dt, order)
    assert e.value.status == status
    if case == "cfl":
        assert "ratio" in e.value.detail


def test_null_pointers(fd):
    ctx = ctypes.c_void_p()
    assert fd.lib.fd_create(None, 2, None, 1.0, 1.0, 2, None, 0) == -1
    assert fd.lib.fd_create(ctypes.byref(ctx), 2, None, 1.0, 1.0, 2, None, 0) == -1
    assert fd.lib.fd_step(None, 1) == -1
    assert fd.lib.fd_add_source(None, None, 1.0, 0.0, 1.0) == -1
    assert fd.lib.fd_nccl_get_unique_id(None) == -1
    assert fd.lib.fd_last_error()


def test_unstable_flag_skips_cfl_check(fd):
    """FD_FLAG_ALLOW_UNSTABLE passes validation (then needs a device)."""
    vel = np.full((20, 24), 2000.0, np.float32)
    try:
        ctx = fd.fd_create(vel, 10.0, 1e-2, 2, fd.FD_FLAG_ALLOW_UNSTABLE)
        fd.fd_destroy(ctx)
    except fd.FDError as e:
        assert e.status == -5   # no CUDA device on a CPU box: not UNSTABLE


def test_package_fails_loudly_without_the_library(tmp_path):
    """No CPU fallback: importing the binding with libfd.so absent raises
    ImportError naming the build command (checked in a copy of the package
    so the real library stays in place)."""
    import shutil
    import subprocess
    import sys
    pkg = os.path.join(ROOT, "paper_2311_05038_b200")
    dst = tmp_path / "paper_2311_05038_b200"
    shutil.copytree(pkg, dst, ignore=shutil.ignore_patterns("*.so", "build_obj", "__pycache__"))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "try:\n    import paper_2311_05038_b200\nexcept ImportError as e:\n    print('IMPORTERROR', e)\n"
            % str(tmp_path))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120).stdout
    assert "IMPORTERROR" in out and "libfd.so is missing" in out and "no CPU fallback" in out


def test_plane_too_large_for_32bit_offsets(fd):
    """The step kernels keep in-plane offsets in 32 bits: a 3D plane of
    47000 x 47000 points (8 planes: ~70 GB, would fit a B200) is refused with
    FD_ERR_ARG before the model is read (a 1-float buffer is passed)."""
    dims = np.asarray((8, 47000, 47000), np.int64)
    v = np.full(1, 2000.0, np.float32)
    ctx = ctypes.c_void_p()
    st = fd.lib.fd_create(ctypes.byref(ctx), 3, dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 10.0, 1e-3, 2,
                          v.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 0)
    assert st == fd.FD_ERR_ARG and not ctx.value
    assert b"32-bit" in fd.lib.fd_last_error()
