"""fp64 CPU oracle for the acoustic FD time step (arXiv 2311.05038).

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2311_05038_b200`` never imports it and
shares no code with it (the ``workloads`` module, which holds no arithmetic of
the method, feeds inputs to both).

This is a thin ctypes wrapper over ``fd_oracle.c`` (plain fp64 loops, see the
header of that file for the algorithm and its citations).  Every function here
only marshals numpy arrays.

Parity status per function (DESIGN.md section 4 lists the pins):
  coefficients, cfl_max, ricker, second_derivative, time_update, run,
  run_slabs, sponge_profile, run(sponge=...): pinned (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "fd_oracle.c"
_LIB = _HERE / "liboracle.so"

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> Path:
    """Compile fd_oracle.c with gcc (fp64, no FMA contraction, OpenMP)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
            "-fPIC", "-shared", "-o", str(tmp), str(_SRC), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(build()))
        _lib.oracle_coefficients.argtypes = [ctypes.c_int, _f64p]
        _lib.oracle_cfl_max.argtypes = [ctypes.c_int, ctypes.c_int]
        _lib.oracle_cfl_max.restype = ctypes.c_double
        _lib.oracle_ricker.argtypes = [ctypes.c_double] * 3
        _lib.oracle_ricker.restype = ctypes.c_double
        _lib.oracle_second_derivative.argtypes = [
            ctypes.c_int, _i64p, ctypes.c_double, ctypes.c_int, ctypes.c_int, _f64p, _f64p]
        _lib.oracle_time_update.argtypes = [
            ctypes.c_int64, ctypes.c_double, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p]
        run_args = [ctypes.c_int, _i64p, ctypes.c_double, ctypes.c_double, ctypes.c_int, _f64p,
                    ctypes.c_int, _i64p, _f64p, _f64p, _f64p,
                    ctypes.c_int, _i64p, ctypes.c_int64, _f64p, _f64p, _f64p, ctypes.c_int]
        _lib.oracle_run.argtypes = run_args
        _lib.oracle_run_slabs.argtypes = run_args
        _lib.oracle_run_sponge.argtypes = run_args + [ctypes.c_int, ctypes.c_double]
        _lib.oracle_sponge_profile.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_double, _f64p]
        _lib.oracle_partition.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, _i64p, _i64p]
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def coefficients(order: int) -> np.ndarray:
    """c[0..r] of the order-``order`` central second difference (fp64)."""
    c = np.zeros(5)
    if lib().oracle_coefficients(order // 2, _p(c, _f64p)) != 0 or order % 2:
        raise ValueError(f"unsupported order {order}")
    return c[: order // 2 + 1].copy()


def cfl_max(ndim: int, order: int) -> float:
    v = lib().oracle_cfl_max(ndim, order)
    if v < 0:
        raise ValueError("bad ndim/order")
    return v


def ricker(t: float, f: float, t0: float) -> float:
    return lib().oracle_ricker(float(t), float(f), float(t0))


def second_derivative(P: np.ndarray, h: float, order: int, axis: str) -> np.ndarray:
    """fd_pxx / fd_pyy / fd_pzz with the band rule; ``axis`` in 'x','y','z'."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    dims = np.asarray(P.shape, dtype=np.int64)
    out = np.empty_like(P)
    a = {"x": 0, "y": 1, "z": 2}[axis]
    rc = lib().oracle_second_derivative(P.ndim, _p(dims, _i64p), float(h), int(order), a,
                                        _p(P, _f64p), _p(out, _f64p))
    if rc != 0:
        raise ValueError(f"oracle_second_derivative failed ({rc})")
    return out


def time_update(P, Pold, V, Pxx, Pzz, dt, Pyy=None) -> np.ndarray:
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (P, Pold, V, Pxx, Pzz)]
    P, Pold, V, Pxx, Pzz = arrs
    Pyy_ = None if Pyy is None else np.ascontiguousarray(Pyy, dtype=np.float64)
    out = np.empty_like(P)
    rc = lib().oracle_time_update(P.size, float(dt), _p(P, _f64p), _p(Pold, _f64p), _p(V, _f64p),
                                  _p(Pxx, _f64p), None if Pyy_ is None else _p(Pyy_, _f64p),
                                  _p(Pzz, _f64p), _p(out, _f64p))
    if rc != 0:
        raise ValueError("oracle_time_update failed")
    return out


def _pack_sources(sources, ndim):
    # sources: list of (idx tuple, f, t0, amp)
    n = len(sources)
    idx = np.zeros((max(n, 1), ndim), dtype=np.int64)
    f = np.zeros(max(n, 1)); t0 = np.zeros(max(n, 1)); amp = np.zeros(max(n, 1))
    for s, (i, fs, ts, a) in enumerate(sources):
        idx[s] = i; f[s] = fs; t0[s] = ts; amp[s] = a
    return n, idx, f, t0, amp


def sponge_profile(n: int, nb: int, alpha: float) -> np.ndarray:
    """Cerjan damping profile g(j), j = 0..n-1 (R#18; fd_oracle.c)."""
    g = np.zeros(int(n))
    if lib().oracle_sponge_profile(int(n), int(nb), float(alpha), _p(g, _f64p)) != 0:
        raise ValueError("bad sponge profile args")
    return g


def run(vel, h, dt, order, nt, sources=(), receivers=(), P0=None, Pm1=None,
        nthreads: int = 1, nranks: int = 0, sponge=None):
    """Run ``nt`` steps; returns (P^nt, P_mod^{nt-1}, traces[nrec, nt]).

    ``vel``: velocity array (shape = grid, slow->fast); its values are used in
    fp64 exactly as given (pass the fp32 model to compare with the GPU path).
    ``sources``: list of (idx, f_peak, t0, amp); ``receivers``: list of idx.
    ``nranks`` > 0 selects the z-slab mode (bitwise equal by construction).
    ``sponge`` = (nb, alpha) selects the Cerjan absorbing frame (R#18;
    oracle_run_sponge; the returned Pold is the stored P^{nt-1}).
    """
    V = np.ascontiguousarray(vel, dtype=np.float64)
    ndim = V.ndim
    dims = np.asarray(V.shape, dtype=np.int64)
    P = np.zeros_like(V) if P0 is None else np.array(P0, dtype=np.float64, order="C", copy=True)
    Pold = np.zeros_like(V) if Pm1 is None else np.array(Pm1, dtype=np.float64, order="C", copy=True)
    ns, sidx, sf, st0, samp = _pack_sources(list(sources), ndim)
    recs = np.asarray(list(receivers), dtype=np.int64).reshape(-1, ndim)
    nrec = recs.shape[0]
    T = np.zeros((max(nrec, 1), max(int(nt), 1)))
    recs_c = np.ascontiguousarray(recs if nrec else np.zeros((1, ndim), np.int64))
    L = lib()
    args = (ndim, _p(dims, _i64p), float(h), float(dt), int(order), _p(V, _f64p),
            ns, _p(sidx, _i64p), _p(sf, _f64p), _p(st0, _f64p), _p(samp, _f64p),
            nrec, _p(recs_c, _i64p), int(nt), _p(P, _f64p), _p(Pold, _f64p), _p(T, _f64p))
    if sponge is not None:
        if nranks > 0:
            raise ValueError("the sponge oracle has no slab mode")
        rc = L.oracle_run_sponge(*args, int(nthreads), int(sponge[0]), float(sponge[1]))
    else:
        fn = L.oracle_run_slabs if nranks > 0 else L.oracle_run
        rc = fn(*args, nranks if nranks > 0 else int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle run failed ({rc})")
    return P, Pold, T[:nrec, :int(nt)]


def partition(nz: int, nranks: int, rank: int):
    z0 = ctypes.c_int64(); z1 = ctypes.c_int64()
    if lib().oracle_partition(nz, nranks, rank, ctypes.byref(z0), ctypes.byref(z1)) != 0:
        raise ValueError("bad partition args")
    return z0.value, z1.value


def max_threads() -> int:
    return lib().oracle_max_threads()
