"""Thin ctypes binding of libfd.so (include/fd.h).

Argument marshalling only: every step of the method runs in the library's CUDA
kernels.  The function names mirror the C ABI (fd_create, fd_add_source,
fd_set_receivers, fd_step, fd_get_wavefield, fd_get_traces, ...); the
``Simulation`` class is a convenience wrapper over them.  There is no CPU
fallback: if libfd.so is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
# FD_LIB: another in-tree build of the same library (A/B experiments,
# scripts/ab.sh); the default is the package's libfd.so
LIB_PATH = Path(os.environ["FD_LIB"]).resolve() if os.environ.get("FD_LIB") else _PKG / "libfd.so"

FD_OK, FD_ERR_ARG, FD_ERR_RANGE, FD_ERR_UNSTABLE = 0, -1, -2, -3
FD_ERR_NOMEM, FD_ERR_CUDA, FD_ERR_NCCL, FD_ERR_STATE = -4, -5, -6, -7
FD_FIELD_CUR, FD_FIELD_PREV = 0, 1
FD_FLAG_ALLOW_UNSTABLE = 1
FD_OPT_KERNEL, FD_OPT_TILE, FD_OPT_ZCHUNKS, FD_OPT_ASYNC, FD_OPT_GRAPH, FD_OPT_VSLABS = 1, 2, 3, 4, 5, 6
FD_OPT_PROFILE = 7
FD_OPT_TSTEPS, FD_OPT_TB2TILE, FD_OPT_RESERVE = 8, 9, 10
FD_OPT_RESIDENT, FD_OPT_CLUSTER, FD_OPT_TRANSPORT, FD_OPT_KPLANE = 11, 12, 13, 14
FD_PEER_BLOB_BYTES = 512
KERNEL_KINDS = ["fused", "naive", "gather", "inject", "fd_pxx", "fd_pyy", "fd_pzz", "fd_time", "halo",
                "resident"]

EXPORTED = [
    "fd_create", "fd_create_dist", "fd_partition", "fd_nccl_get_unique_id", "fd_add_source",
    "fd_set_receivers", "fd_step", "fd_get_wavefield", "fd_get_traces", "fd_destroy",
    "fd_strerror", "fd_last_error", "fd_set_stream", "fd_set_allocator", "fd_set_wavefield",
    "fd_set_option", "fd_get_info", "fd_get_kernel_times", "fd_reset_kernel_times",
    "fd_peer_export", "fd_peer_import", "fd_peer_detach", "fd_set_sponge",
]


class FDError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status
        self.detail = detail


class FdDist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("device", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p), ("vel_is_slab", ctypes.c_int)]


class FdInfo(ctypes.Structure):
    _fields_ = [("steps_done", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("local_dims", ctypes.c_int64 * 3), ("z0", ctypes.c_int64), ("z1", ctypes.c_int64),
                ("pitch", ctypes.c_int64), ("kernel", ctypes.c_int), ("tile_x", ctypes.c_int),
                ("tile_y", ctypes.c_int), ("rows_per_thread", ctypes.c_int), ("p_stages", ctypes.c_int),
                ("k_stages", ctypes.c_int), ("ctas", ctypes.c_int), ("threads_per_cta", ctypes.c_int),
                ("smem_bytes", ctypes.c_int), ("zchunks", ctypes.c_int), ("order", ctypes.c_int),
                ("device_bytes", ctypes.c_double), ("steps_per_launch", ctypes.c_int),
                ("cluster_ctas", ctypes.c_int), ("kplane", ctypes.c_int), ("comm_nranks", ctypes.c_int),
                ("graph_steps", ctypes.c_int64), ("tb_kind", ctypes.c_int)]

    def as_dict(self) -> dict:
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if name == "local_dims" else v
        return d


_i64p = ctypes.POINTER(ctypes.c_int64)
_f32p = ctypes.POINTER(ctypes.c_float)
_ALLOC_T = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_FREE_T = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    st = ctypes.c_int
    sig = {
        "fd_create": ([ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, _i64p, ctypes.c_double, ctypes.c_double,
                       ctypes.c_int, _f32p, ctypes.c_uint32], st),
        "fd_create_dist": ([ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, _i64p, ctypes.c_double,
                            ctypes.c_double, ctypes.c_int, _f32p, ctypes.c_uint32, ctypes.POINTER(FdDist)], st),
        "fd_partition": ([ctypes.c_int64, ctypes.c_int, ctypes.c_int, _i64p, _i64p], st),
        "fd_nccl_get_unique_id": ([ctypes.c_void_p], st),
        "fd_add_source": ([ctypes.c_void_p, _i64p, ctypes.c_double, ctypes.c_double, ctypes.c_double], st),
        "fd_set_receivers": ([ctypes.c_void_p, ctypes.c_int64, _i64p], st),
        "fd_step": ([ctypes.c_void_p, ctypes.c_int64], st),
        "fd_get_wavefield": ([ctypes.c_void_p, ctypes.c_int, _f32p], st),
        "fd_get_traces": ([ctypes.c_void_p, _f32p, ctypes.c_int64, _i64p], st),
        "fd_destroy": ([ctypes.c_void_p], st),
        "fd_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "fd_last_error": ([], ctypes.c_char_p),
        "fd_set_stream": ([ctypes.c_void_p, ctypes.c_void_p], st),
        "fd_set_allocator": ([_ALLOC_T, _FREE_T, ctypes.c_void_p], st),
        "fd_set_wavefield": ([ctypes.c_void_p, ctypes.c_int, _f32p], st),
        "fd_set_option": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int64], st),
        "fd_get_info": ([ctypes.c_void_p, ctypes.POINTER(FdInfo)], st),
        "fd_get_kernel_times": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), _i64p], st),
        "fd_reset_kernel_times": ([ctypes.c_void_p], st),
        "fd_peer_export": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)], st),
        "fd_peer_import": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], st),
        "fd_peer_detach": ([ctypes.c_void_p], st),
        "fd_set_sponge": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_double], st),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


lib = _load()


def last_error() -> str:
    return (lib.fd_last_error() or b"").decode()


def _check(status: int, where: str):
    if status != FD_OK:
        raise FDError(status, where, last_error())


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


# ------------------------------------------------------ same-name functions
def fd_create(vel: np.ndarray, h: float, dt: float, order: int, flags: int = 0) -> ctypes.c_void_p:
    """fd_create: ``vel`` is the fp32 velocity model (shape = grid, slow->fast)."""
    v = _f32(vel)
    dims = _i64(v.shape)
    ctx = ctypes.c_void_p()
    _check(lib.fd_create(ctypes.byref(ctx), v.ndim, dims.ctypes.data_as(_i64p), float(h), float(dt), int(order),
                         v.ctypes.data_as(_f32p), int(flags)), "fd_create")
    return ctx


def fd_create_dist(vel: np.ndarray, global_dims, h: float, dt: float, order: int, rank: int, nranks: int,
                   device: int = -1, nccl_id: bytes | None = None, vel_is_slab: bool = False,
                   flags: int = 0) -> ctypes.c_void_p:
    v = _f32(vel)
    dims = _i64(global_dims)
    idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    d = FdDist(rank, nranks, device, ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None,
               1 if vel_is_slab else 0)
    ctx = ctypes.c_void_p()
    _check(lib.fd_create_dist(ctypes.byref(ctx), len(dims), dims.ctypes.data_as(_i64p), float(h), float(dt),
                              int(order), v.ctypes.data_as(_f32p), int(flags), ctypes.byref(d)), "fd_create_dist")
    return ctx


def fd_partition(nz: int, nranks: int, rank: int) -> tuple[int, int]:
    z0, z1 = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.fd_partition(nz, nranks, rank, ctypes.byref(z0), ctypes.byref(z1)), "fd_partition")
    return z0.value, z1.value


def fd_nccl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.fd_nccl_get_unique_id(buf), "fd_nccl_get_unique_id")
    return buf.raw


def fd_peer_export(ctx) -> bytes:
    """IPC handles of this rank's field buffers, K and flags (FD_OPT_TRANSPORT=1)."""
    buf = ctypes.create_string_buffer(FD_PEER_BLOB_BYTES)
    n = ctypes.c_size_t()
    _check(lib.fd_peer_export(ctx, buf, FD_PEER_BLOB_BYTES, ctypes.byref(n)), "fd_peer_export")
    return buf.raw[:n.value]


def fd_peer_import(ctx, lo_blob: bytes | None, hi_blob: bytes | None):
    lo = ctypes.create_string_buffer(lo_blob, len(lo_blob)) if lo_blob else None
    hi = ctypes.create_string_buffer(hi_blob, len(hi_blob)) if hi_blob else None
    _check(lib.fd_peer_import(ctx, lo, hi), "fd_peer_import")


def fd_peer_detach(ctx):
    _check(lib.fd_peer_detach(ctx), "fd_peer_detach")


def fd_set_sponge(ctx, width: int, alpha: float = 0.015):
    _check(lib.fd_set_sponge(ctx, int(width), float(alpha)), "fd_set_sponge")


def fd_add_source(ctx, idx, f_peak_hz: float, t0_s: float, amp: float = 1.0):
    i = _i64(idx)
    _check(lib.fd_add_source(ctx, i.ctypes.data_as(_i64p), float(f_peak_hz), float(t0_s), float(amp)),
           "fd_add_source")


def fd_set_receivers(ctx, idx):
    i = _i64(idx)
    n = 0 if i.size == 0 else i.shape[0]
    _check(lib.fd_set_receivers(ctx, n, i.ctypes.data_as(_i64p) if n else None), "fd_set_receivers")


def fd_step(ctx, n: int):
    _check(lib.fd_step(ctx, int(n)), "fd_step")


def fd_get_wavefield(ctx, which: int, shape, out: np.ndarray | None = None) -> np.ndarray:
    if out is None:
        out = np.empty(tuple(shape), dtype=np.float32)
    elif out.dtype != np.float32 or not out.flags.c_contiguous or out.size != int(np.prod(shape)):
        raise ValueError("out must be a C-contiguous float32 array of the local field's size")
    _check(lib.fd_get_wavefield(ctx, int(which), out.ctypes.data_as(_f32p)), "fd_get_wavefield")
    return out


def fd_get_traces(ctx, nrec: int, nsteps: int, out: np.ndarray | None = None) -> np.ndarray:
    """Receiver-major traces (nrec, steps done); ``nsteps`` sizes the buffer (>= the
    steps done); ``out``: optional preallocated (e.g. pinned) float32 buffer of >=
    nrec*nsteps.  The C side writes nrec rows of stride = steps done."""
    if out is None:
        out = np.empty(nrec * nsteps, dtype=np.float32)
    else:
        if out.dtype != np.float32 or not out.flags.c_contiguous or out.size < nrec * nsteps:
            raise ValueError("out must be a C-contiguous float32 array of >= nrec*nsteps elements")
    flat = out.reshape(-1)[: nrec * nsteps]
    got = ctypes.c_int64()
    _check(lib.fd_get_traces(ctx, flat.ctypes.data_as(_f32p), flat.size, ctypes.byref(got)), "fd_get_traces")
    return flat[: nrec * got.value].reshape(nrec, got.value)


def fd_destroy(ctx):
    _check(lib.fd_destroy(ctx), "fd_destroy")


def fd_set_stream(ctx, stream_handle: int | None):
    _check(lib.fd_set_stream(ctx, ctypes.c_void_p(stream_handle or 0)), "fd_set_stream")


def fd_set_wavefield(ctx, which: int, field: np.ndarray):
    f = _f32(field)
    _check(lib.fd_set_wavefield(ctx, int(which), f.ctypes.data_as(_f32p)), "fd_set_wavefield")


def fd_set_option(ctx, key: int, value: int):
    _check(lib.fd_set_option(ctx, int(key), int(value)), "fd_set_option")


def fd_get_info(ctx) -> dict:
    info = FdInfo()
    _check(lib.fd_get_info(ctx, ctypes.byref(info)), "fd_get_info")
    return info.as_dict()


def fd_get_kernel_times(ctx) -> dict:
    """{kind: (ms_total, launches)} accumulated while FD_OPT_PROFILE = 1."""
    ms = (ctypes.c_double * len(KERNEL_KINDS))()
    n = (ctypes.c_int64 * len(KERNEL_KINDS))()
    _check(lib.fd_get_kernel_times(ctx, ms, n), "fd_get_kernel_times")
    return {k: (ms[i], n[i]) for i, k in enumerate(KERNEL_KINDS) if n[i]}


def fd_reset_kernel_times(ctx):
    _check(lib.fd_reset_kernel_times(ctx), "fd_reset_kernel_times")


_alloc_keepalive = []


def fd_set_allocator_torch():
    """Route the library's device allocations through torch's caching allocator
    (PyTorch as the memory provider; the library still owns buffer lifetime)."""
    import torch

    def _alloc(nbytes, _user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device())
        except Exception:
            return None

    def _free(ptr, _user):
        torch.cuda.caching_allocator_delete(ptr)

    a, f = _ALLOC_T(_alloc), _FREE_T(_free)
    _alloc_keepalive[:] = [a, f]
    _check(lib.fd_set_allocator(a, f, None), "fd_set_allocator")


def fd_reset_allocator():
    _check(lib.fd_set_allocator(_ALLOC_T(), _FREE_T(), None), "fd_set_allocator")
    _alloc_keepalive.clear()


# ------------------------------------------------------------ convenience
class Simulation:
    """One run of the method through the C ABI (host in, host out: P:115-123)."""

    def __init__(self, vel: np.ndarray, h: float, dt: float, order: int, flags: int = 0, *,
                 dist: dict | None = None, options: dict | None = None, stream: int | None = None):
        if dist:
            self.ctx = fd_create_dist(vel, dist["global_dims"], h, dt, order, dist["rank"], dist["nranks"],
                                      dist.get("device", -1), dist.get("nccl_id"), dist.get("vel_is_slab", False),
                                      flags)
            gd = list(dist["global_dims"])
        else:
            self.ctx = fd_create(vel, h, dt, order, flags)
            gd = list(np.shape(vel))
        self.global_dims = tuple(int(d) for d in gd)
        info = fd_get_info(self.ctx)
        nd = len(self.global_dims)
        self.local_shape = tuple(int(d) for d in info["local_dims"][:nd])
        self.nrec = 0
        for k, v in (options or {}).items():
            fd_set_option(self.ctx, k, v)
        if stream is not None:
            fd_set_stream(self.ctx, stream)

    def add_source(self, idx, f, t0, amp=1.0):
        fd_add_source(self.ctx, idx, f, t0, amp)

    def set_sponge(self, width: int, alpha: float = 0.015):
        """Absorbing Cerjan frame (fd_set_sponge; reading R#18)."""
        fd_set_sponge(self.ctx, width, alpha)

    def set_receivers(self, idx):
        idx = np.asarray(idx, dtype=np.int64).reshape(-1, len(self.global_dims))
        fd_set_receivers(self.ctx, idx)
        self.nrec = idx.shape[0]

    def step(self, n: int):
        fd_step(self.ctx, n)

    def reserve(self, n: int):
        """Finish setup for n more steps (tables, CUDA graphs) outside any timed region."""
        fd_set_option(self.ctx, FD_OPT_RESERVE, n)

    def wavefield(self, which: int = FD_FIELD_CUR, out: np.ndarray | None = None) -> np.ndarray:
        """Copy a field to the host (``out``: optional preallocated, e.g. pinned, buffer)."""
        return fd_get_wavefield(self.ctx, which, self.local_shape, out)

    def set_wavefield(self, which: int, field: np.ndarray):
        fd_set_wavefield(self.ctx, which, field)

    def traces(self, out: np.ndarray | None = None) -> np.ndarray:
        """Receiver-major traces (``out``: optional preallocated, e.g. pinned, buffer)."""
        return fd_get_traces(self.ctx, self.nrec, self.info()["steps_done"], out)

    def info(self) -> dict:
        return fd_get_info(self.ctx)

    def kernel_times(self) -> dict:
        return fd_get_kernel_times(self.ctx)

    def reset_kernel_times(self):
        fd_reset_kernel_times(self.ctx)

    def close(self):
        if self.ctx:
            fd_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
