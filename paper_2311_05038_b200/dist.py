"""Multi-process harness for the z-slab decomposition.

One process per GPU (launched by torchrun); torch.distributed is the plumbing:
it broadcasts the NCCL unique id from rank 0, assembles traces and gathers the
wavefield.  The per-step halo exchange itself runs inside libfd.so (NCCL
send/recv on the library's comm stream), never through torch.

Everything here is argument marshalling and host-side assembly; it does no
arithmetic of the method.
"""
from __future__ import annotations

import numpy as np

from . import fd as _fd


def partition(nz: int, nranks: int, rank: int) -> tuple[int, int]:
    """The owned planes [z0, z1) of a slab (same rule as the C ABI)."""
    return _fd.fd_partition(nz, nranks, rank)


def bootstrap_nccl_id(make_id=None) -> bytes:
    """Rank 0 creates a 128-byte ncclUniqueId; every rank receives it."""
    import torch.distributed as dist
    make_id = make_id or _fd.fd_nccl_get_unique_id
    box = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(box, src=0)
    uid = box[0]
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128
    return bytes(uid)


def create(vel_slab: np.ndarray, global_dims, h: float, dt: float, order: int, *, device: int = -1,
           nccl_id: bytes | None = None, flags: int = 0, options: dict | None = None,
           stream: int | None = None, transport: str = "nccl",
           sponge: tuple | None = None) -> "_fd.Simulation":
    """Create this rank's slab context; ``vel_slab`` holds only the owned planes.

    ``sponge``: (width, alpha) of the absorbing frame (fd_set_sponge), applied
    here because the peer transport fixes the context's configuration when
    it exchanges the IPC blobs below.

    ``transport``: "nccl" (halo send/recv on the library's comm stream) or
    "peer" (FD_OPT_TRANSPORT=1: the boundary launches store their planes into
    the neighbours' halos through CUDA IPC mappings; this function exchanges
    the IPC blobs with torch.distributed)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    if transport not in ("nccl", "peer"):
        raise ValueError(f"transport must be 'nccl' or 'peer', not {transport!r}")
    peer = transport == "peer" and world > 1
    if peer:
        options = {**(options or {}), _fd.FD_OPT_TRANSPORT: 1}
    elif nccl_id is None and world > 1:
        nccl_id = bootstrap_nccl_id()
    sim, err = None, None
    try:
        sim = _fd.Simulation(vel_slab, h, dt, order, flags,
                             dist={"global_dims": tuple(global_dims), "rank": rank, "nranks": world,
                                   "device": device, "nccl_id": nccl_id, "vel_is_slab": True},
                             options=options, stream=stream)
        if sponge:
            sim.set_sponge(*sponge)
    except _fd.FDError as e:
        err = e
    # every rank must have a context before anyone steps (NCCL is initialised
    # collectively at the first fd_step): fail everywhere if one rank failed
    if not all_ok(err is None):
        if sim is not None:
            sim.close()
        raise err if err is not None else RuntimeError("fd_create_dist failed on another rank")
    if peer:
        blob, err = None, None
        try:
            blob = _fd.fd_peer_export(sim.ctx)
        except _fd.FDError as e:
            err = e
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)
        if err is None and all(b is not None for b in blobs):
            try:
                _fd.fd_peer_import(sim.ctx, blobs[rank - 1] if rank > 0 else None,
                                   blobs[rank + 1] if rank < world - 1 else None)
            except _fd.FDError as e:
                err = e
        if not all_ok(err is None):
            sim.close()
            raise err if err is not None else RuntimeError("peer transport setup failed on another rank")
    return sim


def close(sim) -> None:
    """Collective teardown of a slab context (every rank calls it).

    Peer transport: the neighbours' last boundary stores and flag signals
    target this rank's exported buffers, so no rank may free them while
    another still has them mapped: synchronise and unmap (fd_peer_detach),
    barrier, then free (fd_destroy).  NCCL transport: barrier, then free."""
    import torch.distributed as dist
    if sim is None or not sim.ctx:
        return
    _fd.fd_peer_detach(sim.ctx)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
    sim.close()


def all_ok(ok: bool) -> bool:
    """True iff every rank reports ok (guards collective steps after a local failure)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([0 if ok else 1], dtype=torch.int32)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item()) == 0


def assemble_traces(local: np.ndarray) -> np.ndarray:
    """Sum the per-rank trace matrices: rows of receivers owned by other ranks
    are exactly 0 on each rank (fd_get_traces), so the sum is exact."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float32)).clone()
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def gather_wavefield(local: np.ndarray, dst: int = 0):
    """Concatenate the ranks' owned planes along z on rank ``dst`` (None elsewhere)."""
    import torch.distributed as dist
    parts = [None] * dist.get_world_size() if dist.get_rank() == dst else None
    dist.gather_object(np.ascontiguousarray(local), parts, dst=dst)
    if dist.get_rank() != dst:
        return None
    return np.concatenate(parts, axis=0)


def max_over_ranks(x: float) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
