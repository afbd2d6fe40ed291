"""B200-native acoustic finite-difference hot path of arXiv 2311.05038.

The product is the C-ABI library ``libfd.so`` (include/fd.h) built from
``csrc/``; ``fd`` is its thin ctypes binding.  Importing this package loads the
library and fails loudly if it is missing: there is no CPU fallback.
"""
from .fd import (  # noqa: F401
    FD_ERR_ARG, FD_ERR_CUDA, FD_ERR_NCCL, FD_ERR_NOMEM, FD_ERR_RANGE, FD_ERR_STATE, FD_ERR_UNSTABLE, FD_OK,
    FD_FIELD_CUR, FD_FIELD_PREV, FD_FLAG_ALLOW_UNSTABLE, FD_OPT_ASYNC, FD_OPT_GRAPH, FD_OPT_KERNEL,
    FD_OPT_PROFILE, FD_OPT_RESERVE, FD_OPT_RESIDENT, FD_OPT_CLUSTER, FD_OPT_TRANSPORT, FD_OPT_KPLANE, FD_OPT_TB2TILE, FD_OPT_TILE,
    FD_OPT_TSTEPS, FD_PEER_BLOB_BYTES, fd_peer_export, fd_peer_import,
    FD_OPT_VSLABS, FD_OPT_ZCHUNKS, FDError, Simulation, fd_add_source, fd_create, fd_create_dist, fd_destroy,
    fd_get_info, fd_get_kernel_times, fd_get_traces, fd_get_wavefield, fd_nccl_get_unique_id, fd_partition,
    fd_set_option, fd_set_receivers, fd_set_sponge, fd_set_stream, fd_set_wavefield, fd_step, lib,
)
