/*
 * fd.h -- C ABI of the B200-native acoustic finite-difference hot path.
 *
 * The method (Hadjigeorgiou et al., arXiv 2311.05038, "An approach to
 * performance portability through generic programming"):
 *   Eq. 1: d2P/dt2 = v^2 (d2P/dx2 + d2P/dz2) + S(t),
 *   discretised by Listing 3's WaveSimulator::run() body:
 *   add_source; fd_pzz; fd_pxx; fd_time; swap(Pold,P); swap(P,Pnew).
 * One fd_step = that body, i.e. the leapfrog update
 *   p_next = 2 p - p_prev + (v dt)^2 Lap_h(p)     (with the band rule),
 * executed on the GPU as ONE fused kernel per step.
 * The readings of the paper's gaps (stencil order, boundary, source, receivers,
 * precision, CFL, 3D) are DESIGN.md section 3, "R#n" below.
 *
 * Conventions for every function:
 *   - returns fd_status; FD_OK (0) on success, a negative code otherwise, with a
 *     human-readable detail in fd_last_error() (thread-local).  The library
 *     never aborts the process.
 *   - all host pointers are caller-owned; they are read or written only during
 *     the call and never retained (the start/stop protocol of P:115-123:
 *     inputs are copied in at creation, outputs copied out on request).
 *   - arrays are row-major with the SLOWEST axis first: 2D (nz, nx), 3D
 *     (nz, ny, nx); x is the fastest axis (R#11).  Grid indices are int64.
 *   - one context must not be used from two threads at once; distinct contexts
 *     are independent.
 *   - after FD_ERR_CUDA / FD_ERR_NCCL the context is poisoned: only fd_destroy
 *     is valid on it.
 */
#ifndef FD_H
#define FD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fd_ctx fd_ctx; /* opaque; owns all device memory of one run */

typedef enum {
    FD_OK = 0,
    FD_ERR_ARG = -1,      /* invalid argument (null pointer, bad ndim/order/dims/h/dt, v<=0 or non-finite, f<=0) */
    FD_ERR_RANGE = -2,    /* a source/receiver index outside the (global) grid */
    FD_ERR_UNSTABLE = -3, /* max(v) dt / h above the CFL limit of R#8 (message carries the ratio) */
    FD_ERR_NOMEM = -4,    /* device or host allocation failed */
    FD_ERR_CUDA = -5,     /* CUDA runtime/driver failure (context poisoned) */
    FD_ERR_NCCL = -6,     /* NCCL failure or NCCL unavailable (context poisoned) */
    FD_ERR_STATE = -7     /* call not valid in the current state (see each function) */
} fd_status;

enum { FD_FIELD_CUR = 0,   /* P^k after k steps (before the injection of w_k)          */
       FD_FIELD_PREV = 1   /* P_mod^{k-1}: the previous field INCLUDING its injection  */
};                         /*   (Listing 3 rotation: swap(Pold,P) after add_source) */

enum { FD_FLAG_ALLOW_UNSTABLE = 1u /* skip the CFL refusal (S:553 --allow-unstable) */ };

/* ------------------------------------------------------------------ setup */

/* Create a single-GPU context on the current CUDA device.
 *   ndim   2 or 3 (the paper is 2D; 3D adds d2/dy2 with the same rule, R#10)
 *   dims   ndim extents, slow->fast; each >= order+1 (grid at least the stencil)
 *   h      uniform grid spacing (one _dh; R#9), > 0
 *   dt     time step (_dt), > 0
 *   order  spatial order 2|4|6|8 of the central second differences (R#1, R#2)
 *   vel    host, prod(dims) fp32 velocities, all finite and > 0; copied.
 *          Stored on the device as K = (v dt / h)^2 / scale (computed in fp64,
 *          rounded once), the only per-point coefficient of the update (R#7).
 *          Validated on the device after the one copy (the K conversion
 *          kernel checks each entry and reduces max(v) for the CFL check);
 *          pinned host memory makes the copy asynchronous DMA.
 *   flags  FD_FLAG_ALLOW_UNSTABLE to skip the CFL check (R#8).
 * Initial state: P^0 = P^-1 = 0 (R#12), no sources, no receivers, k = 0.
 * Errors: FD_ERR_ARG, FD_ERR_UNSTABLE, FD_ERR_NOMEM, FD_ERR_CUDA.  On error *out = NULL. */
fd_status fd_create(fd_ctx **out, int ndim, const int64_t *dims, double h, double dt,
                    int order, const float *vel, uint32_t flags);

/* Distributed (one process per GPU, z-slab decomposition). */
typedef struct {
    int rank, nranks;      /* this process's slab and the number of slabs             */
    int device;            /* CUDA device ordinal to use (-1: the current device)     */
    const void *nccl_id;   /* 128-byte ncclUniqueId from fd_nccl_get_unique_id on rank 0,
                              broadcast by the caller (e.g. torch.distributed); may be
                              NULL when nranks == 1 or with FD_OPT_TRANSPORT = 1       */
    int vel_is_slab;       /* 0: vel holds the global model; 1: only this rank's planes
                              [z0, z1) of fd_partition                                 */
} fd_dist;

/* Same as fd_create for the slab [z0, z1) = fd_partition(global_dims[0], nranks, rank).
 * Source/receiver indices stay GLOBAL.  Halo exchange of r planes per face per step
 * over NCCL send/recv.  Errors as fd_create, plus FD_ERR_NCCL. */
fd_status fd_create_dist(fd_ctx **out, int ndim, const int64_t *global_dims, double h,
                         double dt, int order, const float *vel, uint32_t flags,
                         const fd_dist *dist);

/* Pure: the owned z range of a slab.  nz split evenly, the first nz % nranks slabs
 * get one extra plane.  FD_ERR_ARG if nranks < 1, rank outside [0,nranks), nz < nranks. */
fd_status fd_partition(int64_t nz, int nranks, int rank, int64_t *z0, int64_t *z1);

/* Writes a fresh 128-byte ncclUniqueId to out128.  FD_ERR_NCCL if NCCL is unavailable. */
fd_status fd_nccl_get_unique_id(void *out128);

/* Peer transport (FD_OPT_TRANSPORT = 1): the step kernels store
 * their boundary planes straight into the z-neighbours' halo planes (CUDA IPC
 * mappings over NVLink) and a flag in the neighbour's memory orders the steps;
 * no NCCL.  Protocol, before the first fd_step:
 *   fd_peer_export(ctx, blob, cap, &len)  -- allocates all four field buffers and
 *       the flags, freezes the options and writes an opaque blob
 *       (<= FD_PEER_BLOB_BYTES) of IPC handles of this rank's field buffers, K and
 *       flags (sources / receivers / initial fields may still be set after it);
 *   the caller exchanges the blobs (e.g. torch.distributed all_gather);
 *   fd_peer_import(ctx, lo_blob, hi_blob) -- the blobs of rank - 1 and rank + 1
 *       (NULL at the global faces); opens the mappings.
 * Errors: FD_ERR_STATE (not a multi-rank context with FD_OPT_TRANSPORT = 1, after
 * the first fd_step, custom allocator set, blob of another grid), FD_ERR_ARG (cap
 * too small, missing blob), FD_ERR_CUDA (IPC failure). */
enum { FD_PEER_BLOB_BYTES = 512 };
fd_status fd_peer_export(fd_ctx *ctx, void *blob, size_t cap, size_t *len);
fd_status fd_peer_import(fd_ctx *ctx, const void *lo_blob, const void *hi_blob);
/* Teardown of the peer transport (collective order): every rank
 * calls fd_peer_detach -- it synchronises the context's streams (its last
 * pushes and signals into the neighbours' memory are done) and closes the IPC
 * mappings -- then a barrier, then fd_destroy (which frees the exported
 * buffers).  No fd_step afterwards (FD_ERR_STATE).  A no-op on other contexts.
 * A neighbour that stops signalling (failed or exited rank) is detected by a
 * bounded wait (FD_PEER_TIMEOUT_S seconds, default 60): the next fd_step returns
 * FD_ERR_STATE and the context is poisoned.  Errors: FD_ERR_ARG, FD_ERR_CUDA. */
fd_status fd_peer_detach(fd_ctx *ctx);

/* Absorbing sponge frame (reading R#18 -- the paper is silent on
 * boundaries, the band rule R#3 stays on the derivatives).  Cerjan et al. (1985):
 * within `width` cells of each face, g(j) = exp(-(alpha (width - d))^2), d = min(j,
 * n-1-j), G = g_z (g_y g_x) (fp64 per axis, rounded once to fp32), and each step is
 *   P^{k+1} = G (2 P^k - G P^{k-1} + K S(P^k))        (fp32: G * fma(K, S, fma(2, p, -(G pp))))
 * on the stored fields -- Cerjan's damp-both-levels-after-the-step, so
 * fd_get_wavefield(PREV) is the stored level (Cerjan's is G * PREV).  width 0 (the
 * default) disables it; G = 1 keeps every kernel bitwise on the band-rule path.
 * Classic values: width 20, alpha 0.015.  Before the first fd_step.
 * Errors: FD_ERR_ARG (width < 0, alpha < 0 or not finite), FD_ERR_STATE. */
fd_status fd_set_sponge(fd_ctx *ctx, int width, double alpha);

/* Register a point source (add_source; R#4, R#5): before the stencil of step k,
 * P[idx] += amp * R(k dt) with the Ricker wavelet R(t) = (1 - 2 pi^2 f^2 (t-t0)^2)
 * exp(-pi^2 f^2 (t-t0)^2), evaluated in fp64 and rounded once to fp32.
 * Several sources (even at one point) add in registration order.  At most 16.
 *   idx  ndim global indices, slow->fast.
 * Errors: FD_ERR_ARG (null, f_peak_hz <= 0, non-finite t0/amp, too many sources),
 *         FD_ERR_RANGE (idx outside the grid), FD_ERR_STATE (after the first fd_step). */
fd_status fd_add_source(fd_ctx *ctx, const int64_t *idx, double f_peak_hz, double t0_s,
                        double amp);

/* Register receivers (R#6), replacing any previous set: trace sample k of receiver j is
 * P^{k+1}[idx_j], the newest field after step k (before the injection of w_{k+1}).
 *   idx  nrec x ndim global indices (row j = receiver j), slow->fast; nrec >= 0.
 * Errors: FD_ERR_ARG, FD_ERR_RANGE, FD_ERR_STATE (after the first fd_step). */
fd_status fd_set_receivers(fd_ctx *ctx, int64_t nrec, const int64_t *idx);

/* ------------------------------------------------------------------- run */

/* Advance n >= 0 time steps (n repetitions of the run() body, R#15).  Synchronous:
 * returns after the device work is complete (or enqueued when a stream was set
 * with fd_set_stream and FD_OPT_ASYNC is 1).  Errors: FD_ERR_ARG (n < 0),
 * FD_ERR_CUDA, FD_ERR_NCCL, FD_ERR_NOMEM (trace buffer growth). */
fd_status fd_step(fd_ctx *ctx, int64_t n);

/* Copy a field to host_out (prod(local dims) floats; local = the slab in distributed
 * mode, the whole grid otherwise).  which = FD_FIELD_CUR | FD_FIELD_PREV.
 * Errors: FD_ERR_ARG, FD_ERR_CUDA. */
fd_status fd_get_wavefield(fd_ctx *ctx, int which, float *host_out);

/* Copy the traces recorded so far to host_out as a receiver-major nrec x nsteps matrix
 * (row j = receiver j in registration order).  cap = capacity of host_out in floats;
 * *nsteps_out = steps recorded.  In distributed mode rows of receivers owned by other
 * ranks are exactly 0 (sum across ranks to assemble).  The transposition from the
 * device's step-major record runs on the device (a temporary nrec x nsteps buffer);
 * one copy reaches host_out (pinned host memory makes it a direct DMA).
 * Errors: FD_ERR_ARG (null), FD_ERR_STATE (no receivers, or cap < nrec*nsteps),
 * FD_ERR_NOMEM (temporary buffer), FD_ERR_CUDA. */
fd_status fd_get_traces(fd_ctx *ctx, float *host_out, int64_t cap, int64_t *nsteps_out);

/* Release everything.  NULL -> FD_OK. */
fd_status fd_destroy(fd_ctx *ctx);

const char *fd_strerror(fd_status s); /* static string for a status code      */
const char *fd_last_error(void);      /* thread-local detail of the last error */

/* ------------------------------------------------------ interop and hooks */

/* Launch all device work of ctx on this cudaStream_t (e.g. torch's current stream);
 * NULL = the legacy default stream.  Errors: FD_ERR_ARG. */
fd_status fd_set_stream(fd_ctx *ctx, void *cuda_stream);

/* Process-global device allocator (e.g. torch's caching allocator); call before any
 * fd_create.  alloc(bytes, user) returns device memory or NULL; free_(ptr, user).
 * Passing NULL for both restores cudaMalloc/cudaFree.  Errors: FD_ERR_STATE if
 * contexts are alive. */
fd_status fd_set_allocator(void *(*alloc)(size_t bytes, void *user),
                           void (*free_)(void *ptr, void *user), void *user);

/* Test hook: set P^0 (which = FD_FIELD_CUR) or P^-1 (FD_FIELD_PREV) from host
 * (prod(local dims) floats).  Only before the first fd_step, else FD_ERR_STATE. */
fd_status fd_set_wavefield(fd_ctx *ctx, int which, const float *host_in);

/* Tuning / debug options; set before the first fd_step (else FD_ERR_STATE).
 *   FD_OPT_KERNEL    0 auto (fused TMA kernel), 1 naive reference kernels (debug,
 *                    three launches per step), 2 fused TMA kernel, 3 the paper's
 *                    unfused decomposition (Listing 3: fd_pzz, [fd_pyy], fd_pxx,
 *                    fd_time as separate kernels with derivative fields; the
 *                    Fig. 5 experiment); all bitwise equal
 *   FD_OPT_TILE      index into the compiled tile table (-1 = auto); see fd_get_info
 *   FD_OPT_ZCHUNKS   z-chunks per x-y tile column (0 = auto)
 *   FD_OPT_ASYNC     1: fd_step returns without synchronising the stream
 *   FD_OPT_GRAPH     1: replay fd_step's launches from CUDA graphs (default 1)
 *   FD_OPT_VSLABS    n >= 1: split the grid into n z-slabs on this one GPU with
 *                    device-copy halo exchange (tests the slab logic)
 *   FD_OPT_PROFILE   1: bracket every launch with CUDA events (fd_get_kernel_times)
 *   FD_OPT_TSTEPS    0 (default) auto: 2 for 3D order 2 and 2D orders 2 and 4 (where
 *                    it is faster) without a pinned FD_OPT_TILE, else 1.  1: one
 *                    step per launch.
 *                    2: temporal blocking -- one launch advances two steps (reads
 *                    p, p_prev, K once, writes both new fields: 10 B instead of
 *                    16 B per grid-point update); bitwise equal
 *                    to single steps.  2D and 3D, orders 2-8; on z-slabs
 *                    (ranks, FD_OPT_VSLABS) 2r + r halo planes per two steps.
 *                    3 or 4: S steps per launch on 2D single-slab contexts
 *                    without the sponge frame, orders with (S-1) r <= 4
 *                    (20 B per point per S updates); other
 *                    contexts FD_ERR_STATE at the first fd_step.  Step counts
 *                    that are not multiples of S end with single steps.
 *   FD_OPT_TB2TILE   index of the temporal-blocking tile configuration (-1 auto)
 *   FD_OPT_RESERVE   n >= 0: finish setup now -- allocate the step tables for n more
 *                    steps and capture the CUDA graphs the next fd_step calls will
 *                    replay -- so no allocation, synchronisation or capture happens
 *                    inside a later timed fd_step (marks the context started)
 *   FD_OPT_RESIDENT  0 (default) auto: single-slab grids of <= 2^17 points with no
 *                    pinned FD_OPT_TILE / FD_OPT_TSTEPS run each fd_step(n) call as
 *                    ONE launch of one thread-block cluster that keeps p, p_prev
 *                    and K in its shared memory for all n steps (halo planes pushed
 *                    through DSMEM, one cluster barrier per step);
 *                    bitwise equal to the other kernels.  1: off.  2: on
 *                    (FD_ERR_STATE at the first fd_step if the grid does not fit)
 *   FD_OPT_CLUSTER   cluster size of FD_OPT_RESIDENT (0 auto = the largest of
 *                    16, 8, 4, 2 that fits; else 2, 4, 8 or 16)
 *   FD_OPT_TRANSPORT halo transport on z-slabs: 0 (default) NCCL send/recv across
 *                    ranks, device copies across virtual slabs; 1 peer: the
 *                    boundary-plane launches store their planes into the
 *                    neighbours' halos in the kernel epilogue (virtual slabs: no
 *                    copies; ranks: fd_peer_export / fd_peer_import, flag sync)
 *   FD_OPT_KPLANE    0 (default) off; 1: when K = (v dt/h)^2/scale is constant on
 *                    every plane of the slow axis (z in 3D, rows in 2D: layered
 *                    and homogeneous models), the tiled kernels read K per plane
 *                    from a table of the same fp32 values instead of streaming
 *                    the K field (SURVEY 8(f) N4 "reduced-byte K"): 12 B instead
 *                    of 16 B per single-step update, 16 B instead of 20 B per
 *                    two-step launch; bitwise the same results.  Checked on the
 *                    device at the first fd_step (bit equality per plane); if
 *                    any plane varies the K field is used.  fd_get_info reports
 *                    which (kplane).  Not with the peer transport across ranks.
 * FD_OPT_ASYNC, FD_OPT_PROFILE and FD_OPT_RESERVE may be set at any time; the others only before
 * the first fd_step.  Errors: FD_ERR_ARG (unknown key / bad value), FD_ERR_STATE. */
enum { FD_OPT_KERNEL = 1, FD_OPT_TILE = 2, FD_OPT_ZCHUNKS = 3, FD_OPT_ASYNC = 4,
       FD_OPT_GRAPH = 5, FD_OPT_VSLABS = 6, FD_OPT_PROFILE = 7, FD_OPT_TSTEPS = 8,
       FD_OPT_TB2TILE = 9, FD_OPT_RESERVE = 10, FD_OPT_RESIDENT = 11, FD_OPT_CLUSTER = 12,
       FD_OPT_TRANSPORT = 13, FD_OPT_KPLANE = 14 };
fd_status fd_set_option(fd_ctx *ctx, int key, int64_t value);

/* Device time per kernel kind accumulated while FD_OPT_PROFILE = 1 (ms and launch
 * counts, arrays of FD_K_COUNT).  Synchronises with the pending events.
 * FD_K_HALO times the halo exchange (copies / NCCL), not a kernel of ours. */
enum { FD_K_FUSED = 0, FD_K_NAIVE = 1, FD_K_GATHER = 2, FD_K_INJECT = 3, FD_K_PXX = 4,
       FD_K_PYY = 5, FD_K_PZZ = 6, FD_K_TIME = 7, FD_K_HALO = 8, FD_K_RESIDENT = 9,
       FD_K_COUNT = 10 };
fd_status fd_get_kernel_times(fd_ctx *ctx, double *ms, int64_t *launches);
fd_status fd_reset_kernel_times(fd_ctx *ctx);

/* Introspection (bench / tests). */
typedef struct {
    int64_t steps_done;        /* k                                                     */
    int64_t kernel_launches;   /* device kernels launched by this context so far         */
    int64_t local_dims[3];     /* slow->fast (unused trailing entries 0)                 */
    int64_t z0, z1;            /* owned global planes                                    */
    int64_t pitch;             /* floats per stored row (>= nx, multiple of 32)          */
    int kernel;                /* 1 naive, 2 fused TMA, 3 unfused decomposition          */
    int tile_x, tile_y, rows_per_thread, p_stages, k_stages;
    int ctas, threads_per_cta, smem_bytes, zchunks;
    int order;
    double device_bytes;       /* bytes of device memory held                           */
    int steps_per_launch;      /* 2 with temporal blocking (FD_OPT_TSTEPS), 0 when each  */
                               /* fd_step call is one cluster launch (FD_OPT_RESIDENT), else 1 */
    int cluster_ctas;          /* CTAs of the resident cluster (FD_OPT_RESIDENT), else 0 */
    int kplane;                /* 1 when the kernels read K per plane (FD_OPT_KPLANE)    */
    int comm_nranks;           /* ranks of the NCCL communicator (ncclCommCount; 0: none) */
    int64_t graph_steps;       /* steps advanced by CUDA-graph replay so far             */
    int tb_kind;               /* multi-step kernel family: 0 TMA-staged tiles (tb2ws,
                                  tb2d, tbs2d), 1 register-streamed 2D strips (rs2d)    */
} fd_info;
fd_status fd_get_info(fd_ctx *ctx, fd_info *out);

#ifdef __cplusplus
}
#endif
#endif /* FD_H */
