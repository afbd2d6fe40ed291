// fd_runtime.cu -- host runtime and C ABI (include/fd.h) of the B200-native
// acoustic FD hot path.  One fused kernel launch per time step; device buffers
// A/B rotate by pointer swap (Listing 3); K = (v dt/h)^2/scale is the
// per-point coefficient (R#7).  See DESIGN.md sections 5-7.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/fd.h"
#include "fd_kernels.cuh"
#include "fd_tables.cuh"
#include "fd_resident.cuh"

using namespace fdk;

// --------------------------------------------------------------------- errors
static thread_local std::string g_last_error;

static fd_status fail(fd_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

#define CUDA_TRY(ctx, expr)                                                                     \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess) {                                                                \
            if (ctx) (ctx)->poisoned = true;                                                    \
            return fail(FD_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),    \
                        __FILE__, __LINE__);                                                    \
        }                                                                                       \
    } while (0)

// ------------------------------------------------------------------ allocator
static void *(*g_alloc)(size_t, void *) = nullptr;
static void (*g_free)(void *, void *) = nullptr;
static void *g_alloc_user = nullptr;
static int g_live_contexts = 0;
static std::mutex g_mu;

static void *dev_alloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (g_alloc) return g_alloc(bytes, g_alloc_user);
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    return p;
}
static void dev_free(void *p) {
    if (!p) return;
    if (g_free) g_free(p, g_alloc_user);
    else cudaFree(p);
}

// ----------------------------------------------------- driver entry (TMA maps)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

// 3D fp32 tensor map over a pitched field: dims (nx, ny, planes), box (bx, by, 1);
// out-of-bounds elements (x < 0, x >= nx, y < 0, y >= ny) are filled with zeros.
static bool make_map(CUtensorMap *m, const float *base, int64_t nx, int64_t ny, int64_t planes, int64_t pitch,
                     int bx, int by, int bz = 1) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * 4), (cuuint64_t)(pitch * ny * 4)};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// ------------------------------------------------------------ kernel tables
// The tiled kernels' compiled configurations live in fd_tab_*.cu (separate
// translation units, compiled in parallel); fd_tables.cuh declares them.
static const std::vector<TileCfg> &tile_table() {
    static const std::vector<TileCfg> t = [] {
        std::vector<TileCfg> v;
        for (auto part : {fdtab::tiles3d_r12, fdtab::tiles3d_r34, fdtab::tiles2d}) {
            auto p = part();
            v.insert(v.end(), p.begin(), p.end());
        }
        return v;
    }();
    return t;
}
static const std::vector<TileCfg> &tb2_table() {
    static const std::vector<TileCfg> t = [] {
        std::vector<TileCfg> v;
        for (auto part : {fdtab::tb2ws, fdtab::tb2d, fdtab::rs2d, fdtab::rs2d_x, fdtab::tbs2d}) {
            auto p = part();
            v.insert(v.end(), p.begin(), p.end());
        }
        return v;
    }();
    return t;
}

// ------------------------------------------------------------------ NCCL (dlopen)
// NCCL is loaded at run time (libnccl.so.2: torch's bundled copy when torch has
// loaded it, else the system one) so the library loads on machines without it.
typedef void *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclFloat32 = 7 };
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
static NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
#define NCCL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
            NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
            NCCL_SYM(CommInitRank, "ncclCommInitRank");
            NCCL_SYM(CommDestroy, "ncclCommDestroy");
            NCCL_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
            NCCL_SYM(CommCount, "ncclCommCount");
            NCCL_SYM(Send, "ncclSend");
            NCCL_SYM(Recv, "ncclRecv");
            NCCL_SYM(GroupStart, "ncclGroupStart");
            NCCL_SYM(GroupEnd, "ncclGroupEnd");
            NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef NCCL_SYM
            api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
                     api.GroupStart && api.GroupEnd && api.GetErrorString;
        }
    }
    return api;
}

// ------------------------------------------------------------------ context
struct SourceDef {
    int64_t g[3];     // global (z, y, x)
    double f, t0, amp;
};
struct RecDef {
    int64_t g[3];
};

// One kernel launch per step over local planes [zlo, zhi) of a slab.
struct Region {
    int32_t zlo = 0, zhi = 0;
    int zchunks = 1;
    int lin = 0;                // tb2d linear mode: units (one wave) sharing the region's blocks; 0: chunked
    int ctas = 0;
    bool boundary = false;      // launched on the comm stream before the exchange
    int32_t *d_rec = nullptr;   // [4 * nrec + units + 1]: z, y, x, id, CSR offsets
    unsigned long long *d_ws = nullptr;   // rs2d work-stealing words, one per warp (fd_rs2d.cuh)
    int nws = 0;
    int nrec = 0;
};

// A z-slab [z0, z1) of the global grid with its own buffers (field buffers:
// halo_planes(r) = 2r planes on each side; K: r).  One per context, except
// FD_OPT_VSLABS (several on one GPU).
struct Slab {
    int64_t z0 = 0, z1 = 0, nz = 0;
    float *F[4] = {nullptr, nullptr, nullptr, nullptr};   // field buffers (F[2], F[3]: TB2 only)
    float *Kh = nullptr;                        // K allocation: r halo planes on each side
    float *K = nullptr;                         // = Kh + r planes (local plane 0)
    float *D[3] = {nullptr, nullptr, nullptr};   // Pxx, Pyy, Pzz (unfused decomposition only)
    float *d_src_raw = nullptr;
    float *kzt = nullptr;                       // FD_OPT_KPLANE: per-plane K, local plane z at kzt[kKzPad + z]
    CUtensorMap mHalo[4], mTile[4], mK;        // single-step kernel maps per field buffer
    CUtensorMap mP0[4], mPm[4], mKe;           // TB2 maps
    std::vector<Region> regions;                // single-step launches
    std::vector<Region> tb2;                    // temporal-blocking launches (own receiver CSRs)
    bool has_lo = false, has_hi = false;        // z-neighbours (rank or virtual slab)
};

struct fd_ctx {
    int ndim = 0, order = 0, R = 0;
    double h = 0, dt = 0;
    int64_t nxg = 0, nyg = 0, nzg = 0;    // global extents (ny = 1 in 2D)
    int64_t z0 = 0, z1 = 0;               // planes owned by this context
    int64_t pitch = 0;
    int rank = 0, nranks = 1, device = 0;
    int H = 0;                            // field-buffer halo planes per side (halo_planes(R))
    bool poisoned = false;
    bool started = false;
    bool injected = false;                // w_k already injected into the CUR buffers
    int64_t k = 0;                        // steps done
    int64_t launches = 0;
    cudaStream_t stream = nullptr;        // user stream (interior kernels)
    cudaStream_t comm_stream = nullptr;   // boundary kernels + NCCL (distributed)
    cudaEvent_t ev_step = nullptr, ev_comm = nullptr;
    int icur = 0, iprev = 1;              // roles of the slabs' field buffers
    std::vector<SourceDef> src;
    std::vector<RecDef> rec;
    std::vector<Slab> slabs;
    float *d_traces = nullptr;            // step-major [trace_cap][nrec]
    int64_t trace_cap = 0;
    float *d_wtab = nullptr;              // [wcap][nsrc]: w_j of source s (fp32 of the fp64 Ricker)
    int64_t wcap = 0;
    int64_t *d_k = nullptr;               // device step counter (graph replays)
    int64_t graph_steps = 0;              // steps advanced by graph replay (fd_get_info)
    cudaStream_t own_stream = nullptr;    // used when no stream was set (capturable)
    // CUDA graphs of G steps (one per starting buffer parity), re-captured when
    // the trace / wavelet tables move
    struct Graph { int icur, iprev, end_icur, end_iprev; cudaGraphExec_t exec; const void *kt, *kw; int64_t launches; };
    std::vector<Graph> graphs;
    bool capturing = false;
    int64_t gk0 = 0;
    // distributed
    ncclComm_t comm = nullptr;
    bool nccl_self = false;               // FD_VSLAB_NCCL=1: virtual-slab halos through NCCL (1-rank comm)
    ncclUniqueId nccl_id;
    bool have_id = false;
    // kernel configuration
    int opt_kernel = 0, opt_tile = -1, opt_zchunks = 0, opt_async = 0, opt_graph = 1, opt_vslabs = 1;
    int opt_profile = 0;
    int opt_tsteps = 0;                   // 0 auto, 1 single steps, S >= 2 temporal blocking (S steps/launch)
    int opt_tb2tile = -1;
    int tb2 = -1, tb2occ = 0;             // chosen tb2_table() entry
    // FD_OPT_RESIDENT: whole fd_step calls in one cluster launch (fd_resident.cuh)
    int opt_resident = 0, opt_cluster = 0;   // 0 auto / 1 off / 2 on; forced cluster size
    bool resident = false;
    int res_nc = 0, res_npmax = 0, res_threads = 0, res_smem = 0;
    int32_t *d_res_rec = nullptr;         // receivers sorted by CTA + offsets
    // FD_OPT_TRANSPORT = 1: in-kernel halo pushes (peer stores) instead of copies / NCCL
    int opt_transport = 0;
    // FD_OPT_KPLANE: K from a per-plane table where it depends on z only
    int opt_kplane = 0;
    bool kplane = false;
    struct Peer {
        float *F[4] = {nullptr, nullptr, nullptr, nullptr};   // the neighbour's field buffers (IPC)
        float *Kh = nullptr;
        int64_t *flags = nullptr;          // the neighbour's flag array
        int64_t nz = 0;
        std::vector<void *> opened;        // IPC mappings to close
    } plo, phi;
    bool peer_imported = false;
    bool frozen = false;                  // fd_peer_export done: options fixed
    int64_t *d_flags = nullptr;           // [0]: written by rank - 1, [1]: by rank + 1 (exchange counts)
    int *h_perr = nullptr, *d_perr = nullptr;   // peer_wait timeout flag (mapped pinned host int)
    bool peer_detached = false;           // fd_peer_detach done: no more steps
    int64_t xcount = 0;                   // exchanges this rank has signalled
    // absorbing sponge frame (fd_set_sponge, R#18)
    int sponge_nb = 0;
    double sponge_alpha = 0;
    float *d_gsp = nullptr;               // g_x[nx], g_y[ny], g_z[nzg] (fp64 profile rounded once)
    bool overlap = false;                 // boundary/interior split on two streams
    int tile = -1, occ = 0, nsm = 148;
    // FD_OPT_PROFILE: CUDA events around every launch, folded into per-kernel sums
    struct Rec { int kid; cudaEvent_t a, b; };
    std::vector<Rec> ev_pending;
    std::vector<cudaEvent_t> ev_pool;
    double kms[FD_K_COUNT] = {0};
    int64_t kcnt[FD_K_COUNT] = {0};
    double dev_bytes = 0;
};

static inline int64_t plane_floats(const fd_ctx *c) { return c->nyg * c->pitch; }
static inline int64_t buf_floats(const fd_ctx *c, const Slab &s) { return (s.nz + 2 * c->H) * plane_floats(c); }
static inline float *cur_buf(const fd_ctx *c, const Slab &s) { return s.F[c->icur]; }
static inline float *prev_buf(const fd_ctx *c, const Slab &s) { return s.F[c->iprev]; }

static double scale_of(int R) { return tap_scale(R); }

// CFL limit of R#8: C_max = 2 / sqrt(D |S(pi)|), S(pi) = sum of the taps with
// alternating signs (integer taps / scale).
static double cfl_limit(int ndim, int R) {
    double s = tap(R, 0);
    for (int m = 1; m <= R; ++m) s += 2.0 * tap(R, m) * ((m & 1) ? -1.0 : 1.0);
    s /= scale_of(R);
    return 2.0 / std::sqrt(ndim * std::fabs(s));
}

// Ricker wavelet, fp64, one rounding to fp32 at the caller.
static double ricker(double t, double f, double t0) {
    const double pi = 3.14159265358979323846;
    const double a = pi * pi * f * f * (t - t0) * (t - t0);
    return (1.0 - 2.0 * a) * std::exp(-a);
}

static fd_status partition(int64_t nz, int nranks, int rank, int64_t *z0, int64_t *z1) {
    if (nranks < 1 || rank < 0 || rank >= nranks || nz < nranks || !z0 || !z1)
        return fail(FD_ERR_ARG, "fd_partition: bad arguments (nz=%lld nranks=%d rank=%d)", (long long)nz, nranks,
                    rank);
    const int64_t base = nz / nranks, extra = nz % nranks;
    *z0 = rank * base + std::min<int64_t>(rank, extra);
    *z1 = *z0 + base + (rank < extra ? 1 : 0);
    return FD_OK;
}

static void free_slab(Slab &s) {
    for (auto &d : s.D) { dev_free(d); d = nullptr; }
    for (auto &f : s.F) { dev_free(f); f = nullptr; }
    dev_free(s.Kh); dev_free(s.d_src_raw); dev_free(s.kzt);
    s.Kh = s.K = s.d_src_raw = s.kzt = nullptr;
    for (auto &r : s.regions) { dev_free(r.d_rec); r.d_rec = nullptr; }
    for (auto &r : s.tb2) { dev_free(r.d_rec); r.d_rec = nullptr; dev_free(r.d_ws); r.d_ws = nullptr; }
}

static void drop_graphs(fd_ctx *c) {
    for (auto &g : c->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
}

static void destroy_all(fd_ctx *c) {
    drop_graphs(c);
    for (auto &s : c->slabs) free_slab(s);
    dev_free(c->d_traces);
    dev_free(c->d_wtab);
    dev_free(c->d_k);
    dev_free(c->d_res_rec);
    dev_free(c->d_gsp);
    c->d_gsp = nullptr;
    for (auto *pr : {&c->plo, &c->phi})
        for (void *m : pr->opened) cudaIpcCloseMemHandle(m);
    c->plo.opened.clear(); c->phi.opened.clear();
    if (c->d_flags) cudaFree(c->d_flags);
    c->d_flags = nullptr;
    if (c->h_perr) cudaFreeHost(c->h_perr);
    c->h_perr = c->d_perr = nullptr;
    c->d_traces = nullptr; c->d_wtab = nullptr; c->d_k = nullptr; c->d_res_rec = nullptr;
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    c->own_stream = nullptr;
    if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
    c->comm = nullptr;
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    for (auto &r : c->ev_pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    c->ev_pending.clear(); c->ev_pool.clear();
    if (c->ev_step) cudaEventDestroy(c->ev_step);
    if (c->ev_comm) cudaEventDestroy(c->ev_comm);
    c->comm_stream = nullptr; c->ev_step = c->ev_comm = nullptr;
}

// Allocate a slab's buffers and upload its K: from host velocities v (the
// slab's planes; K halos zero until exchanged), or -- when v is NULL -- copied
// with its r halo planes from a device K-halo buffer kdevh (planes z - r ..).
// Allocate a slab's buffers (fields zeroed); K is copied from kdevh (another
// context's K halo buffer: virtual slabs) or zeroed for the caller's upload.
static fd_status build_slab(fd_ctx *c, Slab &s, const float *kdevh) {
    const size_t fbytes = (size_t)buf_floats(c, s) * 4;
    const size_t kbytes = (size_t)((s.nz + 2 * c->R) * plane_floats(c)) * 4;
    s.F[0] = (float *)dev_alloc(fbytes);
    s.F[1] = (float *)dev_alloc(fbytes);
    s.Kh = (float *)dev_alloc(kbytes);
    s.K = s.Kh ? s.Kh + c->R * plane_floats(c) : nullptr;
    s.d_src_raw = (float *)dev_alloc(kMaxSources * 4);
    if (!s.F[0] || !s.F[1] || !s.Kh || !s.d_src_raw)
        return fail(FD_ERR_NOMEM, "device allocation of %.3f GB failed", (2.0 * fbytes + kbytes) / 1e9);
    c->dev_bytes += 2.0 * fbytes + kbytes;
    if (kdevh) CUDA_TRY(c, cudaMemcpy(s.Kh, kdevh, kbytes, cudaMemcpyDeviceToDevice));
    else CUDA_TRY(c, cudaMemset(s.Kh, 0, kbytes));      // K uploaded by the caller (create_impl)
    CUDA_TRY(c, cudaMemset(s.F[0], 0, fbytes));
    CUDA_TRY(c, cudaMemset(s.F[1], 0, fbytes));
    CUDA_TRY(c, cudaMemset(s.d_src_raw, 0, kMaxSources * 4));
    return FD_OK;
}

static int64_t scan_velocity(const float *v, int64_t n, double *vmax_out) {
    int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), 32);
    nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, n / (1 << 20) + 1));
    std::vector<float> vm((size_t)nt, 0.f);
    std::vector<int64_t> bad((size_t)nt, -1);
    auto work = [&](int t) {
        const int64_t a = n * t / nt, b = n * (t + 1) / nt;
        float m = 0.f;
        for (int64_t i0 = a; i0 < b; i0 += 4096) {
            const int64_t i1 = std::min<int64_t>(b, i0 + 4096);
            int ok = 1;
            float bm = 0.f;
            for (int64_t i = i0; i < i1; ++i) {
                const float x = v[i];
                ok &= (x > 0.f) & (x <= 3.402823466e38f);     // > 0, not NaN, not +inf
                bm = x > bm ? x : bm;
            }
            if (!ok) {
                for (int64_t i = i0; i < i1; ++i)
                    if (!(v[i] > 0.f) || !std::isfinite(v[i])) { bad[t] = i; return; }
            }
            m = std::max(m, bm);
        }
        vm[t] = m;
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto &x : th) x.join();
    double vmax = 0;
    for (int t = 0; t < nt; ++t) {
        if (bad[t] >= 0) return bad[t];
        vmax = std::max(vmax, (double)vm[t]);
    }
    *vmax_out = vmax;
    return -1;
}

static fd_status create_impl(fd_ctx **out, int ndim, const int64_t *dims, double h, double dt, int order,
                             const float *vel, uint32_t flags, int rank, int nranks, int device, int vel_is_slab,
                             const void *nccl_id) {
    if (!out) return fail(FD_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (ndim != 2 && ndim != 3) return fail(FD_ERR_ARG, "ndim must be 2 or 3 (got %d)", ndim);
    if (!dims || !vel) return fail(FD_ERR_ARG, "dims/vel is NULL");
    if (order != 2 && order != 4 && order != 6 && order != 8)
        return fail(FD_ERR_ARG, "order must be 2, 4, 6 or 8 (got %d)", order);
    if (!(h > 0) || !std::isfinite(h)) return fail(FD_ERR_ARG, "h must be > 0");
    if (!(dt > 0) || !std::isfinite(dt)) return fail(FD_ERR_ARG, "dt must be > 0");
    const int R = order / 2;
    for (int a = 0; a < ndim; ++a)
        if (dims[a] < 2 * R + 1)
            return fail(FD_ERR_ARG, "dims[%d]=%lld smaller than the stencil (%d)", a, (long long)dims[a], 2 * R + 1);
    int64_t nzg = dims[0], nyg = ndim == 3 ? dims[1] : 1, nxg = dims[ndim - 1];
    if (nxg > (int64_t)1 << 30 || nyg > (int64_t)1 << 30 || nzg > (int64_t)1 << 30)
        return fail(FD_ERR_ARG, "dims too large");
    // the step kernels keep in-plane offsets (y * pitch + x, pitch = nx rounded
    // up to 32 floats) in 32 bits; one 64-bit base per plane
    if (ndim == 3 && (nyg + 4 * R) * ((nxg + 31) / 32 * 32 + 32) >= ((int64_t)1 << 31))
        return fail(FD_ERR_ARG, "plane of %lld x %lld points too large (32-bit in-plane offsets)",
                    (long long)nyg, (long long)nxg);
    int64_t z0 = 0, z1 = nzg;
    if (nranks > 1 || rank != 0) {
        fd_status s = partition(nzg, nranks, rank, &z0, &z1);
        if (s) return s;
        if (nranks > 1 && z1 - z0 < 2 * R)
            return fail(FD_ERR_ARG, "slab of %lld planes thinner than 2r=%d", (long long)(z1 - z0), 2 * R);
    }
    const int64_t nz = z1 - z0;
    const int64_t plane = nyg * nxg;
    const float *vloc = vel + (vel_is_slab ? 0 : z0 * plane);
    const int64_t nloc = nz * plane;
    const double lim = cfl_limit(ndim, R);
    auto cfl_fail = [&](double vmax) -> fd_status {
        const double ratio = vmax * dt / h;
        if (!(flags & FD_FLAG_ALLOW_UNSTABLE) && ratio > lim)
            return fail(FD_ERR_UNSTABLE, "unstable: max(v)*dt/h = %.6f exceeds the CFL limit %.6f (ratio %.4f)",
                        ratio, lim, ratio / lim);
        return FD_OK;
    };
    auto bad_fail = [&](int64_t i) {
        return fail(FD_ERR_ARG, "velocity[%lld] = %g is not finite and > 0", (long long)i, (double)vloc[i]);
    };
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        // no device: the host validation still decides the error class
        cudaGetLastError();
        double vmax = 0;
        const int64_t bad = scan_velocity(vloc, nloc, &vmax);
        if (bad >= 0) return bad_fail(bad);
        fd_status s = cfl_fail(vmax);
        if (s) return s;
        return fail(FD_ERR_CUDA, "no CUDA device available");
    }
    if (device >= 0) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return fail(FD_ERR_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
    }
    fd_ctx *c = new fd_ctx();
    c->ndim = ndim; c->order = order; c->R = R; c->H = halo_planes(R); c->h = h; c->dt = dt;
    c->nxg = nxg; c->nyg = nyg; c->nzg = nzg; c->z0 = z0; c->z1 = z1;
    c->rank = rank; c->nranks = nranks;
    cudaGetDevice(&c->device);
    cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device);
    c->pitch = (nxg + 31) / 32 * 32;
    if (nranks > 1 && nccl_id) {
        memcpy(&c->nccl_id, nccl_id, sizeof(ncclUniqueId));
        c->have_id = true;
    }
    // one slab now; FD_OPT_VSLABS re-splits before the first step (keeps the model)
    c->slabs.resize(1);
    Slab &s = c->slabs[0];
    s.z0 = z0; s.z1 = z1; s.nz = nz;
    fd_status st = build_slab(c, s, nullptr);
    if (st == FD_OK) {
        // Model upload (P:119 copy-in): one H2D copy into the pitched K buffer,
        // then one kernel converts v to K and validates the model on the device
        // (finite and > 0, the max for the CFL check of R#8) -- a host scan of
        // the model cost as much as the copy (C3: 512 MB); an invalid model
        // frees everything and reports as the host check did.
        unsigned *d_vmax = nullptr;
        unsigned long long *d_bad = nullptr;
        cudaError_t e = cudaMalloc(&d_vmax, 16);    // [0]: max bits, bytes 8..15: bad index
        if (e == cudaSuccess) {
            d_bad = reinterpret_cast<unsigned long long *>(d_vmax + 2);
            e = cudaMemset(d_vmax, 0, sizeof(unsigned));
        }
        if (e == cudaSuccess) e = cudaMemset(d_bad, 0xff, sizeof(unsigned long long));
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(s.K, c->pitch * 4, vloc, nxg * 4, nxg * 4, nyg * nz, cudaMemcpyHostToDevice, 0);
        if (e == cudaSuccess) {
            const int64_t rows = nyg * nz;
            const int blocks = (int)std::min<int64_t>((rows * nxg + 255) / 256, 148 * 32);
            velocity_to_K_kernel<<<blocks, 256>>>(s.K, rows, nxg, c->pitch, dt, h, scale_of(R), 0, d_vmax, d_bad);
            e = cudaGetLastError();
        }
        unsigned vbits = 0;
        unsigned long long bad = ~0ull;
        if (e == cudaSuccess) e = cudaMemcpy(&vbits, d_vmax, sizeof vbits, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost);
        if (d_vmax) cudaFree(d_vmax);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        float vmaxf;
        memcpy(&vmaxf, &vbits, sizeof vmaxf);
        if (e != cudaSuccess) st = fail(FD_ERR_CUDA, "device setup failed: %s", cudaGetErrorString(e));
        else if (bad != ~0ull) st = bad_fail((int64_t)bad);
        else st = cfl_fail((double)vmaxf);
    }
    if (st != FD_OK) {
        destroy_all(c);
        delete c;
        return st;
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        ++g_live_contexts;
    }
    *out = c;
    return FD_OK;
}

// ------------------------------------------------------------ kernel choice
// Resident CTAs per SM of a configuration: the minimum over the compiled
// variants this context may launch (band rule or sponge, with or without the
// peer pushes, with or without per-plane K) -- not over every variant: a
// heavier unused one must not halve the chunking's slot count.
static int occupancy(const fd_ctx *c, const TileCfg &t) {
    const int base = c->sponge_nb > 0 ? kVarSponge : 0;
    int best = -1;
    for (int v = 0; v < kVariants; ++v) {
        if (!t.kernel[v]) continue;
        if ((v & kVarSponge) != base) continue;
        if ((v & kVarPeer) && c->opt_transport != 1) continue;
        if ((v & kVarKPlane) && !c->opt_kplane) continue;
        int n = 0;
        cudaFuncSetAttribute(t.kernel[v], cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, t.kernel[v], t.threads, t.smem) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        best = best < 0 ? n : std::min(best, n);
    }
    return std::max(best, 0);
}

static int64_t ntiles_of(const fd_ctx *c, const TileCfg &t) {
    return ((c->nxg + t.tx - 1) / t.tx) * ((c->nyg + t.ty - 1) / t.ty);
}

// z-chunks for a span of planes: fill one wave of resident CTAs (chunk-major
// order keeps neighbours in step for L2 halo reuse), chunks >= max(4r, 8) planes.
// z-chunks for a span of planes.  Measured on B200 (scripts/tune.py,
// profiles/tune_r01.md): several waves of short-ish units beat one wave of
// long ones (better balance across the 148 SMs), and within that the wave
// fill units / (waves * slots) decides.  Aim at ~6 waves (3D) / ~3 waves (2D,
// whose CTAs are short), then pick among nearby counts the best
// fill x (chunk / (chunk + warm-up planes)).
static int chunks_for(const fd_ctx *c, const TileCfg &t, int occ, int64_t span) {
    if (t.kind == 1) return 1;   // rs2d: one receiver list per column strip, persistent grid (rs2d_ctas)
    if (c->opt_zchunks > 0) return (int)std::min<int64_t>(c->opt_zchunks, std::max<int64_t>(1, span));
    const int64_t slots = (int64_t)c->nsm * std::max(occ, 1), ntiles = ntiles_of(c, t);
    // 3D: chunks of >= max(4r, 8) planes (the 2r warm-up planes stay small);
    // 2D: >= 2 row blocks per chunk
    const int64_t minp = c->ndim == 3 ? std::max(4 * c->R, 8) : 2 * t.ty;
    const int64_t chmax = std::max<int64_t>(1, span / minp);
    // 2D two-step launches (tb2d, whose A -> B lag is one row block per chunk)
    // prefer ~2 full waves of longer chunks (r05 sweep on C2 order 2: 9 chunks
    // = 1.95 waves 570 Gpts/s vs 13 = 2.8 waves 556)
    const bool tb2d = c->ndim == 2 && c->tb2 >= 0 && &t == &tb2_table()[c->tb2];
    const int64_t waves_target = c->ndim == 3 ? 6 : (tb2d ? 2 : 3);
    const int64_t target = std::max<int64_t>(1, (waves_target * slots + ntiles / 2) / ntiles);
    // 3D: z-chunks of at most 128 planes.  The co-resident CTAs of a wave
    // stream neighbouring tiles through z in step and share their x-y halos
    // in L2; over longer chunks they drift apart and the halos come from DRAM
    // again (r2, C4 1024^3 two-step: 2 chunks of 512 planes 572 Gpts/s with
    // 14.3 GB read per launch, 8 chunks of 128 planes 626; C5:1 603 -> 623)
    const int64_t chmin = c->ndim == 3 ? std::min<int64_t>(chmax, (span + 127) / 128) : 1;
    int64_t best = 1;
    double bscore = -1;
    for (int64_t ch = std::max<int64_t>({(int64_t)1, target - 3, chmin}); ch <= std::max(target, chmin) + 3; ++ch) {
        const int64_t cc = std::min(ch, chmax);
        const int64_t units = ntiles * cc, waves = (units + slots - 1) / slots;
        const double fill = (double)units / (double)(waves * slots);
        const double len = (double)span / (double)cc;
        // ~half the 2r warm-up planes' cost (3D); the A -> B lag of one row
        // block per chunk (2D two-step)
        const double warm = c->ndim == 3 ? c->R : (tb2d ? (double)t.ty * (t.steps - 1) : 0.0);
        const double score = fill * len / (len + warm);
        if (score > bscore + 1e-9) { bscore = score; best = cc; }
    }
    return (int)best;
}

// rs2d (register-streamed 2D strips): a persistent grid -- one wave of resident
// CTAs, fewer when the region has under 16 rows per warp -- whose warps cut
// the column strips into pieces and balance by work stealing (fd_rs2d.cuh).
// FD_OPT_ZCHUNKS pins the CTA count (tests: a few warps, many pieces each).
static int rs2d_ctas(const fd_ctx *c, const TileCfg &t, int occ, int64_t span) {
    if (c->opt_zchunks > 0) return (int)std::min<int64_t>(c->opt_zchunks, (int64_t)c->nsm * std::max(occ, 1));
    const int64_t ntx = (c->nxg + t.tx - 1) / t.tx;
    const int64_t want = (ntx * span + (int64_t)t.ny * 16 - 1) / ((int64_t)t.ny * 16);
    return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->nsm * std::max(occ, 1), want));
}

// 2D two-step launches (tb2d) can split the region's ntx * nb row blocks into
// one wave of equal contiguous ranges ("linear" units that cross column
// boundaries): one pipeline warm-up per CTA and no wave tail, vs the chunked
// split's whole columns x z-chunks.  Opt-in (FD_TB2D_LINEAR=1): r2 A/B on C2
// (Gpts/s, linear vs chunked) 64-column tiles 331 vs 556 (order 2) and 319
// vs 501 (order 4) -- the co-running CTAs sit ~900 rows apart in the same
// columns instead of side by side in one z band, and lose the L2 sharing of
// the x halos; 56-column tiles 547 vs 535 and 512 vs 490.  FD_OPT_ZCHUNKS
// pins the chunked split.
static int lin_units(const fd_ctx *c, const TileCfg &t, int occ, int64_t span) {
    const bool tb2d = c->ndim == 2 && c->tb2 >= 0 && &t == &tb2_table()[c->tb2];
    static const bool on = [] { const char *e = getenv("FD_TB2D_LINEAR"); return e && e[0] == '1'; }();
    if (!tb2d || t.kind != 0 || c->opt_zchunks > 0 || !on) return 0;
    const int64_t nb = (span + t.ty - 1) / t.ty, V = ((c->nxg + t.tx - 1) / t.tx) * nb;
    return (int)std::max<int64_t>(1, std::min<int64_t>(V, (int64_t)c->nsm * std::max(occ, 1)));
}

// Preferred tile per (ndim, r), from the r01 sweep: 3D r=1 128x16 (428 Gpts/s
// on C3), r=2 128x32 (410), r>=3 64x16 with 2 rows/thread (379 at r=4); 2D
// 64x32 blocks with 3 ring slots (363 / 347 on C2).  Falls back to the first
// tile that fits when the preferred one does not.
static bool preferred(const fd_ctx *c, const TileCfg &t) {
    if (c->ndim == 3) {
        if (c->R == 1) return t.tx == 128 && t.ty == 16 && t.dp == 2;
        if (c->R == 2) return t.tx == 128 && t.ty == 32 && t.dp == 2;
        return t.tx == 64 && t.ty == 16 && t.ny == 2 && t.dp == 2;
    }
    return t.tx == 64 && t.ty == 32 && t.ny == 4 && t.dp == 3;
}

// The sponge frame and the peer transport run the kernel variants compiled
// for the "full" table entries only.
static bool needs_full(const fd_ctx *c) { return c->sponge_nb > 0 || c->opt_transport == 1; }
// FD_OPT_KPLANE is optional: a pinned tuning-only tile (no KZ variants) keeps
// the K field instead of failing
static bool prefers_full(const fd_ctx *c) { return needs_full(c) || c->opt_kplane; }

static void choose_tile(fd_ctx *c, int64_t span) {
    (void)span;
    const auto &tab = tile_table();
    int bi = -1, bocc = 0;
    for (int pass = 0; pass < 2 && bi < 0; ++pass)
        for (int i = 0; i < (int)tab.size(); ++i) {
            const TileCfg &t = tab[i];
            if (t.ndim != c->ndim || t.r != c->R) continue;
            if (c->opt_tile >= 0 ? i != c->opt_tile : (pass == 0 && !preferred(c, t))) continue;
            if (needs_full(c) && !t.full()) continue;   // sponge / peer variants compiled for full entries
            if (pass == 0 && c->opt_tile < 0 && prefers_full(c) && !t.full()) continue;
            const int occ = occupancy(c, t);
            if (occ <= 0) continue;
            bi = i; bocc = occ;
            break;
        }
    c->tile = bi;
    c->occ = bocc;
}

static fd_status make_maps(fd_ctx *c, Slab &s) {
    const TileCfg &t = tile_table()[c->tile];
    const int64_t planes = s.nz + 2 * c->H;
    // 3D: boxes (x, y) of one plane; 2D: boxes of pbz / tbz rows (nyg = 1)
    const int hy = c->ndim == 3 ? c->R : 0;
    const int pby = c->ndim == 3 ? t.ty + 2 * hy : 1, tby = c->ndim == 3 ? t.ty : 1;
    bool ok = make_map(&s.mK, s.K, c->nxg, c->nyg, s.nz, c->pitch, t.tbw, tby, t.tbz);
    for (int b = 0; b < 4 && ok; ++b) {
        if (!s.F[b]) continue;
        ok = make_map(&s.mHalo[b], s.F[b], c->nxg, c->nyg, planes, c->pitch, t.pbw, pby, t.pbz) &&
             make_map(&s.mTile[b], s.F[b], c->nxg, c->nyg, planes, c->pitch, t.tbw, tby, t.tbz);
    }
    if (!ok) {
        c->poisoned = true;
        return fail(FD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    }
    return FD_OK;
}

// Receivers of a region, sorted by (work unit, z) with CSR offsets per unit
// (fused kernel) -- or a flat list (naive kernel).
static fd_status upload_region_receivers(fd_ctx *c, const Slab &s, Region &g, const TileCfg *t) {
    dev_free(g.d_rec);
    g.d_rec = nullptr;
    struct L { int32_t unit, z, y, x, id, key; };
    std::vector<L> loc;
    int ntx = 1, ntiles = 1;
    if (t) {
        ntx = (int)((c->nxg + t->tx - 1) / t->tx);
        ntiles = (int)ntiles_of(c, *t);
    }
    const int64_t span = g.zhi - g.zlo;
    for (size_t j = 0; j < c->rec.size(); ++j) {
        const int64_t lz = c->rec[j].g[0] - s.z0;
        if (lz < g.zlo || lz >= g.zhi) continue;
        L l{0, (int32_t)lz, (int32_t)c->rec[j].g[1], (int32_t)c->rec[j].g[2], (int32_t)j, 0};
        if (t && g.lin > 0) {
            // linear units (tb2d): block v = column * nb + row block, unit u
            // holds [V u / G, V (u+1) / G); sorted by (unit, v, z)
            const int64_t nb = (span + t->ty - 1) / t->ty, V = (int64_t)ntx * nb;
            const int64_t v = (l.x / t->tx) * nb + (lz - g.zlo) / t->ty;
            l.unit = (int32_t)(((v + 1) * g.lin - 1) / V);
            l.key = (int32_t)v;
        } else if (t) {
            // the chunk containing plane lz, as the kernels split [zlo, zhi):
            // 3D by planes, 2D by whole blocks of ty rows
            int ch = 0;
            const int64_t nb = (span + t->ty - 1) / t->ty;
            for (int q = 0; q < g.zchunks; ++q) {
                const int64_t first = c->ndim == 3 ? g.zlo + (span * q) / g.zchunks
                                                   : g.zlo + ((nb * q) / g.zchunks) * t->ty;
                if (first <= lz) ch = q;
            }
            l.unit = ch * ntiles + (c->ndim == 3 ? (l.y / t->ty) * ntx : 0) + (l.x / t->tx);
        }
        loc.push_back(l);
    }
    std::stable_sort(loc.begin(), loc.end(), [](const L &a, const L &b) {
        return a.unit != b.unit ? a.unit < b.unit : (a.key != b.key ? a.key < b.key : a.z < b.z);
    });
    const int nunits = t ? (g.lin > 0 ? g.lin : ntiles * g.zchunks) : 0;
    const int n = (int)loc.size();
    g.nrec = n;
    std::vector<int32_t> h((size_t)4 * n + nunits + 1, 0);
    for (int i = 0; i < n; ++i) {
        h[i] = loc[i].z; h[n + i] = loc[i].y; h[2 * n + i] = loc[i].x; h[3 * n + i] = loc[i].id;
    }
    int32_t *off = h.data() + 4 * n;
    for (int u = 0, i = 0; u <= nunits; ++u) {
        while (i < n && loc[i].unit < u) ++i;
        off[u] = i;
    }
    g.d_rec = (int32_t *)dev_alloc(h.size() * 4);
    if (!g.d_rec) return fail(FD_ERR_NOMEM, "receiver table allocation failed");
    CUDA_TRY(c, cudaMemcpy(g.d_rec, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    // rs2d work stealing: one 64-bit word per warp (rows < 2^20, units < 2^14;
    // FD_RS_STEAL=0: static split)
    dev_free(g.d_ws);
    g.d_ws = nullptr;
    g.nws = 0;
    static const bool steal = [] { const char *e = getenv("FD_RS_STEAL"); return !(e && e[0] == '0'); }();
    if (t && t->kind == 1 && g.lin == 0 && steal && span < (1 << 20) - 4096 && nunits < (1 << 14)) {
        g.nws = rs2d_ctas(c, *t, c->tb2occ, span) * t->ny;
        g.d_ws = (unsigned long long *)dev_alloc((size_t)g.nws * 8);
        if (!g.d_ws) return fail(FD_ERR_NOMEM, "work-stealing array allocation failed");
        CUDA_TRY(c, cudaMemset(g.d_ws, 0, (size_t)g.nws * 8));
    }
    return FD_OK;
}

// Re-split the single slab into n virtual slabs on this GPU (FD_OPT_VSLABS).
static fd_status split_virtual(fd_ctx *c, int n) {
    if (n <= 1) return FD_OK;
    if (c->nranks > 1) return fail(FD_ERR_STATE, "FD_OPT_VSLABS is for single-process contexts");
    const int64_t nz = c->z1 - c->z0;
    if (nz < (int64_t)n * 2 * c->R) return fail(FD_ERR_ARG, "too many virtual slabs for nz=%lld", (long long)nz);
    // the new slabs take their planes of K and of both fields (fd_set_wavefield
    // may have set them) from the single slab by device copies
    const int64_t pf = plane_floats(c);
    Slab o = c->slabs[0];
    std::vector<Slab> ns((size_t)n);
    c->dev_bytes = 0;
    fd_status st = FD_OK;
    for (int q = 0; q < n && st == FD_OK; ++q) {
        Slab &s = ns[q];
        int64_t a, b;
        partition(nz, n, q, &a, &b);
        s.z0 = c->z0 + a; s.z1 = c->z0 + b; s.nz = b - a;
        st = build_slab(c, s, o.Kh + a * pf);     // K planes a - r .. b + r
        if (st) break;
        const size_t bytes = (size_t)(s.nz * pf) * 4;
        for (int f = 0; f < 2; ++f)
            CUDA_TRY(c, cudaMemcpy(s.F[f] + c->H * pf, o.F[f] + (c->H + a) * pf, bytes, cudaMemcpyDeviceToDevice));
    }
    free_slab(o);
    c->slabs.swap(ns);
    return st;
}

struct XBuf { int b, depth; };
static fd_status exchange(fd_ctx *c, std::initializer_list<XBuf> xs, cudaStream_t st);

// ------------------------------------------------------------ cluster-resident runs
// Auto threshold: grids up to this many points run whole fd_step calls in one
// cluster launch (launch-bound sizes).
constexpr int64_t kResidentAutoPoints = (int64_t)1 << 17;

static const void *resident_fn(int R, int ndim) {
    switch (R * 10 + ndim) {
    case 12: return (const void *)resident_kernel<1, 2>;
    case 13: return (const void *)resident_kernel<1, 3>;
    case 22: return (const void *)resident_kernel<2, 2>;
    case 23: return (const void *)resident_kernel<2, 3>;
    case 32: return (const void *)resident_kernel<3, 2>;
    case 33: return (const void *)resident_kernel<3, 3>;
    case 42: return (const void *)resident_kernel<4, 2>;
    default: return (const void *)resident_kernel<4, 3>;
    }
}

// Largest cluster (16, 8, 4, 2 CTAs, or the forced size) whose CTAs hold
// their planes of p, p_prev (each with r halo planes per side) and K in
// shared memory, own >= r planes each and can be co-scheduled.
static bool resident_config(fd_ctx *c) {
    if (c->nranks != 1 || c->slabs.size() != 1) return false;
    const int64_t nz = c->nzg, PS = c->nyg * c->nxg;
    int maxsm = 0;
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    const void *fn = resident_fn(c->R, c->ndim);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int cands[4] = {16, 8, 4, 2};
    for (int nc : cands) {
        if (c->opt_cluster > 0 && nc != c->opt_cluster) continue;
        if (nz / nc < c->R || nz / nc < 1) continue;
        const int64_t npmax = (nz + nc - 1) / nc;
        const int64_t smem = (2 * (npmax + 2 * c->R) + npmax) * PS * 4;
        if (smem > maxsm) continue;
        const int64_t work = (nz / nc) * PS;
        const int threads = (int)std::min<int64_t>(1024, std::max<int64_t>(32, (work + 31) / 32 * 32));
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = nc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(nc); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = (size_t)smem;
        cfg.attrs = at; cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            continue;
        }
        c->res_nc = nc; c->res_npmax = (int)npmax; c->res_threads = threads; c->res_smem = (int)smem;
        return true;
    }
    return false;
}

// Receivers sorted by owning CTA (plane split of resident_kernel) + offsets.
static fd_status upload_resident_receivers(fd_ctx *c) {
    const int nc = c->res_nc, n = (int)c->rec.size();
    const int64_t nz = c->nzg;
    std::vector<std::pair<int, int>> ord;          // (cta, receiver)
    for (int j = 0; j < n; ++j) {
        int cta = 0;
        while (cta + 1 < nc && nz * (cta + 1) / nc <= c->rec[j].g[0]) ++cta;
        ord.push_back({cta, j});
    }
    std::stable_sort(ord.begin(), ord.end());
    std::vector<int32_t> h((size_t)4 * n + nc + 1, 0);
    for (int i = 0; i < n; ++i) {
        const RecDef &r = c->rec[ord[i].second];
        h[i] = (int32_t)r.g[0]; h[n + i] = (int32_t)r.g[1]; h[2 * n + i] = (int32_t)r.g[2];
        h[3 * n + i] = ord[i].second;
    }
    for (int q = 0, i = 0; q <= nc; ++q) {
        while (i < n && ord[i].first < q) ++i;
        h[4 * n + q] = i;
    }
    c->d_res_rec = (int32_t *)dev_alloc(h.size() * 4);
    if (!c->d_res_rec) return fail(FD_ERR_NOMEM, "receiver table allocation failed");
    CUDA_TRY(c, cudaMemcpy(c->d_res_rec, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    return FD_OK;
}

// The launches of one slab: [0, nz) -- or, with the overlapped schedule, the
// boundary planes that feed the exchange ([0, bw) and [nz - bw, nz) where a
// neighbour exists) first, then the interior.  bw = r for single steps, 2r
// with temporal blocking (the neighbour reads 2r planes of P^{k+2}).
static void split_regions(const fd_ctx *c, const Slab &s, bool overlap, int32_t bw, const TileCfg *t, int occ,
                          std::vector<Region> &out) {
    out.clear();
    const int32_t nz = (int32_t)s.nz;
    auto add = [&](int32_t lo, int32_t hi, bool boundary) {
        if (hi <= lo) return;
        Region g;
        g.zlo = lo; g.zhi = hi; g.boundary = boundary;
        g.zchunks = t ? chunks_for(c, *t, occ, hi - lo) : 1;
        g.lin = t ? lin_units(c, *t, occ, hi - lo) : 0;
        out.push_back(g);
    };
    if (!overlap) { add(0, nz, false); return; }
    const int32_t lo_end = s.has_lo ? std::min(bw, nz) : 0;
    const int32_t hi_beg = s.has_hi ? std::max(nz - bw, lo_end) : nz;
    if (s.has_lo) add(0, lo_end, true);
    if (s.has_hi) add(hi_beg, nz, true);
    add(lo_end, hi_beg, false);
}

// FD_OPT_KPLANE: per slab, the table of K per plane
// over the K halo buffer's planes (local -r .. nz + r - 1; zero beyond) and
// a check that every plane is constant.  The tiled kernels' KZ variants run
// only when all planes of all slabs are; otherwise the K field is used.
static fd_status build_kplane(fd_ctx *c) {
    int *d_bad = (int *)dev_alloc(sizeof(int));
    if (!d_bad) return fail(FD_ERR_NOMEM, "K-plane flag allocation failed");
    CUDA_TRY(c, cudaDeviceSynchronize());
    CUDA_TRY(c, cudaMemset(d_bad, 0, sizeof(int)));
    for (auto &s : c->slabs) {
        const size_t tb = (size_t)(s.nz + 2 * kKzPad) * 4;
        s.kzt = (float *)dev_alloc(tb);
        if (!s.kzt) { dev_free(d_bad); return fail(FD_ERR_NOMEM, "K-plane table allocation failed"); }
        c->dev_bytes += (double)tb;
        CUDA_TRY(c, cudaMemset(s.kzt, 0, tb));
        const int64_t planes = s.nz + 2 * c->R;
        const int blocks = (int)std::min<int64_t>((planes * c->nyg * c->nxg + 255) / 256, (int64_t)c->nsm * 16);
        kplane_table_kernel<<<blocks, 256>>>(s.Kh, planes, c->nyg, c->nxg, c->pitch, s.kzt + kKzPad - c->R, d_bad);
        CUDA_TRY(c, cudaGetLastError());
    }
    int bad = 0;
    CUDA_TRY(c, cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost));
    dev_free(d_bad);
    c->kplane = (bad == 0);
    return FD_OK;
}

static fd_status prepare(fd_ctx *c) {
    fd_status st = split_virtual(c, c->opt_vslabs);
    if (st) return st;
    {
        // test hook (FD_VSLAB_NCCL=1): virtual slabs exchange their halos with
        // NCCL send/recv over a one-rank communicator (self peer) instead of
        // device copies -- the NCCL calls, grouping and graph capture of the
        // multi-rank exchange run on a single GPU (NCCL refuses two ranks on
        // one device)
        const char *e = getenv("FD_VSLAB_NCCL");
        if (e && e[0] == '1' && c->slabs.size() > 1 && c->nranks == 1 && c->opt_transport == 0) {
            if (!nccl().ok) return fail(FD_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
            ncclUniqueId id;
            ncclResult_t r = nccl().GetUniqueId(&id);
            if (!r) r = nccl().CommInitRank(&c->comm, 1, id, 0);
            if (r) {
                c->poisoned = true;
                return fail(FD_ERR_NCCL, "ncclCommInitRank (self): %s", nccl().GetErrorString(r));
            }
            c->nccl_self = true;
        }
    }
    if (!c->stream) {
        // no stream set: an own non-blocking stream (capturable for graphs)
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
    }
    c->d_k = (int64_t *)dev_alloc(sizeof(int64_t));
    if (!c->d_k) return fail(FD_ERR_NOMEM, "step counter allocation failed");
    if (c->sponge_nb > 0) {
        // Cerjan profile per axis (R#18), fp64 rounded once: g = exp(-(alpha (nb - d))^2)
        // for d = min(j, n-1-j) < nb, else 1; z over the GLOBAL planes
        std::vector<float> h;
        auto axis = [&](int64_t n) {
            for (int64_t j = 0; j < n; ++j) {
                const int64_t d = std::min(j, n - 1 - j);
                const double a = c->sponge_alpha * (double)(c->sponge_nb - d);
                h.push_back(d < c->sponge_nb ? (float)std::exp(-(a * a)) : 1.0f);
            }
        };
        axis(c->nxg);
        if (c->ndim == 3) axis(c->nyg); else h.push_back(1.0f);
        axis(c->nzg);
        c->d_gsp = (float *)dev_alloc(h.size() * 4);
        if (!c->d_gsp) return fail(FD_ERR_NOMEM, "sponge table allocation failed");
        CUDA_TRY(c, cudaMemcpy(c->d_gsp, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    }
    if (c->opt_resident != 1 && c->opt_kernel == 0) {
        // auto: small single-slab grids with no pinned tile / step mode
        const bool want = c->opt_resident == 2 ||
                          (c->nxg * c->nyg * c->nzg <= kResidentAutoPoints && c->opt_tile < 0 &&
                           c->opt_tsteps == 0 && c->opt_vslabs == 1 && c->nranks == 1 &&
                           c->opt_transport == 0);
        if (want) {
            c->resident = resident_config(c);
            if (!c->resident && c->opt_resident == 2)
                return fail(FD_ERR_STATE, "FD_OPT_RESIDENT=2: the grid does not fit one cluster's shared memory "
                                          "(single-slab contexts, >= r planes per CTA)");
            if (c->resident) {
                c->opt_tsteps = 1;
                return upload_resident_receivers(c);
            }
        }
    } else if (c->opt_resident == 2) {
        return fail(FD_ERR_STATE, "FD_OPT_RESIDENT=2 needs the fused path (FD_OPT_KERNEL 0 or 2)");
    }
    int64_t maxnz = 0;
    for (auto &s : c->slabs) maxnz = std::max(maxnz, s.nz);
    if (c->opt_kernel == 0) {
        choose_tile(c, maxnz);
        if (c->tile < 0) return fail(FD_ERR_CUDA, "no fused kernel configuration fits this device");
        const TileCfg &t = tile_table()[c->tile];
        for (int v = 0; v < kVariants; ++v)
            if (t.kernel[v])
                CUDA_TRY(c, cudaFuncSetAttribute(t.kernel[v], cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem));
    }
    if (c->opt_tsteps == 0) {
        // auto: temporal blocking where it is faster (r04 sweeps: 3D order 2
        // 582 vs 426 Gpts/s on C3 -- order 4 375 vs 421 stays single; 2D order 2
        // 554 vs 400 and order 4 486 vs 397 on C2 -- orders 6/8 stay single)
        // unless a single-step tile is pinned
        const bool tb_wins = c->ndim == 3 ? c->R == 1 : c->R <= 2;
        c->opt_tsteps = (tb_wins && c->opt_kernel == 0 && c->opt_tile < 0) ? 2 : 1;
        // 2D orders 2 / 4 / 6 on one slab with the band rule: four / three /
        // three steps per pass in the register-streamed kernel (r3, C2: 723 /
        // 622 / 441 Gpts/s vs 562 / 500 two-step tb2d and 390 single-step;
        // DESIGN.md section 5.12); order 8 stays on single steps (319 vs 385)
        if (c->ndim == 2 && c->R <= 3 && c->opt_kernel == 0 && c->opt_tile < 0 && c->nranks == 1 &&
            c->slabs.size() == 1 && c->sponge_nb == 0 && c->opt_transport == 0 && c->opt_tb2tile < 0)
            c->opt_tsteps = c->R == 1 ? 4 : 3;
    }
    const bool multi = c->nranks > 1 || c->slabs.size() > 1;
    // overlapped schedule (boundary planes + exchange on the comm stream,
    // interior on the user stream): NCCL ranks, and virtual slabs, which run
    // the identical schedule with device-copy halos.  Single steps exchange r
    // planes of P per face; temporal blocking 2r of P^{k+2} and r of P^{k+1}
    // per two steps.
    const bool overlap = multi && c->opt_kernel == 0;
    c->overlap = overlap;
    if (c->opt_transport == 1 && (!multi || c->opt_kernel != 0))
        return fail(FD_ERR_STATE, "FD_OPT_TRANSPORT=1 needs z-slabs (ranks or FD_OPT_VSLABS) and the fused kernels");
    for (size_t q = 0; q < c->slabs.size(); ++q) {
        Slab &s = c->slabs[q];
        s.has_lo = c->nranks > 1 ? c->rank > 0 : q > 0;
        s.has_hi = c->nranks > 1 ? c->rank < c->nranks - 1 : q + 1 < c->slabs.size();
        if (c->opt_kernel == 0) {
            st = make_maps(c, s);
            if (st) return st;
        }
        if (c->opt_kernel == 3) {
            // derivative fields of the unfused decomposition (pitched like K)
            const size_t db = (size_t)(s.nz * plane_floats(c)) * 4;
            for (int a = 0; a < 3; ++a) {
                if (a == 1 && c->ndim == 2) continue;
                s.D[a] = (float *)dev_alloc(db);
                if (!s.D[a]) return fail(FD_ERR_NOMEM, "derivative field allocation failed");
                // the pitch padding is never written but read by fd_time's edge quads
                CUDA_TRY(c, cudaMemset(s.D[a], 0, db));
                c->dev_bytes += (double)db;
            }
        }
        // single steps between temporal-blocking launches refresh 2r halo planes
        const int32_t bw = c->opt_tsteps >= 2 ? c->H : c->R;
        split_regions(c, s, overlap, bw, c->opt_kernel != 0 ? nullptr : &tile_table()[c->tile], c->occ, s.regions);
        for (auto &g : s.regions) {
            st = upload_region_receivers(c, s, g, c->opt_kernel != 0 ? nullptr : &tile_table()[c->tile]);
            if (st) return st;
        }
    }
    if (c->opt_tsteps >= 2) {
        // temporal blocking: 2 steps per launch (3D orders 2-8, 2D; slabs, ranks,
        // sponge, peer pushes), S >= 3 (2D single-slab band-rule contexts)
        if (c->opt_kernel != 0) return fail(FD_ERR_STATE, "FD_OPT_TSTEPS >= 2 needs the fused kernel");
        if (c->opt_tsteps >= 3 && (c->ndim != 2 || multi || c->sponge_nb > 0 || c->opt_transport == 1))
            return fail(FD_ERR_STATE, "FD_OPT_TSTEPS=%d: 2D single-slab contexts without the sponge frame",
                        c->opt_tsteps);
        const auto &tb = tb2_table();
        for (int i = 0; i < (int)tb.size() && c->tb2 < 0; ++i) {
            if (tb[i].r != c->R || tb[i].ndim != c->ndim || tb[i].steps != c->opt_tsteps ||
                (c->opt_tb2tile >= 0 && i != c->opt_tb2tile))
                continue;
            if (needs_full(c) && !tb[i].full()) continue;
            const int occ = occupancy(c, tb[i]);
            if (occ > 0) { c->tb2 = i; c->tb2occ = occ; }
        }
        if (c->tb2 < 0)
            return fail(c->opt_tsteps >= 3 ? FD_ERR_STATE : FD_ERR_CUDA,
                        "no %d-steps-per-launch configuration for this order / device", c->opt_tsteps);
        const TileCfg &t = tb[c->tb2];
        for (int v = 0; v < kVariants; ++v)
            if (t.kernel[v])
                CUDA_TRY(c, cudaFuncSetAttribute(t.kernel[v], cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem));
        const TileCfg &ts = tile_table()[c->tile];
        for (auto &s : c->slabs) {
            const size_t fbytes = (size_t)buf_floats(c, s) * 4;
            for (int b = 2; b < 4; ++b) {
                if (s.F[b]) continue;                  // fd_peer_export allocated it
                s.F[b] = (float *)dev_alloc(fbytes);
                if (!s.F[b]) return fail(FD_ERR_NOMEM, "temporal-blocking buffer allocation failed");
                CUDA_TRY(c, cudaMemset(s.F[b], 0, fbytes));
                c->dev_bytes += (double)fbytes;
            }
            const int64_t planes = s.nz + 2 * c->H;
            // 3D boxes (x, y rows, 1 plane); 2D boxes (x, 1, z rows).  K through
            // its halo buffer: stage A reads K on the r planes beyond the slab.
            const bool d3 = c->ndim == 3;
            const int py = d3 ? t.pbz : 1, pz = d3 ? 1 : t.pbz, ey = d3 ? t.tbz : 1, ez = d3 ? 1 : t.tbz;
            const int sy = d3 ? ts.ty + 2 * c->R : 1, sz = d3 ? 1 : ts.pbz, ty1 = d3 ? ts.ty : 1, tz1 = d3 ? 1 : ts.tbz;
            bool ok = make_map(&s.mKe, s.Kh, c->nxg, c->nyg, s.nz + 2 * c->R, c->pitch, t.tbw, ey, ez);
            for (int b = 0; b < 4 && ok; ++b)
                ok = make_map(&s.mP0[b], s.F[b], c->nxg, c->nyg, planes, c->pitch, t.pbw, py, pz) &&
                     make_map(&s.mPm[b], s.F[b], c->nxg, c->nyg, planes, c->pitch, t.tbw, ey, ez) &&
                     make_map(&s.mHalo[b], s.F[b], c->nxg, c->nyg, planes, c->pitch, ts.pbw, sy, sz) &&
                     make_map(&s.mTile[b], s.F[b], c->nxg, c->nyg, planes, c->pitch, ts.tbw, ty1, tz1);
            if (!ok) {
                c->poisoned = true;
                return fail(FD_ERR_CUDA, "cuTensorMapEncodeTiled failed (temporal blocking)");
            }
            split_regions(c, s, overlap, c->H, &t, c->tb2occ, s.tb2);
            for (auto &g : s.tb2) {
                st = upload_region_receivers(c, s, g, &t);
                if (st) return st;
            }
        }
    }
    if (overlap) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        CUDA_TRY(c, cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_step, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
    }
    if (c->nranks > 1 && c->opt_transport == 1) {
        // peer transport: fd_peer_export / fd_peer_import set up the mappings
        // (the K halos go with the first exchange)
        if (!c->peer_imported)
            return fail(FD_ERR_STATE, "FD_OPT_TRANSPORT=1: call fd_peer_export / fd_peer_import before fd_step");
    } else if (c->nranks > 1) {
        if (!nccl().ok) return fail(FD_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
        if (!c->have_id) return fail(FD_ERR_ARG, "nccl_id is NULL with nranks > 1 (NCCL transport)");
        ncclResult_t r = nccl().CommInitRank(&c->comm, c->nranks, c->nccl_id, c->rank);
        if (r != 0) {
            c->poisoned = true;
            return fail(FD_ERR_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
        }
        // K halos (static; read by the temporal-blocking kernel) once
        st = exchange(c, {{-1, c->R}}, c->stream);
        if (st) return st;
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    // per-plane K once K and its halos are final (peer-transport ranks receive
    // K's halos with the first exchange: they keep the K field)
    const bool kz_compiled = c->tile >= 0 && tile_table()[c->tile].full() &&
                             (c->opt_tsteps < 2 || (c->tb2 >= 0 && tb2_table()[c->tb2].kernel[kVarKPlane]));
    if (c->opt_kplane && c->opt_kernel == 0 && !c->resident && !(c->nranks > 1 && c->opt_transport == 1) &&
        kz_compiled) {
        st = build_kplane(c);
        if (st) return st;
    }
    return FD_OK;
}

// Grow the step-indexed device tables to cover steps [0, steps_needed):
// traces (rows 0..steps_needed-1) and the wavelet table (w_0..w_steps_needed,
// the last step injects w_{k+1}).  Doubling growth; moves invalidate graphs.
static fd_status ensure_tables(fd_ctx *c, int64_t steps_needed) {
    const int64_t nrec = (int64_t)c->rec.size(), nsrc = (int64_t)c->src.size();
    if (nrec > 0 && steps_needed > c->trace_cap) {
        int64_t cap = std::max<int64_t>({steps_needed, 2 * c->trace_cap, 16});
        float *nb = (float *)dev_alloc((size_t)(cap * nrec) * 4);
        if (!nb) return fail(FD_ERR_NOMEM, "trace buffer allocation failed");
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        CUDA_TRY(c, cudaMemset(nb, 0, (size_t)(cap * nrec) * 4));
        if (c->d_traces) {
            CUDA_TRY(c, cudaMemcpy(nb, c->d_traces, (size_t)(c->trace_cap * nrec) * 4, cudaMemcpyDeviceToDevice));
            dev_free(c->d_traces);
        }
        c->d_traces = nb;
        c->trace_cap = cap;
    }
    if (steps_needed + 1 > c->wcap) {
        int64_t cap = std::max<int64_t>({steps_needed + 1, 2 * c->wcap, 16});
        std::vector<float> h((size_t)(cap * std::max<int64_t>(nsrc, 1)), 0.f);
        for (int64_t j = 0; j < cap; ++j)
            for (int64_t q = 0; q < nsrc; ++q)
                h[j * nsrc + q] = (float)(c->src[q].amp * ricker((double)j * c->dt, c->src[q].f, c->src[q].t0));
        float *nb = (float *)dev_alloc(h.size() * 4);
        if (!nb) return fail(FD_ERR_NOMEM, "wavelet table allocation failed");
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        CUDA_TRY(c, cudaMemcpy(nb, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
        dev_free(c->d_wtab);
        c->d_wtab = nb;
        c->wcap = cap;
    }
    return FD_OK;
}

// Kernel parameters of one launch (region g of slab s) for step k.
static void fill_params(const fd_ctx *c, const Slab &s, const Region *g, StepParams &p, int64_t step_k) {
    memset(&p, 0, sizeof p);
    p.nx = c->nxg; p.ny = c->nyg; p.nz = s.nz;
    p.pitch = c->pitch; p.gz0 = s.z0; p.nzg = c->nzg;
    p.zlo = g ? g->zlo : 0;
    p.zhi = g ? g->zhi : (int32_t)s.nz;
    p.nchunks = g ? g->zchunks : 1;
    p.lin = g ? g->lin : 0;
    p.nsrc = (int32_t)c->src.size();
    for (int q = 0; q < p.nsrc; ++q) {
        p.sz[q] = (int32_t)(c->src[q].g[0] - s.z0);
        p.sy[q] = (int32_t)c->src[q].g[1];
        p.sx[q] = (int32_t)c->src[q].g[2];
    }
    p.wtab = c->d_wtab;
    p.src_raw = s.d_src_raw;
    if (g && g->d_rec) {
        const int n = g->nrec;
        p.rec.z = g->d_rec;
        p.rec.y = g->d_rec + n;
        p.rec.x = g->d_rec + 2 * n;
        p.rec.id = g->d_rec + 3 * n;
        p.rec.off = (c->opt_kernel != 0) ? nullptr : g->d_rec + 4 * n;
        p.nrec_local = n;
    }
    p.traces = c->d_traces;
    p.nrec_total = (int32_t)c->rec.size();
    p.gsp = c->d_gsp;
    p.kz = c->kplane ? s.kzt + kKzPad : nullptr;
    // step index: baked (plain launches) or *d_k + offset (graph capture)
    p.k = step_k;
    if (c->capturing) { p.kdev = c->d_k; p.koff = (int32_t)(step_k - c->gk0); }
}

static cudaEvent_t pool_event(fd_ctx *c) {
    if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Run `launch` on stream st; with FD_OPT_PROFILE, bracket it with events.
template <class F>
static void tracked(fd_ctx *c, int kid, cudaStream_t st, F &&launch, bool is_kernel = true) {
    if (is_kernel) ++c->launches;
    if (!c->opt_profile) { launch(); return; }
    cudaEvent_t a = pool_event(c), b = pool_event(c);
    cudaEventRecord(a, st);
    launch();
    cudaEventRecord(b, st);
    c->ev_pending.push_back({kid, a, b});
}

static fd_status fold_times(fd_ctx *c) {
    for (auto &r : c->ev_pending) {
        CUDA_TRY(c, cudaEventSynchronize(r.b));
        float ms = 0;
        CUDA_TRY(c, cudaEventElapsedTime(&ms, r.a, r.b));
        c->kms[r.kid] += ms;
        c->kcnt[r.kid] += 1;
        c->ev_pool.push_back(r.a);
        c->ev_pool.push_back(r.b);
    }
    c->ev_pending.clear();
    return FD_OK;
}

template <int R> static void launch_inject(cudaStream_t st, float *field, const StepParams &p) {
    inject_kernel<R><<<1, 32, 0, st>>>(field, p);
}
template <int R, int NDIM> static void launch_naive(const fd_ctx *c, const Slab &s, cudaStream_t st,
                                                    const StepParams &p) {
    const int64_t total = c->nxg * c->nyg * s.nz;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    naive_step_kernel<R, NDIM><<<blocks, 256, 0, st>>>(p);
}
template <int R> static void launch_gather(cudaStream_t st, int n, const StepParams &p) {
    gather_receivers_kernel<R><<<(n + 127) / 128, 128, 0, st>>>(p);
}

static void dispatch_inject(fd_ctx *c, cudaStream_t st, float *field, const StepParams &p) {
    tracked(c, FD_K_INJECT, st, [&] {
        switch (c->R) {
        case 1: launch_inject<1>(st, field, p); break;
        case 2: launch_inject<2>(st, field, p); break;
        case 3: launch_inject<3>(st, field, p); break;
        default: launch_inject<4>(st, field, p); break;
        }
    });
}

template <int R, int NDIM>
static void launch_unfused(const fd_ctx *c, fd_ctx *cm, const Slab &s, cudaStream_t st, const StepParams &p) {
    // 32 x 8 threads, one quad of x points each; plane-major blocks (fd_kernels.cuh)
    const unsigned gx = (unsigned)((c->nxg + 127) / 128);
    const dim3 grid = NDIM == 3 ? dim3(gx, (unsigned)((c->nyg + 7) / 8), (unsigned)s.nz)
                                : dim3(gx, (unsigned)((s.nz + 7) / 8), 1u);
    const dim3 blk(32, 8);
    // fd_pzz / fd_pyy stream ZB points along their axis per thread
    constexpr int ZB = NDIM == 3 ? 32 : 16;      // 2D: more blocks for the short kernels
    const unsigned nzb = (unsigned)((s.nz + ZB - 1) / ZB);
    const dim3 gz = NDIM == 3 ? dim3(gx, (unsigned)((c->nyg + 7) / 8), nzb)
                              : dim3((unsigned)((c->nxg + 1023) / 1024), nzb, 1u);
    const dim3 gy(gx, (unsigned)((c->nyg + ZB - 1) / ZB), (unsigned)((s.nz + 7) / 8));
    // Listing 3 order: fd_pzz, [fd_pyy], fd_pxx, fd_time
    tracked(cm, FD_K_PZZ, st, [&] { d2_stream_kernel<R, 2, NDIM, ZB><<<gz, blk, 0, st>>>(p, s.D[2]); });
    if (NDIM == 3)
        tracked(cm, FD_K_PYY, st, [&] { d2_stream_kernel<R, 1, NDIM, ZB><<<gy, blk, 0, st>>>(p, s.D[1]); });
    tracked(cm, FD_K_PXX, st, [&] { d2_axis_kernel<R, 0, NDIM><<<grid, blk, 0, st>>>(p, s.D[0]); });
    tracked(cm, FD_K_TIME, st,
            [&] { time_update_kernel<R, NDIM><<<grid, blk, 0, st>>>(p, s.D[0], s.D[1], s.D[2]); });
}

// Programmatic dependent launch of the tiled step kernels (fd_kernels.cuh
// pdl_sync): opt-in (FD_PDL=1), single-slab contexts (the two-stream slab
// schedule orders its launches through events), not while profiling.  r2 A/B
// (Gpts/s, PDL vs plain graph replay): C2 order 4 507.6 vs 500.8, order 2
// 548.9 vs 560.9, C3 620.2 vs 618.8, orders 8 +-0.4 %: no consistent gain
// over graph replay, whose launch gaps are already ~1 us.
static bool use_pdl(const fd_ctx *c) {
    static const bool on = [] { const char *e = getenv("FD_PDL"); return e && e[0] == '1'; }();
    return on && !c->overlap && !c->opt_profile;
}

// In-kernel halo pushes of a boundary launch (FD_OPT_TRANSPORT = 1): buffer b1
// (pnext) pushes `push1` planes per face, b2 (pnext2, two-step kernels) `push2`.
static void set_push(const fd_ctx *c, const Slab &s, StepParams &p, int b1, int push1, int b2, int push2) {
    const size_t q = (size_t)(&s - c->slabs.data());
    auto one = [&](PeerPush &pp, int b, int push) {
        pp = PeerPush{nullptr, nullptr, 0, push};
        if (b < 0) return;
        if (c->nranks > 1) {
            pp.lo = s.has_lo ? c->plo.F[b] : nullptr;
            pp.hi = s.has_hi ? c->phi.F[b] : nullptr;
            pp.lo_z = (int32_t)(c->plo.nz + c->H);
        } else {
            pp.lo = q > 0 ? c->slabs[q - 1].F[b] : nullptr;
            pp.hi = q + 1 < c->slabs.size() ? c->slabs[q + 1].F[b] : nullptr;
            pp.lo_z = q > 0 ? (int32_t)(c->slabs[q - 1].nz + c->H) : 0;
        }
    };
    one(p.peer1, b1, push1);
    one(p.peer2, b2, push2);
}

static void launch_region(fd_ctx *c, Slab &s, Region &g, cudaStream_t st) {
    StepParams p;
    fill_params(c, s, &g, p, c->k);
    float *cur = cur_buf(c, s), *prev = prev_buf(c, s);
    p.pnext = prev;
    p.p = cur;
    p.K = s.K;
    if (c->opt_kernel == 1 || c->opt_kernel == 3) {
        // reference paths: naive fused stencil (1) or the paper's unfused
        // decomposition (3); then receivers and injection as separate launches
        if (c->opt_kernel == 1) {
            tracked(c, FD_K_NAIVE, st, [&] {
                switch (c->R * 10 + c->ndim) {
                case 12: launch_naive<1, 2>(c, s, st, p); break;
                case 13: launch_naive<1, 3>(c, s, st, p); break;
                case 22: launch_naive<2, 2>(c, s, st, p); break;
                case 23: launch_naive<2, 3>(c, s, st, p); break;
                case 32: launch_naive<3, 2>(c, s, st, p); break;
                case 33: launch_naive<3, 3>(c, s, st, p); break;
                case 42: launch_naive<4, 2>(c, s, st, p); break;
                default: launch_naive<4, 3>(c, s, st, p); break;
                }
            });
        } else {
            switch (c->R * 10 + c->ndim) {
            case 12: launch_unfused<1, 2>(c, c, s, st, p); break;
            case 13: launch_unfused<1, 3>(c, c, s, st, p); break;
            case 22: launch_unfused<2, 2>(c, c, s, st, p); break;
            case 23: launch_unfused<2, 3>(c, c, s, st, p); break;
            case 32: launch_unfused<3, 2>(c, c, s, st, p); break;
            case 33: launch_unfused<3, 3>(c, c, s, st, p); break;
            case 42: launch_unfused<4, 2>(c, c, s, st, p); break;
            default: launch_unfused<4, 3>(c, c, s, st, p); break;
            }
        }
        if (g.nrec > 0) {
            tracked(c, FD_K_GATHER, st, [&] {
                switch (c->R) {
                case 1: launch_gather<1>(st, g.nrec, p); break;
                case 2: launch_gather<2>(st, g.nrec, p); break;
                case 3: launch_gather<3>(st, g.nrec, p); break;
                default: launch_gather<4>(st, g.nrec, p); break;
                }
            });
        }
        if (p.nsrc > 0) dispatch_inject(c, st, prev, p);
        return;
    }
    const TileCfg &t = tile_table()[c->tile];
    p.ntx = (int32_t)((c->nxg + t.tx - 1) / t.tx);
    p.nty = (int32_t)((c->nyg + t.ty - 1) / t.ty);
    const dim3 grid((unsigned)(p.ntx * p.nty * p.nchunks));
    g.ctas = (int)grid.x;
    const CUtensorMap &mp = s.mHalo[c->icur];
    const CUtensorMap &mpp = s.mTile[c->iprev];
    const bool push = c->opt_transport == 1 && g.boundary;
    if (push) set_push(c, s, p, c->iprev, c->opt_tsteps >= 2 ? c->H : c->R, -1, 0);
    const launch_fused_t go = t.launch[(c->d_gsp ? kVarSponge : 0) | (push ? kVarPeer : 0) | (c->kplane ? kVarKPlane : 0)];
    tracked(c, FD_K_FUSED, st, [&] { go(grid, t.smem, st, mp, mpp, s.mK, p, use_pdl(c)); });
}

// Halo exchange of `depth` planes per face of field buffer b (b = -1: K).
// Owned planes [0, nz) of a field buffer live at buffer planes [H, H + nz)
// (H = halo_planes(r) = 2r; K: r); the lower halo receives the neighbour's
// top `depth` owned planes at [H - depth, H), the upper halo its bottom ones at
// [H + nz, H + nz + depth).  Virtual slabs: device copies on stream st.
// Ranks: NCCL send/recv in one group (same issue order on both sides of a
// face, so the messages of several buffers pair up).
static fd_status exchange(fd_ctx *c, std::initializer_list<XBuf> xs, cudaStream_t st) {
    const int64_t pf = plane_floats(c);
    auto base = [&](Slab &s, int b) { return b < 0 ? s.Kh : s.F[b]; };
    auto hoff = [&](int b) -> int64_t { return b < 0 ? c->R : c->H; };
    if (c->nranks > 1) {
        Slab &s = c->slabs[0];
        NcclApi &n = nccl();
        ncclResult_t r = n.GroupStart();
        for (const XBuf &x : xs) {
            float *buf = base(s, x.b);
            const int64_t H = hoff(x.b), d = x.depth;
            const size_t cnt = (size_t)(d * pf);
            if (c->rank > 0) {
                if (!r) r = n.Send(buf + H * pf, cnt, kNcclFloat32, c->rank - 1, c->comm, st);
                if (!r) r = n.Recv(buf + (H - d) * pf, cnt, kNcclFloat32, c->rank - 1, c->comm, st);
            }
            if (c->rank < c->nranks - 1) {
                if (!r) r = n.Send(buf + (H + s.nz - d) * pf, cnt, kNcclFloat32, c->rank + 1, c->comm, st);
                if (!r) r = n.Recv(buf + (H + s.nz) * pf, cnt, kNcclFloat32, c->rank + 1, c->comm, st);
            }
        }
        ncclResult_t r2 = n.GroupEnd();
        if (r || r2) {
            c->poisoned = true;
            return fail(FD_ERR_NCCL, "NCCL halo exchange: %s", n.GetErrorString(r ? r : r2));
        }
        return FD_OK;
    }
    if (c->nccl_self) {
        // virtual slabs over NCCL (test hook): each halo is a send/recv pair to
        // the own rank, issued in the same order so the pairs match
        NcclApi &n = nccl();
        ncclResult_t r = n.GroupStart();
        for (size_t q = 0; q < c->slabs.size(); ++q) {
            Slab &s = c->slabs[q];
            for (const XBuf &x : xs) {
                float *buf = base(s, x.b);
                const int64_t H = hoff(x.b), d = x.depth;
                const size_t cnt = (size_t)(d * pf);
                if (q > 0) {
                    Slab &l = c->slabs[q - 1];
                    if (!r) r = n.Send(base(l, x.b) + (H + l.nz - d) * pf, cnt, kNcclFloat32, 0, c->comm, st);
                    if (!r) r = n.Recv(buf + (H - d) * pf, cnt, kNcclFloat32, 0, c->comm, st);
                }
                if (q + 1 < c->slabs.size()) {
                    Slab &u = c->slabs[q + 1];
                    if (!r) r = n.Send(base(u, x.b) + H * pf, cnt, kNcclFloat32, 0, c->comm, st);
                    if (!r) r = n.Recv(buf + (H + s.nz) * pf, cnt, kNcclFloat32, 0, c->comm, st);
                }
            }
        }
        ncclResult_t r2 = n.GroupEnd();
        if (r || r2) {
            c->poisoned = true;
            return fail(FD_ERR_NCCL, "NCCL halo exchange (virtual slabs): %s", n.GetErrorString(r ? r : r2));
        }
        return FD_OK;
    }
    for (size_t q = 0; q < c->slabs.size(); ++q) {
        Slab &s = c->slabs[q];
        for (const XBuf &x : xs) {
            float *buf = base(s, x.b);
            const int64_t H = hoff(x.b), d = x.depth;
            const size_t bytes = (size_t)(d * pf) * 4;
            if (q > 0) {
                Slab &l = c->slabs[q - 1];
                CUDA_TRY(c, cudaMemcpyAsync(buf + (H - d) * pf, base(l, x.b) + (H + l.nz - d) * pf, bytes,
                                            cudaMemcpyDeviceToDevice, st));
            }
            if (q + 1 < c->slabs.size()) {
                Slab &u = c->slabs[q + 1];
                CUDA_TRY(c, cudaMemcpyAsync(buf + (H + s.nz) * pf, base(u, x.b) + H * pf, bytes,
                                            cudaMemcpyDeviceToDevice, st));
            }
        }
    }
    return FD_OK;
}

// n steps in one cluster launch; the roles swap when n is odd.
static fd_status resident_steps(fd_ctx *c, int64_t n) {
    Slab &s = c->slabs[0];
    while (n > 0) {
        const int32_t m = (int32_t)std::min<int64_t>(n, (int64_t)1 << 30);
        StepParams p;
        fill_params(c, s, nullptr, p, c->k);
        p.K = s.K;
        const int nic = (m & 1) ? c->iprev : c->icur, nip = (m & 1) ? c->icur : c->iprev;
        ResidentArgs ra{cur_buf(c, s), prev_buf(c, s), s.F[nic], s.F[nip], m, c->res_npmax, c->d_res_rec,
                        (int32_t)c->rec.size()};
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c->res_nc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(c->res_nc); cfg.blockDim = dim3(c->res_threads);
        cfg.dynamicSmemBytes = (size_t)c->res_smem; cfg.stream = c->stream;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaError_t e = cudaSuccess;
        void *args[2] = {(void *)&p, (void *)&ra};
        tracked(c, FD_K_RESIDENT, c->stream,
                [&] { e = cudaLaunchKernelExC(&cfg, resident_fn(c->R, c->ndim), args); });
        CUDA_TRY(c, e);
        c->icur = nic; c->iprev = nip;
        c->k += m;
        n -= m;
    }
    return FD_OK;
}

// Ranks with FD_OPT_TRANSPORT = 1.  peer_signal: after this rank's pushes (the
// boundary launches or peer_copy) on stream st, publish the exchange count in
// the neighbours' flags.  peer_wait: before launches that read halos, wait for
// the neighbours' count of the previous exchange (which also orders our next
// pushes after their reads of the halos those pushes overwrite).
// Bound of a peer_wait spin (FD_PEER_TIMEOUT_S, default 60 s): a neighbour that
// failed or died must not hang this rank's streams forever.
static uint64_t peer_timeout_ns() {
    static const uint64_t ns = [] {
        const char *e = getenv("FD_PEER_TIMEOUT_S");
        const double s = e ? atof(e) : 60.0;
        return (uint64_t)((s > 0 ? s : 60.0) * 1e9);
    }();
    return ns;
}
static fd_status check_peer_timeout(fd_ctx *c) {
    if (c->h_perr && *(volatile int *)c->h_perr) {
        c->poisoned = true;
        return fail(FD_ERR_STATE, "peer transport: a neighbour did not signal its halo exchange within %.0f s "
                                  "(failed or exited rank); context poisoned", peer_timeout_ns() * 1e-9);
    }
    return FD_OK;
}
static void peer_signal(fd_ctx *c, cudaStream_t st) {
    ++c->xcount;
    int64_t *lo = c->rank > 0 ? c->plo.flags + 1 : nullptr;            // rank - 1 hears from its upper side
    int64_t *hi = c->rank < c->nranks - 1 ? c->phi.flags : nullptr;    // rank + 1 from its lower side
    peer_signal_kernel<<<1, 1, 0, st>>>(lo, hi, c->xcount);
    ++c->launches;
}
static void peer_wait(fd_ctx *c, cudaStream_t st) {
    peer_wait_kernel<<<1, 1, 0, st>>>(c->d_flags, c->rank > 0, c->rank < c->nranks - 1, c->xcount, c->d_perr,
                                      peer_timeout_ns());
    ++c->launches;
}
// Push `depth` boundary planes of buffer b (-1: K) into the neighbours' halos
// with copies (the first exchange: initial fields and the static K halos).
static fd_status peer_copy(fd_ctx *c, std::initializer_list<XBuf> xs, cudaStream_t st) {
    const int64_t pf = plane_floats(c);
    Slab &s = c->slabs[0];
    for (const XBuf &x : xs) {
        const int64_t H = x.b < 0 ? c->R : c->H, d = x.depth;
        const float *src = x.b < 0 ? s.Kh : s.F[x.b];
        const size_t bytes = (size_t)(d * pf) * 4;
        if (c->rank > 0) {
            float *dst = x.b < 0 ? c->plo.Kh : c->plo.F[x.b];
            CUDA_TRY(c, cudaMemcpyAsync(dst + (H + c->plo.nz) * pf, src + H * pf, bytes, cudaMemcpyDefault, st));
        }
        if (c->rank < c->nranks - 1) {
            float *dst = x.b < 0 ? c->phi.Kh : c->phi.F[x.b];
            CUDA_TRY(c, cudaMemcpyAsync(dst + (H - d) * pf, src + (H + s.nz - d) * pf, bytes, cudaMemcpyDefault, st));
        }
    }
    return FD_OK;
}

static fd_status one_step(fd_ctx *c) {
    fd_status s;
    if (c->overlap) {
        // comm stream: boundary planes -> halo exchange (NCCL or device copies);
        // user stream: interior planes.  Step k+1 starts after both (its
        // boundary kernel overwrites planes that step k's interior kernel reads
        // as p; its kernels read the halos received in step k).
        CUDA_TRY(c, cudaEventRecord(c->ev_step, c->stream));
        CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_step, 0));
        const bool peer_ranks = c->opt_transport == 1 && c->nranks > 1;
        if (peer_ranks) peer_wait(c, c->comm_stream);
        for (auto &sl : c->slabs)
            for (auto &g : sl.regions)
                if (g.boundary) launch_region(c, sl, g, c->comm_stream);
        if (peer_ranks) peer_signal(c, c->comm_stream);
        if (c->opt_transport != 1) {
            const int d = c->opt_tsteps >= 2 ? c->H : c->R;     // = the boundary regions' width
            tracked(c, FD_K_HALO, c->comm_stream, [&] { s = exchange(c, {{c->iprev, d}}, c->comm_stream); },
                    false);
            if (s) return s;
        }
        CUDA_TRY(c, cudaEventRecord(c->ev_comm, c->comm_stream));
        for (auto &sl : c->slabs)
            for (auto &g : sl.regions)
                if (!g.boundary) launch_region(c, sl, g, c->stream);
        CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
    } else {
        for (auto &sl : c->slabs)
            for (auto &g : sl.regions) launch_region(c, sl, g, c->stream);
        if (c->slabs.size() > 1 || c->nranks > 1) {
            // the new P (a single step between temporal-blocking launches
            // needs all 2r halo planes; the new P_prev keeps its valid ones)
            const int d = c->opt_tsteps >= 2 ? c->H : c->R;
            tracked(c, FD_K_HALO, c->stream, [&] { s = exchange(c, {{c->iprev, d}}, c->stream); }, false);
            if (s) return s;
        }
    }
    CUDA_TRY(c, cudaGetLastError());
    std::swap(c->icur, c->iprev);
    ++c->k;
    return FD_OK;
}

// Temporal blocking: steps k and k+1 in one pass (fd_tb2.cuh) per slab region.
// Reads the (cur, prev) buffers, writes P^{k+1} and P^{k+2} into the two free
// ones.  Slabs: 2r halo planes of P^{k+2} (the next pass's P^k, whose taps
// reach 2r beyond the slab) and r of P^{k+1} (read pointwise on the r planes
// beyond the slab) come from the neighbours -- on the overlapped schedule the
// 2r-plane boundary regions run first on the comm stream and feed the
// exchange while the interior region runs on the user stream.
static void launch_tb2(fd_ctx *c, Slab &s, Region &g, int f1, int f2, cudaStream_t st) {
    const TileCfg &t = tb2_table()[c->tb2];
    StepParams p;
    fill_params(c, s, &g, p, c->k);
    p.p = cur_buf(c, s);
    p.pm = prev_buf(c, s);
    p.pnext = s.F[f1];
    p.pnext2 = s.F[f2];
    p.K = s.K;
    p.ntx = (int32_t)((c->nxg + t.tx - 1) / t.tx);
    p.nty = (int32_t)((c->nyg + t.ty - 1) / t.ty);
    p.ws = g.d_ws;
    p.nws = g.nws;
    const dim3 grid((unsigned)(t.kind == 1 ? rs2d_ctas(c, t, c->tb2occ, g.zhi - g.zlo)
                                           : p.lin > 0 ? p.lin : p.ntx * p.nty * p.nchunks));
    g.ctas = (int)grid.x;
    const CUtensorMap &m0 = s.mP0[c->icur], &mm = s.mPm[c->iprev];
    const bool push = c->opt_transport == 1 && g.boundary;
    if (push) set_push(c, s, p, f1, c->R, f2, c->H);
    const launch_fused_t go = t.launch[(c->d_gsp ? kVarSponge : 0) | (push ? kVarPeer : 0) | (c->kplane ? kVarKPlane : 0)];
    tracked(c, FD_K_FUSED, st, [&] { go(grid, t.smem, st, m0, mm, s.mKe, p, use_pdl(c)); });
}

// S steps per launch (S = 2: tb2ws / tb2d; S >= 3: tbs2d, single slab).
static fd_status tb_steps(fd_ctx *c) {
    const int S = tb2_table()[c->tb2].steps;
    int f1 = -1, f2 = -1;
    for (int b = 0; b < 4; ++b)
        if (b != c->icur && b != c->iprev) (f1 < 0 ? f1 : f2) = b;
    fd_status s = FD_OK;
    if (c->overlap) {
        CUDA_TRY(c, cudaEventRecord(c->ev_step, c->stream));
        CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_step, 0));
        const bool peer_ranks = c->opt_transport == 1 && c->nranks > 1;
        if (peer_ranks) peer_wait(c, c->comm_stream);
        for (auto &sl : c->slabs)
            for (auto &g : sl.tb2)
                if (g.boundary) launch_tb2(c, sl, g, f1, f2, c->comm_stream);
        if (peer_ranks) peer_signal(c, c->comm_stream);
        if (c->opt_transport != 1) {
            tracked(c, FD_K_HALO, c->comm_stream,
                    [&] { s = exchange(c, {{f2, c->H}, {f1, c->R}}, c->comm_stream); }, false);
            if (s) return s;
        }
        CUDA_TRY(c, cudaEventRecord(c->ev_comm, c->comm_stream));
        for (auto &sl : c->slabs)
            for (auto &g : sl.tb2)
                if (!g.boundary) launch_tb2(c, sl, g, f1, f2, c->stream);
        CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
    } else {
        for (auto &sl : c->slabs)
            for (auto &g : sl.tb2) launch_tb2(c, sl, g, f1, f2, c->stream);
    }
    CUDA_TRY(c, cudaGetLastError());
    c->iprev = f1;
    c->icur = f2;
    c->k += S;
    return FD_OK;
}

// Advance m steps with plain launches (pairs through temporal blocking).
static fd_status advance_plain(fd_ctx *c, int64_t m) {
    const int S = (c->opt_tsteps >= 2 && c->tb2 >= 0) ? tb2_table()[c->tb2].steps : 1;
    while (m > 0) {
        fd_status s = (S >= 2 && m >= S) ? tb_steps(c) : one_step(c);
        if (s) return s;
        m -= (S >= 2 && m >= S) ? S : 1;
    }
    return FD_OK;
}

// ------------------------------------------------------------ CUDA graphs
// graph_len(c) consecutive steps captured once per starting buffer parity and
// replayed (launch-bound small grids).  Kernels read k = *d_k + offset; the
// graph ends by advancing d_k.  Not used while profiling, nor with the peer
// transport across ranks (its flag waits carry per-exchange counts).
// steps per graph: a multiple of the steps per launch (24 for three-step
// launches, else 16), so no graph holds a single-step remainder launch
static int64_t graph_len(const fd_ctx *c) {
    const int S = (c->opt_tsteps >= 2 && c->tb2 >= 0) ? tb2_table()[c->tb2].steps : 1;
    return S == 3 ? 24 : 16;
}

static bool graphs_usable(const fd_ctx *c) {
    // virtual slabs: the two-stream schedule is captured too (event fork/join).
    // NCCL ranks: the send/recv of the halo exchange are captured with the
    // kernels (NCCL supports stream capture); only after the first plain step,
    // so that NCCL's lazy connection setup has happened outside any capture.
    // Every rank replays the same sequence (the graph choice depends on the
    // buffer roles and the step count only), so the captured sends and
    // receives pair up as the plain ones do.
    const bool ranks_ok = (c->nranks == 1 && !c->comm) || (c->opt_transport == 0 && c->comm && c->injected && c->k > 0);
    return c->opt_graph && ranks_ok && !c->opt_profile && c->d_k && c->stream && !c->resident;
}

// Capture graph_len(c) steps starting from the current buffer roles; the
// entry records the roles it ends in.  Returns the entry index or -1.
static int capture_graph(fd_ctx *c, fd_status *st) {
    const int64_t k0 = c->k, l0 = c->launches;
    const int ic0 = c->icur, ip0 = c->iprev;
    *st = FD_OK;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { cudaGetLastError(); c->opt_graph = 0; return -1; }
    c->capturing = true;
    c->gk0 = k0;
    fd_status s = advance_plain(c, graph_len(c));
    advance_step_kernel<<<1, 1, 0, c->stream>>>(c->d_k, graph_len(c));
    c->capturing = false;
    e = cudaStreamEndCapture(c->stream, &graph);
    fd_ctx::Graph gr{ic0, ip0, c->icur, c->iprev, nullptr, c->d_traces, c->d_wtab, c->launches - l0 + 1};
    c->k = k0; c->icur = ic0; c->iprev = ip0; c->launches = l0;
    if (s) { if (graph) cudaGraphDestroy(graph); *st = s; return -1; }
    if (e != cudaSuccess || !graph) {
        cudaGetLastError();
        c->opt_graph = 0;                 // fall back to plain launches
        return -1;
    }
    e = cudaGraphInstantiate(&gr.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c->opt_graph = 0;
        return -1;
    }
    c->graphs.push_back(gr);
    return (int)c->graphs.size() - 1;
}

// FD_OPT_RESERVE: prepare the context, grow the step tables for n more steps
// and capture the graphs the next fd_step calls will replay, so that none of
// that setup (allocation, synchronisation, capture) lands inside a timed region.
static fd_status reserve_steps(fd_ctx *c, int64_t n) {
    fd_status s;
    if (!c->started) {
        s = prepare(c);
        if (s) return s;
        c->started = true;
    }
    s = ensure_tables(c, c->k + n);
    if (s) return s;
    if (graphs_usable(c) && n >= graph_len(c)) {
        int ic = c->icur, ip = c->iprev;
        for (int guard = 0; guard < 8; ++guard) {
            const int sic = c->icur, sip = c->iprev;
            c->icur = ic; c->iprev = ip;
            int gi = -1;
            for (size_t q = 0; q < c->graphs.size(); ++q)
                if (c->graphs[q].icur == ic && c->graphs[q].iprev == ip && c->graphs[q].kt == c->d_traces &&
                    c->graphs[q].kw == c->d_wtab)
                    gi = (int)q;
            if (gi < 0) gi = capture_graph(c, &s);
            c->icur = sic; c->iprev = sip;
            if (s) return s;
            if (gi < 0) break;
            const int nic = c->graphs[gi].end_icur, nip = c->graphs[gi].end_iprev;
            if (nic == c->icur && nip == c->iprev) break;
            if (nic == ic && nip == ip) break;
            ic = nic; ip = nip;
        }
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return FD_OK;
}

// ======================================================================== C ABI
extern "C" {

fd_status fd_create(fd_ctx **out, int ndim, const int64_t *dims, double h, double dt, int order, const float *vel,
                    uint32_t flags) {
    return create_impl(out, ndim, dims, h, dt, order, vel, flags, 0, 1, -1, 0, nullptr);
}

fd_status fd_create_dist(fd_ctx **out, int ndim, const int64_t *global_dims, double h, double dt, int order,
                         const float *vel, uint32_t flags, const fd_dist *dist) {
    if (!dist) return fail(FD_ERR_ARG, "dist is NULL");
    return create_impl(out, ndim, global_dims, h, dt, order, vel, flags, dist->rank, dist->nranks, dist->device,
                       dist->vel_is_slab, dist->nccl_id);
}

fd_status fd_partition(int64_t nz, int nranks, int rank, int64_t *z0, int64_t *z1) {
    return partition(nz, nranks, rank, z0, z1);
}

fd_status fd_nccl_get_unique_id(void *out128) {
    if (!out128) return fail(FD_ERR_ARG, "out128 is NULL");
    NcclApi &n = nccl();
    if (!n.ok) return fail(FD_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
    ncclUniqueId id;
    ncclResult_t r = n.GetUniqueId(&id);
    if (r) return fail(FD_ERR_NCCL, "ncclGetUniqueId: %s", n.GetErrorString(r));
    memcpy(out128, &id, sizeof id);
    return FD_OK;
}

static fd_status check_ctx(fd_ctx *c) {
    if (!c) return fail(FD_ERR_ARG, "context is NULL");
    if (c->poisoned) return fail(FD_ERR_STATE, "context is poisoned by an earlier CUDA/NCCL error");
    return FD_OK;
}

static fd_status check_index(fd_ctx *c, const int64_t *idx, int64_t g[3]) {
    if (c->ndim == 2) { g[0] = idx[0]; g[1] = 0; g[2] = idx[1]; }
    else { g[0] = idx[0]; g[1] = idx[1]; g[2] = idx[2]; }
    if (g[0] < 0 || g[0] >= c->nzg || g[1] < 0 || g[1] >= c->nyg || g[2] < 0 || g[2] >= c->nxg)
        return fail(FD_ERR_RANGE, "index (%lld, %lld, %lld) outside the grid", (long long)g[0], (long long)g[1],
                    (long long)g[2]);
    return FD_OK;
}

fd_status fd_set_sponge(fd_ctx *c, int width, double alpha) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (width < 0 || !(alpha >= 0) || !std::isfinite(alpha)) return fail(FD_ERR_ARG, "width >= 0, alpha >= 0 finite");
    if (c->started || c->frozen) return fail(FD_ERR_STATE, "fd_set_sponge only before the first fd_step");
    c->sponge_nb = width;
    c->sponge_alpha = alpha;
    return FD_OK;
}

fd_status fd_add_source(fd_ctx *c, const int64_t *idx, double f, double t0, double amp) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!idx) return fail(FD_ERR_ARG, "idx is NULL");
    if (!(f > 0) || !std::isfinite(f)) return fail(FD_ERR_ARG, "f_peak_hz must be > 0");
    if (!std::isfinite(t0) || !std::isfinite(amp)) return fail(FD_ERR_ARG, "t0/amp must be finite");
    if (c->started) return fail(FD_ERR_STATE, "sources cannot change after the first fd_step");
    if ((int)c->src.size() >= kMaxSources) return fail(FD_ERR_ARG, "at most %d sources", kMaxSources);
    SourceDef d;
    s = check_index(c, idx, d.g);
    if (s) return s;
    d.f = f; d.t0 = t0; d.amp = amp;
    c->src.push_back(d);
    return FD_OK;
}

fd_status fd_set_receivers(fd_ctx *c, int64_t nrec, const int64_t *idx) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (nrec < 0 || (nrec > 0 && !idx)) return fail(FD_ERR_ARG, "bad nrec/idx");
    if (nrec > (int64_t)1 << 28) return fail(FD_ERR_ARG, "too many receivers");
    if (c->started) return fail(FD_ERR_STATE, "receivers cannot change after the first fd_step");
    std::vector<RecDef> r((size_t)nrec);
    for (int64_t j = 0; j < nrec; ++j) {
        s = check_index(c, idx + j * c->ndim, r[j].g);
        if (s) return s;
    }
    c->rec.swap(r);
    return FD_OK;
}

fd_status fd_step(fd_ctx *c, int64_t n) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (n < 0) return fail(FD_ERR_ARG, "n must be >= 0");
    if (n == 0) return FD_OK;
    if (c->peer_detached) return fail(FD_ERR_STATE, "fd_step after fd_peer_detach");
    s = check_peer_timeout(c);
    if (s) return s;
    if (!c->started) {
        s = prepare(c);
        if (s) return s;
        c->started = true;
    }
    s = ensure_tables(c, c->k + n);
    if (s) return s;
    if (!c->injected) {
        // add_source of step k on the current field by the owning slab;
        // later injections are eager.  Then refresh the halos of P.
        for (auto &sl : c->slabs) {
            StepParams p;
            fill_params(c, sl, nullptr, p, c->k - 1);   // w_{(k-1)+1} = w_k
            if (p.nsrc > 0) dispatch_inject(c, c->stream, cur_buf(c, sl), p);
        }
        if (c->nranks > 1 && c->opt_transport == 1) {
            // peer transport: push the initial halos (and K's, once) with copies
            if (c->opt_tsteps >= 2) s = peer_copy(c, {{c->icur, c->H}, {c->iprev, c->R}, {-1, c->R}}, c->stream);
            else s = peer_copy(c, {{c->icur, c->R}}, c->stream);
            if (s) return s;
            peer_signal(c, c->stream);
        } else if (c->slabs.size() > 1 || c->nranks > 1) {
            // halos of P (2r for temporal blocking) and, for temporal
            // blocking, r of P_prev (fd_set_wavefield may have set it)
            if (c->opt_tsteps >= 2) s = exchange(c, {{c->icur, c->H}, {c->iprev, c->R}}, c->stream);
            else s = exchange(c, {{c->icur, c->R}}, c->stream);
            if (s) return s;
        }
        c->injected = true;
    }
    int64_t i = 0;
    if (c->resident) {
        s = resident_steps(c, n);
        if (s) return s;
        i = n;
    }
    if (c->comm && c->opt_transport == 0 && c->k == 0 && c->opt_graph && !c->opt_profile && !c->resident &&
        n - i > graph_len(c)) {
        // NCCL exchanges are captured only after a first plain pass (NCCL's
        // lazy connection setup must happen outside any capture)
        const int S = (c->opt_tsteps >= 2 && c->tb2 >= 0) ? tb2_table()[c->tb2].steps : 1;
        s = advance_plain(c, S);
        if (s) return s;
        i += S;
    }
    if (graphs_usable(c) && n - i >= graph_len(c)) {
        // replay G-step graphs; the device counter d_k carries k
        set_step_kernel<<<1, 1, 0, c->stream>>>(c->d_k, c->k);
        ++c->launches;
        for (; n - i >= graph_len(c); i += graph_len(c)) {
            int gi = -1;
            for (size_t q = 0; q < c->graphs.size(); ++q) {
                auto &g = c->graphs[q];
                if (g.icur != c->icur || g.iprev != c->iprev) continue;
                if (g.kt != c->d_traces || g.kw != c->d_wtab) {   // tables moved: re-capture
                    cudaGraphExecDestroy(g.exec);
                    c->graphs.erase(c->graphs.begin() + q);
                    break;
                }
                gi = (int)q;
                break;
            }
            if (gi < 0) {
                gi = capture_graph(c, &s);
                if (s) return s;
                if (gi < 0) break;               // capture unsupported: plain launches
            }
            auto &g = c->graphs[gi];
            CUDA_TRY(c, cudaGraphLaunch(g.exec, c->stream));
            c->k += graph_len(c);
            c->graph_steps += graph_len(c);
            c->icur = g.end_icur;
            c->iprev = g.end_iprev;
            c->launches += g.launches;
        }
    }
    s = advance_plain(c, n - i);
    if (s) return s;
    if (!c->opt_async) {
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        s = check_peer_timeout(c);
        if (s) return s;
    }
    if (c->comm && nccl().CommGetAsyncError) {
        ncclResult_t ae = 0;
        nccl().CommGetAsyncError(c->comm, &ae);
        if (ae) {
            c->poisoned = true;
            return fail(FD_ERR_NCCL, "NCCL async error: %s", nccl().GetErrorString(ae));
        }
    }
    return FD_OK;
}

fd_status fd_get_wavefield(fd_ctx *c, int which, float *host_out) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!host_out) return fail(FD_ERR_ARG, "host_out is NULL");
    if (which != FD_FIELD_CUR && which != FD_FIELD_PREV) return fail(FD_ERR_ARG, "which must be CUR or PREV");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const int64_t pf = plane_floats(c);
    for (auto &sl : c->slabs) {
        const float *buf = which == FD_FIELD_CUR ? cur_buf(c, sl) : prev_buf(c, sl);
        float *dst = host_out + (sl.z0 - c->z0) * c->nyg * c->nxg;
        CUDA_TRY(c, cudaMemcpy2D(dst, c->nxg * 4, buf + (int64_t)c->H * pf, c->pitch * 4, c->nxg * 4,
                                 c->nyg * sl.nz, cudaMemcpyDeviceToHost));
        if (which == FD_FIELD_CUR && c->injected && !c->src.empty()) {
            // the CUR buffer already holds w_k (eager injection): restore the raw
            // P^k at each source point from the value recorded before its first add
            std::vector<float> raw(c->src.size());
            CUDA_TRY(c, cudaMemcpy(raw.data(), sl.d_src_raw, raw.size() * 4, cudaMemcpyDeviceToHost));
            for (int q = (int)c->src.size() - 1; q >= 0; --q) {
                const int64_t gz = c->src[q].g[0];
                if (gz < sl.z0 || gz >= sl.z1) continue;
                host_out[((gz - c->z0) * c->nyg + c->src[q].g[1]) * c->nxg + c->src[q].g[2]] = raw[q];
            }
        }
    }
    return FD_OK;
}

fd_status fd_get_traces(fd_ctx *c, float *host_out, int64_t cap, int64_t *nsteps_out) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!host_out || !nsteps_out) return fail(FD_ERR_ARG, "host_out/nsteps_out is NULL");
    const int64_t nrec = (int64_t)c->rec.size();
    if (nrec == 0) return fail(FD_ERR_STATE, "no receivers registered");
    if (cap < nrec * c->k)
        return fail(FD_ERR_STATE, "cap %lld < nrec*nsteps = %lld", (long long)cap, (long long)(nrec * c->k));
    *nsteps_out = c->k;
    if (c->k == 0) return FD_OK;
    // step-major -> receiver-major on the device (rows of receivers owned
    // elsewhere are 0), then one copy to the host
    std::vector<unsigned char> own((size_t)nrec, 0);
    for (int64_t j = 0; j < nrec; ++j) own[j] = c->rec[j].g[0] >= c->z0 && c->rec[j].g[0] < c->z1;
    const size_t bytes = (size_t)(nrec * c->k) * 4;
    float *d_out = (float *)dev_alloc(bytes);
    unsigned char *d_own = (unsigned char *)dev_alloc((size_t)nrec);
    if (!d_out || !d_own) {
        dev_free(d_out); dev_free(d_own);
        return fail(FD_ERR_NOMEM, "trace readback buffer allocation failed");
    }
    cudaError_t e = cudaMemcpyAsync(d_own, own.data(), (size_t)nrec, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) {
        const dim3 grid((unsigned)((nrec + 31) / 32), (unsigned)std::min<int64_t>((c->k + 31) / 32, 65535));
        traces_transpose_kernel<<<grid, dim3(32, 8), 0, c->stream>>>(c->d_traces, d_out, nrec, c->k, d_own);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(host_out, d_out, bytes, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    dev_free(d_out);
    dev_free(d_own);
    CUDA_TRY(c, e);
    return FD_OK;
}

// ---- peer transport (include/fd.h): IPC handles of the field buffers, K, flags
struct PeerBlob {
    uint32_t magic, version;
    int64_t nz, nxg, nyg, nzg;
    int32_t H, rank, nbuf, pad;
    cudaIpcMemHandle_t F[4], Kh, flags;
};
static_assert(sizeof(PeerBlob) <= FD_PEER_BLOB_BYTES, "peer blob size");
constexpr uint32_t kPeerMagic = 0x46445042u;   // "FDPB"

fd_status fd_peer_export(fd_ctx *c, void *blob, size_t cap, size_t *len) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!blob || !len) return fail(FD_ERR_ARG, "blob/len is NULL");
    if (cap < sizeof(PeerBlob)) return fail(FD_ERR_ARG, "cap %zu < %zu", cap, sizeof(PeerBlob));
    if (c->nranks < 2 || c->opt_transport != 1)
        return fail(FD_ERR_STATE, "fd_peer_export needs a multi-rank context with FD_OPT_TRANSPORT=1");
    if (c->peer_imported || c->started) return fail(FD_ERR_STATE, "fd_peer_export after fd_peer_import / fd_step");
    if (g_alloc) return fail(FD_ERR_STATE, "FD_OPT_TRANSPORT=1 needs the default allocator (CUDA IPC)");
    // all four field buffers (the two-step kernels' too) and the flags exist
    // from here on; the options are frozen (the mappings depend on them)
    Slab &ss = c->slabs[0];
    const size_t fbytes = (size_t)buf_floats(c, ss) * 4;
    for (int b = 2; b < 4; ++b) {
        if (ss.F[b]) continue;
        ss.F[b] = (float *)dev_alloc(fbytes);
        if (!ss.F[b]) return fail(FD_ERR_NOMEM, "field buffer allocation failed");
        CUDA_TRY(c, cudaMemset(ss.F[b], 0, fbytes));
        c->dev_bytes += (double)fbytes;
    }
    if (!c->h_perr) {
        CUDA_TRY(c, cudaHostAlloc((void **)&c->h_perr, sizeof(int), cudaHostAllocMapped));
        *c->h_perr = 0;
        CUDA_TRY(c, cudaHostGetDevicePointer((void **)&c->d_perr, c->h_perr, 0));
    }
    if (!c->d_flags) {
        CUDA_TRY(c, cudaMalloc(&c->d_flags, 2 * sizeof(int64_t)));
        CUDA_TRY(c, cudaMemset(c->d_flags, 0, 2 * sizeof(int64_t)));
    }
    c->frozen = true;
    // buffers zeroed / uploaded before any neighbour may write their halos
    CUDA_TRY(c, cudaDeviceSynchronize());
    PeerBlob b;
    memset(&b, 0, sizeof b);
    b.magic = kPeerMagic; b.version = 1;
    const Slab &sl = c->slabs[0];
    b.nz = sl.nz; b.nxg = c->nxg; b.nyg = c->nyg; b.nzg = c->nzg;
    b.H = c->H; b.rank = c->rank;
    for (int i = 0; i < 4 && sl.F[i]; ++i, ++b.nbuf) CUDA_TRY(c, cudaIpcGetMemHandle(&b.F[i], sl.F[i]));
    CUDA_TRY(c, cudaIpcGetMemHandle(&b.Kh, sl.Kh));
    CUDA_TRY(c, cudaIpcGetMemHandle(&b.flags, c->d_flags));
    memcpy(blob, &b, sizeof b);
    *len = sizeof b;
    return FD_OK;
}

fd_status fd_peer_import(fd_ctx *c, const void *lo_blob, const void *hi_blob) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (c->nranks < 2 || c->opt_transport != 1 || !c->frozen || c->started)
        return fail(FD_ERR_STATE, "fd_peer_import needs fd_peer_export first (FD_OPT_TRANSPORT=1, nranks > 1)");
    if (c->peer_imported) return fail(FD_ERR_STATE, "fd_peer_import called twice");
    if ((c->rank > 0) != (lo_blob != nullptr) || (c->rank < c->nranks - 1) != (hi_blob != nullptr))
        return fail(FD_ERR_ARG, "rank %d needs %s lower and %s upper blob", c->rank, c->rank > 0 ? "a" : "no",
                    c->rank < c->nranks - 1 ? "an" : "no");
    int nbuf = 0;
    while (nbuf < 4 && c->slabs[0].F[nbuf]) ++nbuf;
    auto open = [&](const void *raw, int want_rank, fd_ctx::Peer &pr) -> fd_status {
        PeerBlob b;
        memcpy(&b, raw, sizeof b);
        if (b.magic != kPeerMagic || b.version != 1 || b.nxg != c->nxg || b.nyg != c->nyg || b.nzg != c->nzg ||
            b.H != c->H || b.rank != want_rank || b.nbuf != nbuf)
            return fail(FD_ERR_STATE, "peer blob does not match this grid / rank %d", want_rank);
        auto map = [&](const cudaIpcMemHandle_t &h, void **out) -> fd_status {
            cudaError_t e = cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return fail(FD_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
            }
            pr.opened.push_back(*out);
            return FD_OK;
        };
        void *p = nullptr;
        for (int i = 0; i < nbuf; ++i) {
            fd_status st = map(b.F[i], &p);
            if (st) return st;
            pr.F[i] = (float *)p;
        }
        fd_status st = map(b.Kh, &p);
        if (st) return st;
        pr.Kh = (float *)p;
        st = map(b.flags, &p);
        if (st) return st;
        pr.flags = (int64_t *)p;
        pr.nz = b.nz;
        return FD_OK;
    };
    if (lo_blob) { s = open(lo_blob, c->rank - 1, c->plo); if (s) return s; }
    if (hi_blob) { s = open(hi_blob, c->rank + 1, c->phi); if (s) return s; }
    c->peer_imported = true;
    return FD_OK;
}

fd_status fd_peer_detach(fd_ctx *c) {
    if (!c) return fail(FD_ERR_ARG, "context is NULL");
    // finish every launch that may store into (or signal) the neighbours'
    // memory, then unmap it; the caller's barrier after this call orders the
    // neighbours' fd_destroy (which frees the exported buffers) after it
    cudaError_t e = cudaSuccess;
    if (c->stream) e = cudaStreamSynchronize(c->stream);
    if (c->comm_stream && e == cudaSuccess) e = cudaStreamSynchronize(c->comm_stream);
    for (auto *pr : {&c->plo, &c->phi}) {
        for (void *m : pr->opened) cudaIpcCloseMemHandle(m);
        pr->opened.clear();
        *pr = fd_ctx::Peer{};
    }
    if (c->peer_imported) c->peer_detached = true;
    CUDA_TRY(c, e);
    return FD_OK;
}

fd_status fd_destroy(fd_ctx *c) {
    if (!c) return FD_OK;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    destroy_all(c);
    delete c;
    std::lock_guard<std::mutex> lk(g_mu);
    --g_live_contexts;
    return FD_OK;
}

const char *fd_strerror(fd_status s) {
    switch (s) {
    case FD_OK: return "ok";
    case FD_ERR_ARG: return "invalid argument";
    case FD_ERR_RANGE: return "index out of range";
    case FD_ERR_UNSTABLE: return "CFL condition violated";
    case FD_ERR_NOMEM: return "out of memory";
    case FD_ERR_CUDA: return "CUDA error";
    case FD_ERR_NCCL: return "NCCL error";
    case FD_ERR_STATE: return "invalid state";
    default: return "unknown status";
    }
}

const char *fd_last_error(void) { return g_last_error.c_str(); }

fd_status fd_set_stream(fd_ctx *c, void *st) {
    fd_status s = check_ctx(c);
    if (s) return s;
    c->stream = (cudaStream_t)st;
    return FD_OK;
}

fd_status fd_set_allocator(void *(*alloc)(size_t, void *), void (*free_)(void *, void *), void *user) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_live_contexts > 0) return fail(FD_ERR_STATE, "fd_set_allocator with live contexts");
    if ((alloc == nullptr) != (free_ == nullptr)) return fail(FD_ERR_ARG, "alloc and free must both be set or NULL");
    g_alloc = alloc;
    g_free = free_;
    g_alloc_user = user;
    return FD_OK;
}

fd_status fd_set_wavefield(fd_ctx *c, int which, const float *host_in) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!host_in) return fail(FD_ERR_ARG, "host_in is NULL");
    if (which != FD_FIELD_CUR && which != FD_FIELD_PREV) return fail(FD_ERR_ARG, "which must be CUR or PREV");
    if (c->started) return fail(FD_ERR_STATE, "fd_set_wavefield only before the first fd_step");
    const int64_t pf = plane_floats(c);
    for (auto &sl : c->slabs) {
        float *buf = which == FD_FIELD_CUR ? cur_buf(c, sl) : prev_buf(c, sl);
        CUDA_TRY(c, cudaMemcpy2D(buf + (int64_t)c->H * pf, c->pitch * 4,
                                 host_in + (sl.z0 - c->z0) * c->nyg * c->nxg, c->nxg * 4, c->nxg * 4,
                                 c->nyg * sl.nz, cudaMemcpyHostToDevice));
    }
    return FD_OK;
}

fd_status fd_set_option(fd_ctx *c, int key, int64_t v) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (key == FD_OPT_ASYNC) { c->opt_async = v ? 1 : 0; return FD_OK; }
    if (key == FD_OPT_RESERVE) {
        if (v < 0) return fail(FD_ERR_ARG, "FD_OPT_RESERVE must be >= 0");
        return reserve_steps(c, v);
    }
    if (key == FD_OPT_PROFILE) {
        s = fold_times(c);
        if (s) return s;
        c->opt_profile = v ? 1 : 0;
        return FD_OK;
    }
    if (c->started || c->frozen)
        return fail(FD_ERR_STATE, "option %d only before the first fd_step / fd_peer_export", key);
    switch (key) {
    case FD_OPT_KERNEL:
        if (v < 0 || v > 3) return fail(FD_ERR_ARG, "FD_OPT_KERNEL must be 0, 1, 2 or 3");
        c->opt_kernel = (v == 2) ? 0 : (int)v;
        return FD_OK;
    case FD_OPT_TILE: {
        const auto &tab = tile_table();
        if (v >= (int64_t)tab.size() || v < -1) return fail(FD_ERR_ARG, "tile index out of range");
        if (v >= 0 && (tab[v].ndim != c->ndim || tab[v].r != c->R))
            return fail(FD_ERR_ARG, "tile %lld is for ndim=%d r=%d", (long long)v, tab[v].ndim, tab[v].r);
        c->opt_tile = (int)v;
        return FD_OK;
    }
    case FD_OPT_ZCHUNKS:
        if (v < 0 || v > 4096) return fail(FD_ERR_ARG, "bad zchunks");
        c->opt_zchunks = (int)v;
        return FD_OK;
    case FD_OPT_TSTEPS:
        if (v < 0 || v > 4) return fail(FD_ERR_ARG, "FD_OPT_TSTEPS must be 0 (auto), 1, 2, 3 or 4");
        c->opt_tsteps = (int)v;
        return FD_OK;
    case FD_OPT_TB2TILE:
        if (v < -1 || v >= (int64_t)tb2_table().size()) return fail(FD_ERR_ARG, "tb2 tile index out of range");
        c->opt_tb2tile = (int)v;
        return FD_OK;
    case FD_OPT_GRAPH: c->opt_graph = v ? 1 : 0; return FD_OK;
    case FD_OPT_TRANSPORT:
        if (v != 0 && v != 1) return fail(FD_ERR_ARG, "FD_OPT_TRANSPORT must be 0 or 1");
        c->opt_transport = (int)v;
        return FD_OK;
    case FD_OPT_KPLANE:
        if (v != 0 && v != 1) return fail(FD_ERR_ARG, "FD_OPT_KPLANE must be 0 or 1");
        c->opt_kplane = (int)v;
        return FD_OK;
    case FD_OPT_RESIDENT:
        if (v < 0 || v > 2) return fail(FD_ERR_ARG, "FD_OPT_RESIDENT must be 0, 1 or 2");
        c->opt_resident = (int)v;
        return FD_OK;
    case FD_OPT_CLUSTER:
        if (v != 0 && v != 2 && v != 4 && v != 8 && v != 16) return fail(FD_ERR_ARG, "FD_OPT_CLUSTER must be 0, 2, 4, 8 or 16");
        c->opt_cluster = (int)v;
        return FD_OK;
    case FD_OPT_VSLABS:
        if (v < 1 || v > 64) return fail(FD_ERR_ARG, "FD_OPT_VSLABS must be in [1, 64]");
        if (c->nranks > 1 && v != 1) return fail(FD_ERR_ARG, "FD_OPT_VSLABS is for single-process contexts");
        c->opt_vslabs = (int)v;
        return FD_OK;
    default: return fail(FD_ERR_ARG, "unknown option %d", key);
    }
}

fd_status fd_get_kernel_times(fd_ctx *c, double *ms, int64_t *launches) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!ms || !launches) return fail(FD_ERR_ARG, "ms/launches is NULL");
    s = fold_times(c);
    if (s) return s;
    for (int i = 0; i < FD_K_COUNT; ++i) { ms[i] = c->kms[i]; launches[i] = c->kcnt[i]; }
    return FD_OK;
}

fd_status fd_reset_kernel_times(fd_ctx *c) {
    fd_status s = check_ctx(c);
    if (s) return s;
    s = fold_times(c);
    if (s) return s;
    for (int i = 0; i < FD_K_COUNT; ++i) { c->kms[i] = 0; c->kcnt[i] = 0; }
    return FD_OK;
}

fd_status fd_get_info(fd_ctx *c, fd_info *o) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!o) return fail(FD_ERR_ARG, "out is NULL");
    memset(o, 0, sizeof *o);
    o->steps_done = c->k;
    o->kernel_launches = c->launches;
    o->local_dims[0] = c->z1 - c->z0;
    if (c->ndim == 3) { o->local_dims[1] = c->nyg; o->local_dims[2] = c->nxg; }
    else o->local_dims[1] = c->nxg;
    o->z0 = c->z0; o->z1 = c->z1;
    o->pitch = c->pitch;
    o->order = c->order;
    o->device_bytes = c->dev_bytes;
    o->steps_per_launch = (c->opt_tsteps >= 2 && c->tb2 >= 0) ? tb2_table()[c->tb2].steps : 1;
    o->tb_kind = (c->opt_tsteps >= 2 && c->tb2 >= 0) ? tb2_table()[c->tb2].kind : 0;
    o->kplane = c->kplane ? 1 : 0;
    o->graph_steps = c->graph_steps;
    if (c->comm && nccl().CommCount) {
        int n = 0;
        if (nccl().CommCount(c->comm, &n) == 0) o->comm_nranks = n;
    }
    if (c->opt_kernel != 0) { o->kernel = c->opt_kernel; return FD_OK; }
    o->kernel = 2;
    if (c->resident) {
        o->steps_per_launch = 0;
        o->cluster_ctas = c->res_nc;
        o->ctas = c->res_nc; o->threads_per_cta = c->res_threads; o->smem_bytes = c->res_smem;
        return FD_OK;
    }
    if (c->opt_tsteps >= 2 && c->tb2 >= 0) {
        const TileCfg &t = tb2_table()[c->tb2];
        o->tile_x = t.tx; o->tile_y = t.ty; o->rows_per_thread = t.ny;
        o->p_stages = 2 * t.r + 1 + t.dp; o->k_stages = t.r + 1 + t.dk;
        o->threads_per_cta = t.threads; o->smem_bytes = t.smem;
        int ctas = 0, zc = 0;
        for (auto &sl : c->slabs)
            for (auto &g : sl.tb2) { ctas += g.lin > 0 ? g.lin : (int)(ntiles_of(c, t) * g.zchunks); zc = std::max(zc, g.zchunks); }
        o->zchunks = zc;
        o->ctas = ctas;
        return FD_OK;
    }
    if (!c->started) choose_tile(c, c->z1 - c->z0);
    if (c->tile >= 0) {
        const TileCfg &t = tile_table()[c->tile];
        o->tile_x = t.tx; o->tile_y = t.ty; o->rows_per_thread = t.ny;
        o->p_stages = t.r + 1 + t.dp; o->k_stages = t.dk + 1;
        o->threads_per_cta = t.threads; o->smem_bytes = t.smem;
        int ctas = 0, zc = 0;
        for (auto &sl : c->slabs)
            for (auto &g : sl.regions) { ctas += (int)(ntiles_of(c, t) * g.zchunks); zc = std::max(zc, g.zchunks); }
        if (!c->started) { zc = chunks_for(c, t, c->occ, c->z1 - c->z0); ctas = (int)(ntiles_of(c, t) * zc); }
        o->ctas = ctas;
        o->zchunks = zc;
    }
    return FD_OK;
}

}  // extern "C"
