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
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fd.h"
#include "fd_kernels.cuh"

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
                     int bx, int by) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * 4), (cuuint64_t)(pitch * ny * 4)};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// ------------------------------------------------------------ kernel table
typedef void (*launch_fused_t)(dim3, int, cudaStream_t, const CUtensorMap &, const CUtensorMap &,
                               const CUtensorMap &, const StepParams &);

struct TileCfg {
    int ndim, r, tx, ty, ny, dp, dk;
    int pbw, tbw;        // TMA box widths (halo'd p row piece, p_prev/K row piece)
    int threads, smem;
    const void *kernel;
    launch_fused_t launch;
};

template <class C>
static void launch_fused(dim3 grid, int smem, cudaStream_t st, const CUtensorMap &a, const CUtensorMap &b,
                         const CUtensorMap &c, const StepParams &p) {
    fused_step_kernel<C><<<grid, C::NTHREADS, smem, st>>>(a, b, c, p);
}

template <int R, int NDIM, int TX, int TY, int NY, int DP, int DK>
static TileCfg make_cfg() {
    using C = Cfg<R, NDIM, TX, TY, NY, DP, DK>;
    return TileCfg{NDIM, R, TX, TY, NY, DP, DK, C::PBW, C::TBW, C::NTHREADS, C::SMEM_BYTES,
                   (const void *)fused_step_kernel<C>, launch_fused<C>};
}

// Compiled tiles.  3D: 4 x-y tiles per r (rows per thread 4 for r <= 2, 2 above,
// to bound the register queue); 2D: row strips of 256/512/1024 columns.
#define CFG3(R, NY) make_cfg<R, 3, 64, 32, NY, 2, 2>(), make_cfg<R, 3, 128, 32, NY, 2, 2>(), \
                    make_cfg<R, 3, 64, 16, NY, 2, 2>(), make_cfg<R, 3, 128, 16, NY, 2, 2>()
#define CFG3W(R, NY) make_cfg<R, 3, 64, 32, NY, 2, 2>(), make_cfg<R, 3, 32, 32, NY, 2, 2>(), \
                     make_cfg<R, 3, 64, 16, NY, 2, 2>(), make_cfg<R, 3, 128, 16, NY, 2, 2>()
#define CFG2(R) make_cfg<R, 2, 256, 1, 1, 6, 6>(), make_cfg<R, 2, 512, 1, 1, 6, 6>(), \
                make_cfg<R, 2, 1024, 1, 1, 4, 4>()
static const std::vector<TileCfg> &tile_table() {
    static const std::vector<TileCfg> t = {CFG3(1, 4), CFG3(2, 4), CFG3W(3, 2), CFG3W(4, 2),
                                           CFG2(1),    CFG2(2),    CFG2(3),    CFG2(4)};
    return t;
}

// ------------------------------------------------------------------ context
struct SourceDef {
    int64_t g[3];     // global (z, y, x)
    double f, t0, amp;
};
struct RecDef {
    int64_t g[3];
};

struct fd_ctx {
    int ndim = 0, order = 0, R = 0;
    double h = 0, dt = 0;
    int64_t nxg = 0, nyg = 0, nzg = 0;    // global extents (ny = 1 in 2D)
    int64_t nz = 0, z0 = 0, z1 = 0;       // local planes [z0, z1)
    int64_t pitch = 0;
    int rank = 0, nranks = 1, device = 0;
    bool poisoned = false;
    bool started = false;
    bool injected = false;                // w_k already injected into the CUR buffer
    int64_t k = 0;                        // steps done
    int64_t launches = 0;
    cudaStream_t stream = nullptr;
    float *A = nullptr, *B = nullptr, *K = nullptr;   // A = current p after even #steps
    bool cur_is_A = true;
    std::vector<SourceDef> src;
    std::vector<RecDef> rec;
    // device-side receiver tables
    int32_t *d_rec = nullptr;             // [5 * nrec_local + nunits + 1]
    int nrec_local = 0;
    float *d_traces = nullptr;            // step-major [trace_cap][nrec]
    int64_t trace_cap = 0;
    float *d_src_raw = nullptr;
    std::vector<float> h_src_raw;
    // kernel configuration
    int opt_kernel = 0, opt_tile = -1, opt_zchunks = 0, opt_async = 0, opt_graph = 1, opt_vslabs = 1;
    int tile = -1, zchunks = 1, ctas = 0;
    CUtensorMap mapA_halo, mapB_halo, mapA_tile, mapB_tile, mapK;
    bool maps_ready = false;
    double dev_bytes = 0;
};

static inline int64_t buf_floats(const fd_ctx *c) { return (c->nz + 2 * c->R) * c->nyg * c->pitch; }
static inline float *cur_buf(fd_ctx *c) { return c->cur_is_A ? c->A : c->B; }
static inline float *prev_buf(fd_ctx *c) { return c->cur_is_A ? c->B : c->A; }

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

static void destroy_buffers(fd_ctx *c) {
    dev_free(c->A); dev_free(c->B); dev_free(c->K);
    dev_free(c->d_rec); dev_free(c->d_traces); dev_free(c->d_src_raw);
    c->A = c->B = c->K = nullptr;
    c->d_rec = nullptr; c->d_traces = nullptr; c->d_src_raw = nullptr;
}

static fd_status create_impl(fd_ctx **out, int ndim, const int64_t *dims, double h, double dt, int order,
                             const float *vel, uint32_t flags, int rank, int nranks, int device, int vel_is_slab) {
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
    int64_t z0 = 0, z1 = nzg;
    if (nranks > 1 || rank != 0) {
        fd_status s = partition(nzg, nranks, rank, &z0, &z1);
        if (s) return s;
        if (z1 - z0 < R) return fail(FD_ERR_ARG, "slab of %lld planes thinner than r=%d", (long long)(z1 - z0), R);
    }
    const int64_t nz = z1 - z0;
    const int64_t plane = nyg * nxg;
    const float *vloc = vel + (vel_is_slab ? 0 : z0 * plane);
    const int64_t nloc = nz * plane;
    // validate velocity and the CFL condition (R#8) on host metadata first
    double vmax = 0;
    for (int64_t i = 0; i < nloc; ++i) {
        const float v = vloc[i];
        if (!(v > 0.f) || !std::isfinite(v))
            return fail(FD_ERR_ARG, "velocity[%lld] = %g is not finite and > 0", (long long)i, (double)v);
        vmax = std::max(vmax, (double)v);
    }
    const double ratio = vmax * dt / h, lim = cfl_limit(ndim, R);
    if (!(flags & FD_FLAG_ALLOW_UNSTABLE) && ratio > lim)
        return fail(FD_ERR_UNSTABLE, "unstable: max(v)*dt/h = %.6f exceeds the CFL limit %.6f (ratio %.4f)", ratio,
                    lim, ratio / lim);

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(FD_ERR_CUDA, "no CUDA device available");
    }
    if (device >= 0) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return fail(FD_ERR_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
    }
    fd_ctx *c = new fd_ctx();
    c->ndim = ndim; c->order = order; c->R = R; c->h = h; c->dt = dt;
    c->nxg = nxg; c->nyg = nyg; c->nzg = nzg; c->z0 = z0; c->z1 = z1; c->nz = nz;
    c->rank = rank; c->nranks = nranks;
    cudaGetDevice(&c->device);
    c->pitch = (nxg + 31) / 32 * 32;
    const size_t fbytes = (size_t)buf_floats(c) * 4;
    const size_t kbytes = (size_t)(nz * nyg * c->pitch) * 4;
    c->A = (float *)dev_alloc(fbytes);
    c->B = (float *)dev_alloc(fbytes);
    c->K = (float *)dev_alloc(kbytes);
    c->d_src_raw = (float *)dev_alloc(kMaxSources * 4);
    if (!c->A || !c->B || !c->K || !c->d_src_raw) {
        destroy_buffers(c);
        delete c;
        return fail(FD_ERR_NOMEM, "device allocation of %.3f GB failed", (2.0 * fbytes + kbytes) / 1e9);
    }
    c->dev_bytes = 2.0 * fbytes + kbytes;
    // K = (v dt / h)^2 / scale in fp64, rounded once (R#7), padded rows zero
    std::vector<float> Kh((size_t)(nz * nyg * c->pitch), 0.f);
    const double sc = scale_of(R);
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < nyg; ++y) {
            const float *vr = vloc + (z * nyg + y) * nxg;
            float *kr = Kh.data() + (z * nyg + y) * c->pitch;
            for (int64_t x = 0; x < nxg; ++x) {
                const double cv = (double)vr[x] * dt / h;
                kr[x] = (float)(cv * cv / sc);
            }
        }
    cudaError_t e = cudaMemcpy(c->K, Kh.data(), kbytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(c->A, 0, fbytes);
    if (e == cudaSuccess) e = cudaMemset(c->B, 0, fbytes);
    if (e == cudaSuccess) e = cudaMemset(c->d_src_raw, 0, kMaxSources * 4);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        destroy_buffers(c);
        delete c;
        return fail(FD_ERR_CUDA, "device setup failed: %s", cudaGetErrorString(e));
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        ++g_live_contexts;
    }
    *out = c;
    return FD_OK;
}

// ------------------------------------------------------------ kernel choice
static int occupancy(const TileCfg &t) {
    int n = 0;
    cudaFuncSetAttribute(t.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, t.kernel, t.threads, t.smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Pick the tile and z-chunk count: prefer one full wave of co-resident CTAs
// (chunk-major order keeps neighbours in step for L2 halo reuse), then the
// smallest halo re-read factor.
static void choose_config(fd_ctx *c, int64_t span) {
    const auto &tab = tile_table();
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    double best = -1;
    int bi = -1, bchunks = 1;
    for (int i = 0; i < (int)tab.size(); ++i) {
        const TileCfg &t = tab[i];
        if (t.ndim != c->ndim || t.r != c->R) continue;
        if (c->opt_tile >= 0 && i != c->opt_tile) continue;
        const int occ = occupancy(t);
        if (occ <= 0) continue;
        const int64_t slots = (int64_t)nsm * occ;
        const int64_t ntiles = ((c->nxg + t.tx - 1) / t.tx) * ((c->nyg + t.ty - 1) / t.ty);
        int64_t chunks = c->opt_zchunks > 0 ? c->opt_zchunks : std::max<int64_t>(1, slots / ntiles);
        chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, span / std::max(4 * c->R, 8)));
        const int64_t units = ntiles * chunks;
        const int64_t waves = (units + slots - 1) / slots;
        const double fill = (double)units / (double)(waves * slots);
        const double halo = (double)(t.tx + 8) * (t.ty + (c->ndim == 3 ? 2 * c->R : 0)) / ((double)t.tx * t.ty);
        const double warm = (double)(2 * c->R * chunks) / (double)span;
        const double bytes = 12.0 + 4.0 * (halo + warm);
        const double score = fill * 16.0 / bytes;
        if (score > best) { best = score; bi = i; bchunks = (int)chunks; }
    }
    c->tile = bi;
    c->zchunks = bchunks;
}

static fd_status prepare(fd_ctx *c) {
    if (c->maps_ready) return FD_OK;
    if (c->opt_kernel == 1) { c->maps_ready = true; return FD_OK; }
    choose_config(c, c->nz);
    if (c->tile < 0) return fail(FD_ERR_CUDA, "no fused kernel configuration fits this device");
    const TileCfg &t = tile_table()[c->tile];
    const int64_t planes = c->nz + 2 * c->R;
    const int hy = c->ndim == 3 ? c->R : 0;
    bool ok = make_map(&c->mapA_halo, c->A, c->nxg, c->nyg, planes, c->pitch, t.pbw, t.ty + 2 * hy) &&
              make_map(&c->mapB_halo, c->B, c->nxg, c->nyg, planes, c->pitch, t.pbw, t.ty + 2 * hy) &&
              make_map(&c->mapA_tile, c->A, c->nxg, c->nyg, planes, c->pitch, t.tbw, t.ty) &&
              make_map(&c->mapB_tile, c->B, c->nxg, c->nyg, planes, c->pitch, t.tbw, t.ty) &&
              make_map(&c->mapK, c->K, c->nxg, c->nyg, c->nz, c->pitch, t.tbw, t.ty);
    if (!ok) {
        c->poisoned = true;
        return fail(FD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    }
    CUDA_TRY(c, cudaFuncSetAttribute(t.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem));
    c->maps_ready = true;
    return FD_OK;
}

// Build device receiver tables: local receivers sorted by (work unit, z), CSR
// offsets per unit (fused) -- or a flat list (naive).
static fd_status upload_receivers(fd_ctx *c) {
    dev_free(c->d_rec);
    c->d_rec = nullptr;
    struct L { int32_t unit, z, y, x, id; };
    std::vector<L> loc;
    int ntx = 1, nty = 1, ntiles = 1;
    const TileCfg *t = c->tile >= 0 ? &tile_table()[c->tile] : nullptr;
    if (t) {
        ntx = (int)((c->nxg + t->tx - 1) / t->tx);
        nty = (int)((c->nyg + t->ty - 1) / t->ty);
        ntiles = ntx * nty;
    }
    for (size_t j = 0; j < c->rec.size(); ++j) {
        const int64_t gz = c->rec[j].g[0];
        if (gz < c->z0 || gz >= c->z1) continue;
        L l{0, (int32_t)(gz - c->z0), (int32_t)c->rec[j].g[1], (int32_t)c->rec[j].g[2], (int32_t)j};
        if (t) {
            const int64_t span = c->nz;
            int ch = 0;
            // chunk containing plane z: the largest ch with floor(span*ch/nchunks) <= z
            for (int q = 0; q < c->zchunks; ++q)
                if ((span * q) / c->zchunks <= l.z) ch = q;
            l.unit = ch * ntiles + (l.y / t->ty) * ntx + (l.x / t->tx);
        }
        loc.push_back(l);
    }
    std::stable_sort(loc.begin(), loc.end(), [](const L &a, const L &b) {
        return a.unit != b.unit ? a.unit < b.unit : a.z < b.z;
    });
    const int nunits = t ? ntiles * c->zchunks : 0;
    const int n = (int)loc.size();
    c->nrec_local = n;
    std::vector<int32_t> h((size_t)5 * n + nunits + 1, 0);
    for (int i = 0; i < n; ++i) {
        h[i] = loc[i].z; h[n + i] = loc[i].y; h[2 * n + i] = loc[i].x; h[3 * n + i] = loc[i].id;
    }
    int32_t *off = h.data() + 4 * n;
    for (int u = 0, i = 0; u <= nunits; ++u) {
        while (i < n && loc[i].unit < u) ++i;
        off[u] = i;
    }
    c->d_rec = (int32_t *)dev_alloc(h.size() * 4);
    if (!c->d_rec) return fail(FD_ERR_NOMEM, "receiver table allocation failed");
    CUDA_TRY(c, cudaMemcpy(c->d_rec, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    return FD_OK;
}

static fd_status ensure_traces(fd_ctx *c, int64_t steps_needed) {
    const int64_t nrec = (int64_t)c->rec.size();
    if (nrec == 0 || steps_needed <= c->trace_cap) return FD_OK;
    int64_t cap = std::max<int64_t>(steps_needed, 2 * c->trace_cap);
    cap = std::max<int64_t>(cap, 16);
    float *nb = (float *)dev_alloc((size_t)(cap * nrec) * 4);
    if (!nb) return fail(FD_ERR_NOMEM, "trace buffer allocation failed");
    CUDA_TRY(c, cudaMemsetAsync(nb, 0, (size_t)(cap * nrec) * 4, c->stream));
    if (c->d_traces) {
        CUDA_TRY(c, cudaMemcpyAsync(nb, c->d_traces, (size_t)(c->trace_cap * nrec) * 4, cudaMemcpyDeviceToDevice,
                                    c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        dev_free(c->d_traces);
    }
    c->d_traces = nb;
    c->trace_cap = cap;
    return FD_OK;
}

static void fill_params(fd_ctx *c, StepParams &p, int64_t step_k) {
    memset(&p, 0, sizeof p);
    p.nx = c->nxg; p.ny = c->nyg; p.nz = c->nz;
    p.pitch = c->pitch; p.gz0 = c->z0; p.nzg = c->nzg;
    p.zlo = 0; p.zhi = (int32_t)c->nz;
    p.nsrc = (int32_t)c->src.size();
    for (int s = 0; s < p.nsrc; ++s) {
        p.sz[s] = (int32_t)(c->src[s].g[0] - c->z0);
        p.sy[s] = (int32_t)c->src[s].g[1];
        p.sx[s] = (int32_t)c->src[s].g[2];
        // w_{k+1}: the value injected into P^{k+1} by this launch (eager form)
        p.w[s] = (float)(c->src[s].amp * ricker((double)(step_k + 1) * c->dt, c->src[s].f, c->src[s].t0));
    }
    p.src_raw = c->d_src_raw;
    const int n = c->nrec_local;
    if (c->d_rec) {
        p.rec.z = c->d_rec;
        p.rec.y = c->d_rec + n;
        p.rec.x = c->d_rec + 2 * n;
        p.rec.id = c->d_rec + 3 * n;
        p.rec.off = (c->opt_kernel == 1) ? nullptr : c->d_rec + 4 * n;
    }
    p.nrec_local = n;
    p.trace_row = c->d_traces ? c->d_traces + step_k * (int64_t)c->rec.size() : nullptr;
}

template <int R> static void launch_inject(fd_ctx *c, float *field, const StepParams &p) {
    inject_kernel<R><<<1, 32, 0, c->stream>>>(field, p);
}
template <int R, int NDIM> static void launch_naive(fd_ctx *c, const StepParams &p) {
    const int64_t total = c->nxg * c->nyg * c->nz;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    naive_step_kernel<R, NDIM><<<blocks, 256, 0, c->stream>>>(p);
}
template <int R> static void launch_gather(fd_ctx *c, const StepParams &p) {
    gather_receivers_kernel<R><<<(c->nrec_local + 127) / 128, 128, 0, c->stream>>>(p);
}

static void dispatch_inject(fd_ctx *c, float *field, const StepParams &p) {
    switch (c->R) {
    case 1: launch_inject<1>(c, field, p); break;
    case 2: launch_inject<2>(c, field, p); break;
    case 3: launch_inject<3>(c, field, p); break;
    default: launch_inject<4>(c, field, p); break;
    }
    ++c->launches;
}

static fd_status one_step(fd_ctx *c) {
    StepParams p;
    fill_params(c, p, c->k);
    float *cur = cur_buf(c), *prev = prev_buf(c);
    p.pnext = prev;
    p.p = cur;
    p.K = c->K;
    if (c->opt_kernel == 1) {
        // naive path: stencil, receivers, injection (three launches)
        switch (c->R * 10 + c->ndim) {
        case 12: launch_naive<1, 2>(c, p); break;
        case 13: launch_naive<1, 3>(c, p); break;
        case 22: launch_naive<2, 2>(c, p); break;
        case 23: launch_naive<2, 3>(c, p); break;
        case 32: launch_naive<3, 2>(c, p); break;
        case 33: launch_naive<3, 3>(c, p); break;
        case 42: launch_naive<4, 2>(c, p); break;
        default: launch_naive<4, 3>(c, p); break;
        }
        ++c->launches;
        if (c->nrec_local > 0) {
            switch (c->R) {
            case 1: launch_gather<1>(c, p); break;
            case 2: launch_gather<2>(c, p); break;
            case 3: launch_gather<3>(c, p); break;
            default: launch_gather<4>(c, p); break;
            }
            ++c->launches;
        }
        if (p.nsrc > 0) dispatch_inject(c, prev, p);
    } else {
        const TileCfg &t = tile_table()[c->tile];
        p.ntx = (int32_t)((c->nxg + t.tx - 1) / t.tx);
        p.nty = (int32_t)((c->nyg + t.ty - 1) / t.ty);
        p.nchunks = c->zchunks;
        const dim3 grid((unsigned)(p.ntx * p.nty * p.nchunks));
        c->ctas = (int)grid.x;
        const CUtensorMap &mp = c->cur_is_A ? c->mapA_halo : c->mapB_halo;
        const CUtensorMap &mpp = c->cur_is_A ? c->mapB_tile : c->mapA_tile;
        t.launch(grid, t.smem, c->stream, mp, mpp, c->mapK, p);
        ++c->launches;
    }
    CUDA_TRY(c, cudaGetLastError());
    c->cur_is_A = !c->cur_is_A;
    ++c->k;
    return FD_OK;
}

// ======================================================================== C ABI
extern "C" {

fd_status fd_create(fd_ctx **out, int ndim, const int64_t *dims, double h, double dt, int order, const float *vel,
                    uint32_t flags) {
    return create_impl(out, ndim, dims, h, dt, order, vel, flags, 0, 1, -1, 0);
}

fd_status fd_create_dist(fd_ctx **out, int ndim, const int64_t *global_dims, double h, double dt, int order,
                         const float *vel, uint32_t flags, const fd_dist *dist) {
    if (!dist) return fail(FD_ERR_ARG, "dist is NULL");
    if (dist->nranks > 1)
        return fail(FD_ERR_NCCL, "multi-rank NCCL contexts are not available in this build");
    return create_impl(out, ndim, global_dims, h, dt, order, vel, flags, dist->rank, dist->nranks, dist->device,
                       dist->vel_is_slab);
}

fd_status fd_partition(int64_t nz, int nranks, int rank, int64_t *z0, int64_t *z1) {
    return partition(nz, nranks, rank, z0, z1);
}

fd_status fd_nccl_get_unique_id(void *out128) {
    if (!out128) return fail(FD_ERR_ARG, "out128 is NULL");
    return fail(FD_ERR_NCCL, "NCCL support is not available in this build");
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
    if (!c->started) {
        s = prepare(c);
        if (s) return s;
        s = upload_receivers(c);
        if (s) return s;
        c->started = true;
    }
    s = ensure_traces(c, c->k + n);
    if (s) return s;
    if (!c->injected) {
        // add_source of step k on the current field; later injections are eager
        StepParams p;
        fill_params(c, p, c->k - 1);   // w_{(k-1)+1} = w_k
        if (p.nsrc > 0) dispatch_inject(c, cur_buf(c), p);
        c->injected = true;
    }
    for (int64_t i = 0; i < n; ++i) {
        s = one_step(c);
        if (s) return s;
    }
    if (!c->opt_async) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return FD_OK;
}

fd_status fd_get_wavefield(fd_ctx *c, int which, float *host_out) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!host_out) return fail(FD_ERR_ARG, "host_out is NULL");
    if (which != FD_FIELD_CUR && which != FD_FIELD_PREV) return fail(FD_ERR_ARG, "which must be CUR or PREV");
    const float *buf = which == FD_FIELD_CUR ? cur_buf(c) : prev_buf(c);
    const float *src = buf + (int64_t)c->R * c->nyg * c->pitch;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    CUDA_TRY(c, cudaMemcpy2D(host_out, c->nxg * 4, src, c->pitch * 4, c->nxg * 4, c->nyg * c->nz,
                             cudaMemcpyDeviceToHost));
    if (which == FD_FIELD_CUR && c->injected && !c->src.empty()) {
        // the CUR buffer already holds w_k (eager injection): restore the raw
        // P^k at each source point from the value recorded before its first add
        std::vector<float> raw(c->src.size());
        CUDA_TRY(c, cudaMemcpy(raw.data(), c->d_src_raw, raw.size() * 4, cudaMemcpyDeviceToHost));
        for (int s2 = (int)c->src.size() - 1; s2 >= 0; --s2) {
            const int64_t gz = c->src[s2].g[0];
            if (gz < c->z0 || gz >= c->z1) continue;
            host_out[((gz - c->z0) * c->nyg + c->src[s2].g[1]) * c->nxg + c->src[s2].g[2]] = raw[s2];
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
    if (cap < nrec * c->k) return fail(FD_ERR_STATE, "cap %lld < nrec*nsteps = %lld", (long long)cap,
                                       (long long)(nrec * c->k));
    *nsteps_out = c->k;
    if (c->k == 0) return FD_OK;
    std::vector<float> tmp((size_t)(nrec * c->k));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    CUDA_TRY(c, cudaMemcpy(tmp.data(), c->d_traces, tmp.size() * 4, cudaMemcpyDeviceToHost));
    // step-major -> receiver-major; rows of receivers owned elsewhere are 0
    std::vector<char> own((size_t)nrec, 0);
    for (int64_t j = 0; j < nrec; ++j) own[j] = c->rec[j].g[0] >= c->z0 && c->rec[j].g[0] < c->z1;
    for (int64_t j = 0; j < nrec; ++j)
        for (int64_t k = 0; k < c->k; ++k) host_out[j * c->k + k] = own[j] ? tmp[k * nrec + j] : 0.f;
    return FD_OK;
}

fd_status fd_destroy(fd_ctx *c) {
    if (!c) return FD_OK;
    if (c->stream) cudaStreamSynchronize(c->stream);
    destroy_buffers(c);
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
    float *buf = which == FD_FIELD_CUR ? cur_buf(c) : prev_buf(c);
    CUDA_TRY(c, cudaMemcpy2D(buf + (int64_t)c->R * c->nyg * c->pitch, c->pitch * 4, host_in, c->nxg * 4,
                             c->nxg * 4, c->nyg * c->nz, cudaMemcpyHostToDevice));
    return FD_OK;
}

fd_status fd_set_option(fd_ctx *c, int key, int64_t v) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (c->started) return fail(FD_ERR_STATE, "options only before the first fd_step");
    switch (key) {
    case FD_OPT_KERNEL:
        if (v < 0 || v > 2) return fail(FD_ERR_ARG, "FD_OPT_KERNEL must be 0, 1 or 2");
        c->opt_kernel = (int)v == 2 ? 0 : (int)v;
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
    case FD_OPT_ASYNC: c->opt_async = v ? 1 : 0; return FD_OK;
    case FD_OPT_GRAPH: c->opt_graph = v ? 1 : 0; return FD_OK;
    case FD_OPT_VSLABS:
        if (v != 1) return fail(FD_ERR_ARG, "virtual slabs are not available in this build");
        c->opt_vslabs = 1;
        return FD_OK;
    default: return fail(FD_ERR_ARG, "unknown option %d", key);
    }
}

fd_status fd_get_info(fd_ctx *c, fd_info *o) {
    fd_status s = check_ctx(c);
    if (s) return s;
    if (!o) return fail(FD_ERR_ARG, "out is NULL");
    memset(o, 0, sizeof *o);
    o->steps_done = c->k;
    o->kernel_launches = c->launches;
    o->local_dims[0] = c->nz;
    if (c->ndim == 3) { o->local_dims[1] = c->nyg; o->local_dims[2] = c->nxg; }
    else o->local_dims[1] = c->nxg;
    o->z0 = c->z0; o->z1 = c->z1;
    o->pitch = c->pitch;
    o->order = c->order;
    o->device_bytes = c->dev_bytes;
    if (c->opt_kernel == 1) { o->kernel = 1; return FD_OK; }
    if (!c->maps_ready) choose_config(c, c->nz);
    o->kernel = 2;
    if (c->tile >= 0) {
        const TileCfg &t = tile_table()[c->tile];
        o->tile_x = t.tx; o->tile_y = t.ty; o->rows_per_thread = t.ny;
        o->p_stages = t.r + 1 + t.dp; o->k_stages = t.dk + 1;
        o->threads_per_cta = t.threads; o->smem_bytes = t.smem;
        o->zchunks = c->zchunks;
        o->ctas = (int)(((c->nxg + t.tx - 1) / t.tx) * ((c->nyg + t.ty - 1) / t.ty) * c->zchunks);
    }
    return FD_OK;
}

}  // extern "C"
