// fd_kernels.cuh -- sm_100a device code of the fused acoustic FD time step.
//
// One launch = one time step of Listing 3's run() body:
//   add_source (eager form, see below) ; fd_pzz ; [fd_pyy] ; fd_pxx ; fd_time ;
//   swap  (host pointer swap, zero bytes)
// fused into one pass that reads p, p_prev, K once and writes p_next once
// (16 B per grid-point update).
//
// Canonical per-point fp32 expression (every GPU variant evaluates exactly this,
// which makes "fused == naive" and "N slabs == 1 slab" bitwise contracts):
//   s_a = c0*p_i ; s_a = fma(c_m, p_{i-m e_a} + p_{i+m e_a}, s_a)  m = 1..r
//   S   = [x in] s_x ; S = [y in] S + s_y ; S = [z in] S + s_z     (band rule, R#3)
//   p_next_i = fma(K_i, S, fma(2, p_i, -p_prev_i))
// with integer-scaled taps c (x1, x12, x180, x5040; the 1/scale is folded into
// K = (v dt / h)^2 / scale, computed once on the host in fp64).
//
// Source injection is applied EAGERLY: the kernel of step k, after
// computing p_next = P^{k+1} at a source point, stores the raw value (for
// readback and receivers) and then adds w_{k+1} in registration order, so the
// memory holds exactly the P that step k+1's add_source would produce.  This
// is the same fp32 add on the same operands as in-place injection.
//
// Memory layout (HBM): each field buffer holds (nz_local + 4r) planes of
// ny rows of `pitch` floats (pitch = nx rounded up to 32 floats = 128 B); plane
// z of the slab lives at buffer plane z + 2r (halo_planes); the 2r planes on
// each side are zero (single GPU / global faces) or halo copies (slabs).  K
// has nz_local planes with the same pitch, plus r halo planes on each side.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace fdk {

constexpr int kMaxSources = 16;
// FD_OPT_KPLANE tables hold kKzPad zero entries beyond each end of a slab's
// planes (the 2D row-block kernels evaluate up to one block past zhi)
constexpr int kKzPad = 512;
// r >= 3 z-tap queues of the single-step 3D kernel shift every kQShift planes
// (scripts/ab_qshift.sh, C3 order 8: 382 / 390 / 389 / 376 Gpts/s for 1 / 2 / 3 / 4)
#ifndef FD_QSHIFT
#define FD_QSHIFT 2
#endif
constexpr int kQShift = FD_QSHIFT;
// packed fp32 (FFMA2/FADD2) evaluation of the canonical expression in the
// single-step 3D kernel's band-rule variants (FD_PACKED=0: scalar).  ncu r05:
// order 8 242 M -> 199 M warp instructions per launch (it stays on the 16 B/pt
// memory wall: 389 Gpts/s either way; --kplane 414 -> 423).  The two-step
// kernel keeps the scalar form: packed, its stage B (one warp per SMSP, the
// critical chain) lost more to FFMA2 latency and math-pipe throttling than
// the 9 % fewer instructions gave back (592 vs 601 Gpts/s).
#ifndef FD_PACKED
#define FD_PACKED 1
#endif
constexpr bool kPackedFp32 = FD_PACKED != 0;

// Integer-scaled central second-difference taps (R#2):
// the exact rationals of order 2r multiplied by scale = 1, 12, 180, 5040.
__host__ __device__ constexpr float tap(int R, int m) {
    return R == 1 ? (m == 0 ? -2.f : 1.f)
         : R == 2 ? (m == 0 ? -30.f : m == 1 ? 16.f : -1.f)
         : R == 3 ? (m == 0 ? -490.f : m == 1 ? 270.f : m == 2 ? -27.f : 2.f)
                  : (m == 0 ? -14350.f : m == 1 ? 8064.f : m == 2 ? -1008.f : m == 3 ? 128.f : -9.f);
}
__host__ __device__ constexpr double tap_scale(int R) {
    return R == 1 ? 1.0 : R == 2 ? 12.0 : R == 3 ? 180.0 : 5040.0;
}

// Field buffers carry 2r halo planes on each side of the owned z range (local
// plane z lives at buffer plane z + 2r): r for a single step, 2r for the
// two-steps-per-launch kernel, whose first stage computes P^{k+1} on r planes
// beyond the slab from P^k taps r further out.  K carries r halo planes
// (K plane z at K-halo-buffer plane z + r; see fd_runtime.cu).
__host__ __device__ constexpr int halo_planes(int R) { return 2 * R; }

struct Receivers {
    const int32_t *off;   // CSR offsets per work unit [nunits + 1] (fused kernel)
    const int32_t *z;     // local plane
    const int32_t *y;
    const int32_t *x;
    const int32_t *id;    // column in the step-major trace row
};

// Transport "peer" (FD_OPT_TRANSPORT): a store of local
// plane z of a field buffer also writes the neighbouring slab's halo copy of
// that plane when z is one of its `push` boundary planes -- through NVLink
// (CUDA IPC mapping) across ranks, plain device memory across virtual slabs.
// Our plane z is the lower neighbour's buffer plane lo_z + z (lo_z = its
// nz + 2r) and the upper neighbour's buffer plane z - nz + 2r.
struct PeerPush {
    float *lo, *hi;         // the neighbours' buffer of the same role, or null
    int32_t lo_z, push;
};

struct StepParams {
    int64_t nx, ny, nz;     // local extents (nz = owned planes)
    int64_t pitch;          // floats per row
    int64_t gz0;            // global z of local plane 0
    int64_t nzg;            // global nz (z band)
    int32_t zlo, zhi;       // local planes computed by this launch
    int32_t ntx, nty;       // tiles along x, y
    int32_t nchunks;        // z-chunks of [zlo, zhi)
    int32_t lin;            // tb2d linear mode: units sharing the ntx * nb blocks (0: chunked)
    float *pnext;           // base of the p_prev buffer (overwritten in place); TB2: the C buffer
    float *pnext2;          // TB2 only: the D buffer (P^{k+2})
    const float *p;         // base of the p buffer (naive kernel, register-streamed 2D kernel)
    const float *pm;        // base of the p_prev buffer (register-streamed 2D kernel)
    const float *K;         // K base (naive kernel only)
    // step index: k, or *kdev + koff when replayed from a CUDA graph
    int64_t k;
    const int64_t *kdev;
    int32_t koff;
    // eager source injection of w_{k+1}
    int32_t nsrc;
    int32_t sz[kMaxSources], sy[kMaxSources], sx[kMaxSources];   // local coords (sz may be outside)
    const float *wtab;      // w_j of source s at wtab[j * nsrc + s] (fp64 Ricker, rounded once)
    float *src_raw;         // [nsrc] raw p_next before the s-th injection
    // receivers
    Receivers rec;
    int32_t nrec_local;     // receivers of this launch's list (naive gather)
    float *traces;          // step-major [k][nrec_total]
    int32_t nrec_total;
    PeerPush peer1, peer2;  // in-kernel halo pushes of pnext / pnext2 (boundary launches)
    const float *gsp;       // sponge frame (R#18): g_x[nx], g_y[ny], g_z[nzg] (global z); null = off
    const float *kz;        // FD_OPT_KPLANE: K of local plane z at kz[z] (z in [-r, nz + r)); the KZ
                            // kernel variants read it instead of the K field
    unsigned long long *ws; // rs2d work stealing: one word per warp of the launch (null: static split)
    int32_t nws;            // words (warps) in ws
};

// Per-plane K (FD_OPT_KPLANE): when K depends on the
// slow axis only (layered models), the KZ variants take K of plane z from a
// table of the same fp32 values instead of streaming the K field -- 12 B
// instead of 16 B per single-step update, bitwise the same result.
__device__ __forceinline__ float kplane(const StepParams &p, int z) { return __ldg(p.kz + z); }
__device__ __forceinline__ float4 splat4(float v) { return make_float4(v, v, v, v); }

// Absorbing sponge frame (fd_set_sponge; reading R#18, Cerjan 1985).  The
// per-axis factors come from the fp32 tables g_x, g_y, g_z (global z); indices
// are clamped into the grid (two-step stage A also evaluates ring points
// outside it, whose values are never used).  Canonical fp32 order:
//   G = g_z * (g_y * g_x),   P^{k+1} = G * fma(K, S, fma(2, p, -(G * p_prev)))
// With G = 1 this is bitwise the canonical fma(K, S, fma(2, p, -p_prev)).  The
// tiled kernels hold a thread's g_x (its 4 x points) and g_y (its rows) in
// registers and load g_z once per plane.
__device__ __forceinline__ float sponge_axis(const StepParams &p, int off, int n, int i) {
    return __ldg(p.gsp + off + min(max(i, 0), n - 1));
}
__device__ __forceinline__ float sponge_gx(const StepParams &p, int x) { return sponge_axis(p, 0, (int)p.nx, x); }
__device__ __forceinline__ float sponge_gy(const StepParams &p, int y) {
    return sponge_axis(p, (int)p.nx, (int)p.ny, y);
}
__device__ __forceinline__ float sponge_gz(const StepParams &p, int gz) {
    return sponge_axis(p, (int)(p.nx + p.ny), (int)p.nzg, gz);
}
// SP: the kernel instantiation with the frame (the tiled kernels are compiled
// both ways so the band-rule path carries no sponge code); the reference
// kernels test p.gsp at run time (time_update_rt).
template <bool SP>
__device__ __forceinline__ float time_update(float K, float S, float pc, float pp, float gz, float gy, float gx) {
    if constexpr (!SP) {
        return __fmaf_rn(K, S, __fmaf_rn(2.f, pc, -pp));
    } else {
        const float G = __fmul_rn(gz, __fmul_rn(gy, gx));
        return __fmul_rn(G, __fmaf_rn(K, S, __fmaf_rn(2.f, pc, -__fmul_rn(G, pp))));
    }
}
__device__ __forceinline__ float time_update_rt(const StepParams &p, float K, float S, float pc, float pp, int gz,
                                                int y, int x) {
    if (!p.gsp) return time_update<false>(K, S, pc, pp, 1.f, 1.f, 1.f);
    return time_update<true>(K, S, pc, pp, sponge_gz(p, gz), sponge_gy(p, y), sponge_gx(p, x));
}

// `off` = offset of the float4 within its plane (y * pitch + x), `plane` = ny * pitch
// True when plane z of this slab is one of the planes pushed to a neighbour.
// The tiled kernels take PEER as a template parameter: only boundary launches
// of the peer transport run the PEER = true instantiation, so the push code
// costs the other launches nothing.
__device__ __forceinline__ bool peer_plane(const PeerPush &pp, int z, int nz) {
    return (pp.lo && z < pp.push) || (pp.hi && z >= nz - pp.push);
}

template <int R>
__device__ __forceinline__ void peer_store4(const PeerPush &pp, int z, int nz, int64_t plane, int64_t off,
                                            const float4 &v) {
#ifdef FD_NO_PEER
    return;
#endif
    if (pp.lo && z < pp.push) *reinterpret_cast<float4 *>(pp.lo + (int64_t)(z + pp.lo_z) * plane + off) = v;
    if (pp.hi && z >= nz - pp.push)
        *reinterpret_cast<float4 *>(pp.hi + (int64_t)(z - nz + halo_planes(R)) * plane + off) = v;
}

__device__ __forceinline__ int64_t step_index(const StepParams &p) { return p.kdev ? *p.kdev + p.koff : p.k; }
__device__ __forceinline__ float *trace_row_of(const StepParams &p, int64_t k) {
    return p.traces ? p.traces + k * p.nrec_total : nullptr;
}
__device__ __forceinline__ const float *w_next_of(const StepParams &p, int64_t k) {
    return p.wtab + (k + 1) * p.nsrc;   // w_{k+1}
}

// Position in an N-slot mbarrier ring: slot and phase parity of a counter
// advanced by one per plane (instead of a division per use).
template <int N>
struct RingPos {
    int slot = 0;
    uint32_t par = 0;
    __device__ __forceinline__ void next() {
        if (++slot == N) { slot = 0; par ^= 1u; }
    }
};

// compile-time loop: f(std::integral_constant<int, B>) ... f(<E-1>)
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// ------------------------------------------------------------------ PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Wait for the phase with the given parity to complete.  try_wait with a
// suspend-time hint parks the waiting warp in the barrier unit instead of
// re-issuing try_wait/branch in a loop (measured: the spin loop was ~30 % of
// the issued instructions of the two-step kernel, profiles/ncu_r03).
#ifndef FD_MBAR_SUSPEND_NS
#define FD_MBAR_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#if FD_MBAR_SUSPEND_NS > 0
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra LAB_WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(FD_MBAR_SUSPEND_NS)
        : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra LAB_WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}
// The TMA producer's wait for a free ring slot: FD_PRODUCER_BACKOFF_NS > 0
// sleeps between polls (the producer lane's polling shares its sub-partition's
// issue slots with consumer warps; ncu r2h: 6.8 % of tb2d's instructions).
#ifndef FD_PRODUCER_BACKOFF_NS
#define FD_PRODUCER_BACKOFF_NS 0
#endif
__device__ __forceinline__ void mbar_wait_producer(uint64_t *bar, uint32_t parity) {
#if FD_PRODUCER_BACKOFF_NS > 0
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(FD_PRODUCER_BACKOFF_NS);
    }
#else
    mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y,
                                            int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ float4 lds128(const float *p) { return *reinterpret_cast<const float4 *>(p); }

// Programmatic dependent launch (r2, FD_PDL): a step kernel launched with the
// programmatic-serialization attribute may start while the previous step
// kernel of the stream drains; everything before this point (barrier init,
// tensor-map prefetch) overlaps that tail, everything after it (every read
// of the fields the previous launch wrote, every write of the buffers it
// reads) waits for the previous grid's completion and memory flush.  The
// trigger lets the next launch be scheduled once every CTA of this one has
// started.  Without the attribute griddepcontrol.wait returns at once.
__device__ __forceinline__ void pdl_sync() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ float f4(const float4 &v, int e) {
    return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}
__device__ __forceinline__ void f4set(float4 &v, int e, float s) {
    if (e == 0) v.x = s; else if (e == 1) v.y = s; else if (e == 2) v.z = s; else v.w = s;
}

// ------------------------------------------------------------ packed FP32 (sm_100)
// Blackwell issues two fp32 operations per instruction (FFMA2 / FADD2 /
// FMUL2, PTX fma/add/mul.rn.f32x2) at the scalar rate in flops
// (scripts/ffma2_probe.cu: 73.8 vs 72.2 Tflop/s), i.e. half the issue slots.
// Each lane is the same round-to-nearest operation on the same operands as
// the scalar instruction, so the packed evaluation is bitwise the canonical
// per-point expression.  Pairs are (e, e+1) of a thread's 4 x points: the y
// and z taps and K / p_prev come from float4 registers as aligned pairs;
// x taps at odd distance straddle two float4s and are summed per lane.
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 up2(u64 v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// pair (e0, e0+1) of a float4, e0 in {0, 2}
__device__ __forceinline__ u64 pr2(const float4 &v, int e0) { return e0 == 0 ? pk2(v.x, v.y) : pk2(v.z, v.w); }
// fma(tap_m, s, acc) per lane; a unit tap is an exact add (as the scalar
// compiler emits for __fmaf_rn(1, s, acc))
template <int R, int M>
__device__ __forceinline__ u64 tapfma2(u64 s, u64 acc) {
    constexpr float t = tap(R, M);
    if constexpr (t == 1.0f) return add2(s, acc);
    else return fma2(pk2(t, t), s, acc);
}

// One row of a thread: the canonical expression (band rule, no sponge) for
// its 4 x points, packed.  a = the x row (L4 | M4 | R4, centre M4); yn(o) /
// zn(o) = the float4 of the y / z neighbour at signed offset o; inx per x
// point, iny / inz per row / plane; k4, pp4 = K and p_prev.
template <int R, bool HASY, class YN, class ZN>
__device__ __forceinline__ float4 stencil_row4(const float (&a)[12], YN yn, ZN zn, const bool (&inx)[4], bool iny,
                                               bool inz, const float4 &k4, const float4 &pp4) {
    constexpr float c0 = tap(R, 0);
    float res[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int e0 = 2 * h;
        const u64 c0pc = mul2(pk2(c0, c0), pk2(a[4 + e0], a[5 + e0]));
        u64 sx = c0pc;
        static_for<1, R + 1>([&](auto mm) {
            constexpr int m = decltype(mm)::value;
            u64 sum;
            if constexpr ((m & 1) == 0) sum = add2(pk2(a[4 + e0 - m], a[5 + e0 - m]), pk2(a[4 + e0 + m], a[5 + e0 + m]));
            else sum = pk2(__fadd_rn(a[4 + e0 - m], a[4 + e0 + m]), __fadd_rn(a[5 + e0 - m], a[5 + e0 + m]));
            sx = tapfma2<R, m>(sum, sx);
        });
        const float2 sxf = up2(sx);
        u64 S = pk2(inx[e0] ? sxf.x : 0.f, inx[e0 + 1] ? sxf.y : 0.f);
        if constexpr (HASY) {
            u64 sy = c0pc;
            static_for<1, R + 1>([&](auto mm) {
                constexpr int m = decltype(mm)::value;
                sy = tapfma2<R, m>(add2(pr2(yn(-m), e0), pr2(yn(m), e0)), sy);
            });
            const u64 t = add2(S, sy);
            S = iny ? t : S;
        }
        u64 sz = c0pc;
        static_for<1, R + 1>([&](auto mm) {
            constexpr int m = decltype(mm)::value;
            sz = tapfma2<R, m>(add2(pr2(zn(-m), e0), pr2(zn(m), e0)), sz);
        });
        {
            const u64 t = add2(S, sz);
            S = inz ? t : S;
        }
        const u64 base = pk2(__fmaf_rn(2.f, a[4 + e0], -f4(pp4, e0)), __fmaf_rn(2.f, a[5 + e0], -f4(pp4, e0 + 1)));
        const float2 o = up2(fma2(pr2(k4, e0), S, base));
        res[e0] = o.x;
        res[e0 + 1] = o.y;
    }
    return make_float4(res[0], res[1], res[2], res[3]);
}


// Warp-parallel receiver recording.  The unit's receivers are sorted by z, so
// those with z in [zlo, zhi) form a run starting at rp; 32 of them are matched
// per round (one per lane).  owner(i, lane, yy, e) returns true when receiver
// i's value is register out[yy].e of lane `lane` of THIS warp; the value moves
// by shuffle.  Every lane must call (warp-uniform); returns the index past the
// run.  Replaces a per-thread serial scan whose dependent loads cost ~10 us on
// a 256-receiver row.
// `recx` (optional): also require x in [xlo, xhi) -- a unit that crosses
// columns (tb2d linear mode) holds the next column's receivers of the same
// rows right after this block's.
template <int NY, class Owner>
__device__ __forceinline__ int warp_record(const float4 (&out)[NY], const int32_t *recz, const int32_t *recid,
                                           int rp, int rend, int zlo, int zhi, float *trace_row, Owner owner,
                                           const int32_t *recx = nullptr, int xlo = 0, int xhi = 0) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int i = rp + lane;
        const bool valid = i < rend && recz[i] >= zlo && recz[i] < zhi && (!recx || (recx[i] >= xlo && recx[i] < xhi));
        const unsigned m = __ballot_sync(0xffffffffu, valid);
        if (!m) break;
        int src = lane, yy = 0, e = 0;
        const bool mine = valid && owner(i, src, yy, e);
        float v = 0.f;
#pragma unroll
        for (int q = 0; q < NY; ++q)
#pragma unroll
            for (int ee = 0; ee < 4; ++ee) {
                const float t = __shfl_sync(0xffffffffu, f4(out[q], ee), mine ? src : lane);
                if (q == yy && ee == e) v = t;
            }
        if (mine && trace_row) trace_row[recid[i]] = v;
        const int n = __popc(m);
        rp += n;
        if (n < 32) break;
    }
    return rp;
}

// ------------------------------------------------------------ compile-time config
// TMA boxes are at most 256 elements per dimension and their rows a multiple
// of 16 B: a wide 2D row strip is fetched as `pieces(w)` equal boxes.
constexpr int pieces(int w) {
    for (int n = 1; n <= w; ++n)
        if (w % n == 0 && (w / n) % 4 == 0 && w / n <= 256) return n;
    return -1;
}

template <int R_, int NDIM_, int TX_, int TY_, int NY_, int DP_, int DK_>
struct Cfg {
    static constexpr int R = R_, NDIM = NDIM_, TX = TX_, TY = TY_, NY = NY_, DP = DP_, DK = DK_;
    static constexpr int HY = (NDIM == 3) ? R : 0;                // y halo rows
    static constexpr int BX = TX + 8;                             // x halo: 4-float aligned each side
    static constexpr int BY = TY + 2 * HY;
    static constexpr int NPP = pieces(BX), PBW = BX / NPP;       // p box: (PBW, BY, 1) x NPP
    static constexpr int NTP = pieces(TX), TBW = TX / NTP;       // tile box: (TBW, TY, 1) x NTP
    // TMA writes each box at a 128-B aligned SMEM address: multi-box rows (2D)
    // place box i at i*PPAD floats; pcol() maps a tile column to its SMEM column
    static constexpr int PPAD = (NPP == 1) ? BX : ((PBW + 31) / 32) * 32;
    static constexpr int P_FLOATS = (((NPP == 1 ? BX * BY : NPP * PPAD)) + 31) / 32 * 32;
    __device__ static constexpr int pcol(int c) { return NPP == 1 ? c : (c / PBW) * PPAD + c % PBW; }
    static constexpr int T_FLOATS = TX * TY;
    static constexpr int K_FLOATS = 2 * T_FLOATS;                 // p_prev tile + K tile
    static constexpr uint32_t P_BYTES = BX * BY * 4;
    static constexpr uint32_t T_BYTES = T_FLOATS * 4;
    static constexpr int NSP = R + 1 + DP;                        // p-plane ring
    static constexpr int NSK = DK + 1;                            // (p_prev, K) ring
    static constexpr int NTX = TX / 4, NTY = TY / NY;
    static constexpr int NCONS = NTX * NTY;
    static constexpr int NWC = NCONS / 32;
    static constexpr int NTHREADS = NCONS + 32;                   // + one producer warp
    static constexpr int SMEM_FLOATS = NSP * P_FLOATS + NSK * K_FLOATS;
    static constexpr int SMEM_BYTES = SMEM_FLOATS * 4 + (2 * NSP + 2 * NSK) * 8 + 16;
    static_assert(TX % 4 == 0 && TY % NY == 0, "tile");
    static_assert(NCONS % 32 == 0, "consumer threads must be whole warps");
    static_assert(NPP > 0 && NTP > 0 && BY <= 256 && TY <= 256, "TMA box limit");
    static_assert((NPP == 1 && NTP == 1) || BY == 1, "multi-box rows only for 1-row planes (2D)");
    static_assert(R >= 1 && R <= 4, "r");
};

// ------------------------------------------------------------------ fused kernel
// grid = ntx * nty * nchunks CTAs; CTA b handles tile (b % ntiles) of z-chunk
// (b / ntiles) (chunk-major, so co-resident CTAs stream the same z region and
// share x-y halos in L2).  Warp NWC is the TMA producer; warps 0..NWC-1 compute.
template <class C, bool SP, bool PEER, bool KZ>
__global__ void __launch_bounds__(C::NTHREADS)
fused_step_kernel(const __grid_constant__ CUtensorMap map_p,    // p buffer, box (BX, BY, 1)
                  const __grid_constant__ CUtensorMap map_pp,   // p_prev buffer, box (TX, TY, 1)
                  const __grid_constant__ CUtensorMap map_k,    // K, box (TX, TY, 1)
                  const StepParams prm) {
    constexpr int R = C::R;
    extern __shared__ __align__(128) float smem[];
    float *sP = smem;                                   // NSP * P_FLOATS
    float *sK = smem + C::NSP * C::P_FLOATS;            // NSK * K_FLOATS
    uint64_t *bars = reinterpret_cast<uint64_t *>(sK + C::NSK * C::K_FLOATS);
    uint64_t *fullP = bars, *emptyP = bars + C::NSP;
    uint64_t *fullK = bars + 2 * C::NSP, *emptyK = fullK + C::NSK;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ntiles = prm.ntx * prm.nty;
    const int unit = blockIdx.x;
    const int chunk = unit / ntiles;
    const int tile = unit - chunk * ntiles;
    const int x0 = (tile % prm.ntx) * C::TX;
    const int y0 = (tile / prm.ntx) * C::TY;
    const int span = prm.zhi - prm.zlo;
    const int z0 = prm.zlo + (int)(((int64_t)span * chunk) / prm.nchunks);
    const int z1 = prm.zlo + (int)(((int64_t)span * (chunk + 1)) / prm.nchunks);

    if (tid == 0) {
        for (int i = 0; i < C::NSP; ++i) { mbar_init(&fullP[i], 1); mbar_init(&emptyP[i], C::NWC); }
        for (int i = 0; i < C::NSK; ++i) { mbar_init(&fullK[i], 1); mbar_init(&emptyK[i], C::NWC); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_sync();
    if (z1 <= z0) return;

    // Load l = 0 .. nload-1 brings p plane j = z0 - R + l (buffer plane j + R,
    // halo'd x-y tile) into p slot l % NSP; for l >= 2R it also brings the
    // p_prev and K tiles of plane z = j - R into (p_prev, K) slot (l-2R) % NSK.
    // Slot release (consumers, one arrive per warp):
    //   warm-up / tail planes (j < z0 or j >= z1): right after the column read;
    //   planes z in [z0, z1): after their update at iteration z + R.
    const int nload = (z1 - z0) + 2 * R;
    if (warp == C::NWC) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            tma_prefetch_desc(&map_p); tma_prefetch_desc(&map_pp); tma_prefetch_desc(&map_k);
            for (int l = 0; l < nload; ++l) {
                const int j = z0 - R + l;
                const int s = l % C::NSP;
                mbar_wait_producer(&emptyP[s], ((l / C::NSP) & 1) ^ 1);
                mbar_expect_tx(&fullP[s], C::P_BYTES);
#pragma unroll
                for (int pc = 0; pc < C::NPP; ++pc)
                    tma_load_3d(sP + s * C::P_FLOATS + pc * C::PPAD, &map_p, &fullP[s], x0 - 4 + pc * C::PBW,
                                y0 - C::HY, j + halo_planes(R));
                if (l >= 2 * R) {
                    const int z = j - R, kl = l - 2 * R, ks = kl % C::NSK;
                    mbar_wait_producer(&emptyK[ks], ((kl / C::NSK) & 1) ^ 1);
                    mbar_expect_tx(&fullK[ks], (KZ ? 1 : 2) * C::T_BYTES);
                    float *dst = sK + ks * C::K_FLOATS;
#pragma unroll
                    for (int pc = 0; pc < C::NTP; ++pc) {
                        tma_load_3d(dst + pc * C::TBW, &map_pp, &fullK[ks], x0 + pc * C::TBW, y0, z + halo_planes(R));
                        if constexpr (!KZ)
                            tma_load_3d(dst + C::T_FLOATS + pc * C::TBW, &map_k, &fullK[ks], x0 + pc * C::TBW, y0, z);
                    }
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int tx = tid % C::NTX, ty = tid / C::NTX;
    const int xb = x0 + 4 * tx;                   // first of this thread's 4 x points
    const int yb = y0 + ty * C::NY;               // first of its NY rows
    const int nx = (int)prm.nx, ny = (int)prm.ny;   // 32-bit index math (dims <= 2^30)
    const int cL = C::pcol(4 * tx), cM = C::pcol(4 * tx + 4), cR = C::pcol(4 * tx + 8);
    const int pitch = (int)prm.pitch;
    const int64_t pstride = (int64_t)ny * prm.pitch;   // floats per buffer plane
    const int roff = yb * pitch + xb;             // this thread's first row within a plane
    uint32_t vmask = 0;                           // rows inside the grid
#pragma unroll
    for (int yy = 0; yy < C::NY; ++yy)
        if (yb + yy < ny) vmask |= 1u << yy;

    bool inx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) inx[e] = (xb + e >= R) && (xb + e < nx - R);
    bool iny[C::NY];
#pragma unroll
    for (int yy = 0; yy < C::NY; ++yy) iny[yy] = (C::NDIM == 3) && (yb + yy >= R) && (yb + yy < ny - R);
    float sgx[4], sgy[C::NY];                     // sponge factors (SP only)
#pragma unroll
    for (int e = 0; e < 4; ++e) sgx[e] = SP ? sponge_gx(prm, xb + e) : 1.f;
#pragma unroll
    for (int yy = 0; yy < C::NY; ++yy) sgy[yy] = SP ? sponge_gy(prm, yb + yy) : 1.f;

    // sources that fall in this CTA's tile and chunk
    uint32_t smask = 0;
    for (int s = 0; s < prm.nsrc; ++s)
        if (prm.sx[s] >= x0 && prm.sx[s] < x0 + C::TX && prm.sy[s] >= y0 && prm.sy[s] < y0 + C::TY &&
            prm.sz[s] >= z0 && prm.sz[s] < z1)
            smask |= 1u << s;
    int rp = prm.rec.off ? prm.rec.off[unit] : 0;
    const int rend = prm.rec.off ? prm.rec.off[unit + 1] : 0;
    int rnext_z = (rp < rend) ? prm.rec.z[rp] : INT32_MAX;

    const int64_t kk = step_index(prm);
    float *const trace_row = trace_row_of(prm, kk);
    const float *const wn = w_next_of(prm, kk);

    // z-tap queue: r <= 2 rotates over Q = 2r+1 entries; r >= 3 keeps
    // Q + kQShift - 1 entries and shifts by kQShift every kQShift planes
    constexpr int QU = (2 * R + 1 <= 5) ? 1 : kQShift;
    constexpr int QN = (QU == 1) ? 2 * R + 1 : 2 * R + QU;
    float4 q[QN][C::NY];
#pragma unroll
    for (int i = 0; i < QN; ++i)
#pragma unroll
        for (int yy = 0; yy < C::NY; ++yy) q[i][yy] = make_float4(0.f, 0.f, 0.f, 0.f);

    constexpr float c0 = tap(R, 0);
    constexpr int Q = 2 * R + 1;
    // queue entry of logical position i (plane j - 2r + i) at phase ph
    auto qslot = [](int ph, int i) constexpr { return QU == 1 ? (ph + i) % Q : ph + i; };
    RingPos<C::NSP> pl;                 // p load l (full wait)
    RingPos<C::NSP> pz{C::NSP - R, 0u}; // p load l - r (plane z: x-y taps)
    RingPos<C::NSK> pk;                 // (p_prev, K) plane kl = l - 2r

    // One plane of the stream.  For r <= 2 the register queue rotates instead
    // of shifting: at phase PH (= l mod Q, a compile-time constant) the logical
    // queue entry i (plane j - 2r + i) lives in q[(PH + i) % Q], so no register
    // moves are spent per plane (a shift costs 2r MOVs per point).
    auto plane = [&](const int l, auto ph) {
        constexpr int PH = decltype(ph)::value;
        const int j = z0 - R + l;
        const int s = pl.slot;
        mbar_wait(&fullP[s], pl.par);
        const float *tp = sP + s * C::P_FLOATS;
        // append this thread's column of plane j (logical entry 2r)
#pragma unroll
        for (int yy = 0; yy < C::NY; ++yy)
            q[qslot(PH, 2 * R)][yy] = lds128(tp + (ty * C::NY + yy + C::HY) * C::BX + cM);
        if (j < z0 || j >= z1) {               // z-taps only: slot free now
            __syncwarp();
            if (lane == 0) mbar_arrive(&emptyP[s]);
        }
        pl.next();
        if (l < 2 * R) { pz.next(); return; }

        const int z = j - R;                       // plane computed now
        const int sz_ = pz.slot;                   // its p tile (x-y taps)
        pz.next();
        const float *tz = sP + sz_ * C::P_FLOATS;
        const int ks = pk.slot;
        mbar_wait(&fullK[ks], pk.par);
        pk.next();
        const float *tk = sK + ks * C::K_FLOATS;
        const int gz = (int)prm.gz0 + z;
        const bool inz = (gz >= R) && (gz < (int)prm.nzg - R);
        [[maybe_unused]] const float sgz = SP ? sponge_gz(prm, gz) : 1.f;
        const float kzv = KZ ? kplane(prm, z) : 0.f;

        float4 col[C::NY + 2 * C::HY];
        if (C::NDIM == 3) {
#pragma unroll
            for (int i = 0; i < C::NY + 2 * C::HY; ++i)
                col[i] = lds128(tz + (ty * C::NY + i) * C::BX + cM);
        }
        float4 out[C::NY];
#pragma unroll
        for (int yy = 0; yy < C::NY; ++yy) {
            const float *row = tz + (ty * C::NY + yy + C::HY) * C::BX;
            const float4 L4 = lds128(row + cL), M4 = q[qslot(PH, R)][yy], R4 = lds128(row + cR);
            const float a[12] = {L4.x, L4.y, L4.z, L4.w, M4.x, M4.y, M4.z, M4.w,
                                 R4.x, R4.y, R4.z, R4.w};
            const float4 pp4 = lds128(tk + (ty * C::NY + yy) * C::TX + 4 * tx);
            const float4 kk4 = KZ ? splat4(kzv) : lds128(tk + C::T_FLOATS + (ty * C::NY + yy) * C::TX + 4 * tx);
            if constexpr (!SP && kPackedFp32) {
                out[yy] = stencil_row4<R, C::NDIM == 3>(
                    a, [&](int o) { return col[yy + C::HY + o]; }, [&](int o) { return q[qslot(PH, R + o)][yy]; }, inx,
                    iny[yy], inz, kk4, pp4);
            } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float pc = a[4 + e];
                float sx = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m)
                    sx = __fmaf_rn(tap(R, m), __fadd_rn(a[4 + e - m], a[4 + e + m]), sx);
                float S = inx[e] ? sx : 0.f;
                if (C::NDIM == 3) {
                    float sy = __fmul_rn(c0, pc);
#pragma unroll
                    for (int m = 1; m <= R; ++m)
                        sy = __fmaf_rn(tap(R, m),
                                       __fadd_rn(f4(col[yy + C::HY - m], e), f4(col[yy + C::HY + m], e)), sy);
                    S = iny[yy] ? __fadd_rn(S, sy) : S;
                }
                float szz = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m)
                    szz = __fmaf_rn(tap(R, m),
                                    __fadd_rn(f4(q[qslot(PH, R - m)][yy], e), f4(q[qslot(PH, R + m)][yy], e)), szz);
                S = inz ? __fadd_rn(S, szz) : S;
                const float upd = time_update<SP>(f4(kk4, e), S, pc, f4(pp4, e), sgz, sgy[yy], sgx[e]);
                f4set(out[yy], e, upd);
            }
            }
        }
        // release the (p_prev, K) slot and the p slot of plane z (x-y taps done)
        __syncwarp();
        if (lane == 0) { mbar_arrive(&emptyK[ks]); mbar_arrive(&emptyP[sz_]); }

        // receivers (raw P^{k+1}) -- before the injection
        if (rnext_z == z) {
            rp = warp_record<C::NY>(out, prm.rec.z, prm.rec.id, rp, rend, z, z + 1, trace_row,
                                    [&](int i, int &ln, int &yy, int &e) {
                                        const int dy = prm.rec.y[i] - y0, dx = prm.rec.x[i] - x0;
                                        const int t = (dy / C::NY) * C::NTX + dx / 4;
                                        if ((t >> 5) != warp) return false;
                                        ln = t & 31; yy = dy % C::NY; e = dx & 3;
                                        return true;
                                    });
            rnext_z = (rp < rend) ? prm.rec.z[rp] : INT32_MAX;
        }
        // eager injection of w_{k+1} (registration order)
        if (smask) {
            for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                if (!((smask >> s2) & 1u) || prm.sz[s2] != z) continue;
                const int dy = prm.sy[s2] - yb, dx = prm.sx[s2] - xb;
                if (dy >= 0 && dy < C::NY && dx >= 0 && dx < 4) {
#pragma unroll
                    for (int yy = 0; yy < C::NY; ++yy)
                        if (yy == dy) {
                            const float v = f4(out[yy], dx);
                            prm.src_raw[s2] = v;
                            f4set(out[yy], dx, __fadd_rn(v, wn[s2]));
                        }
                }
            }
        }
        // store p_next in place of p_prev (float4; rows outside the grid skipped)
        if (xb < pitch) {
            float *dst = prm.pnext + (int64_t)(z + halo_planes(R)) * pstride + roff;
#pragma unroll
            for (int yy = 0; yy < C::NY; ++yy)
                if ((vmask >> yy) & 1u) *reinterpret_cast<float4 *>(dst + yy * pitch) = out[yy];
            if (PEER && peer_plane(prm.peer1, z, (int)prm.nz)) {
#pragma unroll
                for (int yy = 0; yy < C::NY; ++yy)
                    if ((vmask >> yy) & 1u)
                        peer_store4<R>(prm.peer1, z, (int)prm.nz, pstride, (int64_t)(roff + yy * pitch), out[yy]);
            }
        }
    };
    if constexpr (Q <= 5) {
        // r <= 2: rotate (Q copies of the plane body)
        for (int l0 = 0; l0 < nload; l0 += Q)
            static_for<0, Q>([&](auto ph) {
                if (l0 + decltype(ph)::value < nload) plane(l0 + decltype(ph)::value, ph);
            });
    } else {
        // r >= 3: full rotation needs 7-9 body copies, which cost more in
        // instruction cache than the 2r moves per point they save (measured: C3
        // order 8 379 -> 359 Gpts/s).  Instead kQShift body copies run on a
        // queue of 2r + kQShift entries (phase PH uses entries PH .. PH + 2r),
        // then the queue shifts by kQShift: 2r moves per kQShift planes.
        for (int l0 = 0; l0 < nload; l0 += QU) {
            static_for<0, QU>([&](auto ph) {
                if (l0 + decltype(ph)::value < nload) plane(l0 + decltype(ph)::value, ph);
            });
#pragma unroll
            for (int i = 0; i < 2 * R; ++i)
#pragma unroll
                for (int yy = 0; yy < C::NY; ++yy) q[i][yy] = q[i + QU][yy];
        }
    }
}

// ------------------------------------------------------------------ 2D tile kernel
// 2D grids (nz, nx): each CTA owns a column of TX x-points and a z-chunk of
// row blocks; it streams TY-row blocks down z.  Each block is ONE TMA box of
// (TX+8) x (TY+2r) p values (z halo rows included, re-read from L2) plus the
// p_prev and K blocks, through an NS-slot mbarrier ring.  x taps and z taps
// both come from SMEM (no register queue), in the canonical order: x term,
// then z term (the 2D z axis plays the role of the 3D y axis of the tile).
template <int R_, int TX_, int TY_, int NY_, int NS_>
struct Cfg2 {
    static constexpr int R = R_, TX = TX_, TY = TY_, NY = NY_, NS = NS_;
    static constexpr int NDIM = 2;
    static constexpr int BX = TX + 8, BZ = TY + 2 * R;
    static constexpr int P_FLOATS = (BX * BZ + 31) / 32 * 32;
    static constexpr int T_FLOATS = TX * TY;
    static constexpr int STAGE = P_FLOATS + 2 * T_FLOATS;
    static constexpr uint32_t STAGE_BYTES = (BX * BZ + 2 * T_FLOATS) * 4;
    static constexpr int NTX = TX / 4, NTY = TY / NY;
    static constexpr int NCONS = NTX * NTY, NWC = NCONS / 32, NTHREADS = NCONS + 32;
    static constexpr int SMEM_BYTES = NS * STAGE * 4 + 2 * NS * 8 + 16;
    // box shapes for the host (x, y, z): p (BX, 1, BZ), tiles (TX, 1, TY)
    static constexpr int PBW = BX, TBW = TX, PBZ = BZ, TBZ = TY;
    static_assert(BX <= 256 && BZ <= 256 && TY <= 256, "TMA box limit");
    static_assert(TX % 4 == 0 && TY % NY == 0 && NCONS % 32 == 0, "tile");
};

template <class C, bool SP, bool PEER, bool KZ>
__global__ void __launch_bounds__(C::NTHREADS)
tile2d_step_kernel(const __grid_constant__ CUtensorMap map_p,    // p buffer, box (BX, 1, BZ)
                   const __grid_constant__ CUtensorMap map_pp,   // p_prev buffer, box (TX, 1, TY)
                   const __grid_constant__ CUtensorMap map_k,    // K, box (TX, 1, TY)
                   const StepParams prm) {
    constexpr int R = C::R;
    extern __shared__ __align__(128) float smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::NS * C::STAGE);
    uint64_t *empty = full + C::NS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int unit = blockIdx.x;
    const int chunk = unit / prm.ntx;
    const int x0 = (unit - chunk * prm.ntx) * C::TX;
    const int span = prm.zhi - prm.zlo;
    const int nb = (span + C::TY - 1) / C::TY;
    const int b0 = (int)(((int64_t)nb * chunk) / prm.nchunks);
    const int b1 = (int)(((int64_t)nb * (chunk + 1)) / prm.nchunks);
    if (tid == 0) {
        for (int i = 0; i < C::NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], C::NWC); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_sync();
    if (b1 <= b0) return;
    const int nload = b1 - b0;

    if (warp == C::NWC) {
        if (lane == 0) {
            tma_prefetch_desc(&map_p); tma_prefetch_desc(&map_pp); tma_prefetch_desc(&map_k);
            for (int l = 0; l < nload; ++l) {
                const int s = l % C::NS;
                const int rb = prm.zlo + (b0 + l) * C::TY;          // first local row of the block
                mbar_wait_producer(&empty[s], ((l / C::NS) & 1) ^ 1);
                mbar_expect_tx(&full[s], C::STAGE_BYTES - (KZ ? C::T_FLOATS * 4 : 0));
                float *st = smem + s * C::STAGE;
                tma_load_3d(st, &map_p, &full[s], x0 - 4, 0, rb - R + halo_planes(R));   // rows rb - r ..
                tma_load_3d(st + C::P_FLOATS, &map_pp, &full[s], x0, 0, rb + halo_planes(R));
                if constexpr (!KZ) tma_load_3d(st + C::P_FLOATS + C::T_FLOATS, &map_k, &full[s], x0, 0, rb);
            }
        }
        return;
    }

    const int tx = tid % C::NTX, ty = tid / C::NTX;
    const int xb = x0 + 4 * tx;
    const int nx = (int)prm.nx;
    bool inx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) inx[e] = (xb + e >= R) && (xb + e < nx - R);
    float sgx[4];                                 // sponge factors (SP only)
#pragma unroll
    for (int e = 0; e < 4; ++e) sgx[e] = SP ? sponge_gx(prm, xb + e) : 1.f;
    uint32_t smask = 0;
    const int zc0 = prm.zlo + b0 * C::TY, zc1 = min(prm.zhi, prm.zlo + b1 * C::TY);
    for (int q = 0; q < prm.nsrc; ++q)
        if (prm.sx[q] >= x0 && prm.sx[q] < x0 + C::TX && prm.sz[q] >= zc0 && prm.sz[q] < zc1) smask |= 1u << q;
    int rp = prm.rec.off ? prm.rec.off[unit] : 0;
    const int rend = prm.rec.off ? prm.rec.off[unit + 1] : 0;
    int rnext_z = (rp < rend) ? prm.rec.z[rp] : INT32_MAX;
    constexpr float c0 = tap(R, 0);
    const int64_t kk = step_index(prm);
    float *const trace_row = trace_row_of(prm, kk);
    const float *const wn = w_next_of(prm, kk);

    RingPos<C::NS> pr;
    for (int l = 0; l < nload; ++l) {
        const int s = pr.slot;
        const int rb = prm.zlo + (b0 + l) * C::TY;
        const int zt = rb + ty * C::NY;                   // first row of this thread
        mbar_wait(&full[s], pr.par);
        pr.next();
        const float *tp = smem + s * C::STAGE;
        const float *tk = tp + C::P_FLOATS;
        float4 col[C::NY + 2 * R];
#pragma unroll
        for (int i = 0; i < C::NY + 2 * R; ++i) col[i] = lds128(tp + (ty * C::NY + i) * C::BX + 4 + 4 * tx);
        float4 out[C::NY];
#pragma unroll
        for (int yy = 0; yy < C::NY; ++yy) {
            const float *row = tp + (ty * C::NY + yy + R) * C::BX + 4 * tx;
            const float4 L4 = lds128(row), M4 = col[yy + R], R4 = lds128(row + 8);
            const float a[12] = {L4.x, L4.y, L4.z, L4.w, M4.x, M4.y, M4.z, M4.w, R4.x, R4.y, R4.z, R4.w};
            const float4 pp4 = lds128(tk + (ty * C::NY + yy) * C::TX + 4 * tx);
            const float4 kk4 = KZ ? splat4(kplane(prm, zt + yy))
                                  : lds128(tk + C::T_FLOATS + (ty * C::NY + yy) * C::TX + 4 * tx);
            const int gz = (int)prm.gz0 + zt + yy;
            const bool inz = (gz >= R) && (gz < (int)prm.nzg - R);
            const float sgz = SP ? sponge_gz(prm, gz) : 1.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float pc = a[4 + e];
                float sx = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m) sx = __fmaf_rn(tap(R, m), __fadd_rn(a[4 + e - m], a[4 + e + m]), sx);
                float S = inx[e] ? sx : 0.f;
                float sz = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m)
                    sz = __fmaf_rn(tap(R, m), __fadd_rn(f4(col[yy + R - m], e), f4(col[yy + R + m], e)), sz);
                S = inz ? __fadd_rn(S, sz) : S;
                f4set(out[yy], e, time_update<SP>(f4(kk4, e), S, pc, f4(pp4, e), sgz, 1.f, sgx[e]));
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);

        // receivers in this block (sorted by row), raw values before injection
        if (rnext_z < rb + C::TY) {
            rp = warp_record<C::NY>(out, prm.rec.z, prm.rec.id, rp, rend, rb, rb + C::TY, trace_row,
                                    [&](int i, int &ln, int &yy, int &e) {
                                        const int dz = prm.rec.z[i] - rb, dx = prm.rec.x[i] - x0;
                                        const int t = (dz / C::NY) * C::NTX + dx / 4;
                                        if ((t >> 5) != warp) return false;
                                        ln = t & 31; yy = dz % C::NY; e = dx & 3;
                                        return true;
                                    });
            rnext_z = (rp < rend) ? prm.rec.z[rp] : INT32_MAX;
        }
        if (smask) {
            for (int q = 0; q < prm.nsrc; ++q) {
                if (!((smask >> q) & 1u)) continue;
                const int dz = prm.sz[q] - zt, dx = prm.sx[q] - xb;
                if (dz >= 0 && dz < C::NY && dx >= 0 && dx < 4) {
#pragma unroll
                    for (int yy = 0; yy < C::NY; ++yy)
                        if (yy == dz) {
                            const float v = f4(out[yy], dx);
                            prm.src_raw[q] = v;
                            f4set(out[yy], dx, __fadd_rn(v, wn[q]));
                        }
                }
            }
        }
        if (xb < (int)prm.pitch) {
            float *dst = prm.pnext + (int64_t)(zt + halo_planes(R)) * prm.pitch + xb;
#pragma unroll
            for (int yy = 0; yy < C::NY; ++yy)
                if (zt + yy < prm.zhi) *reinterpret_cast<float4 *>(dst + (int64_t)yy * prm.pitch) = out[yy];
            if (PEER) {
#pragma unroll
                for (int yy = 0; yy < C::NY; ++yy)
                    if (zt + yy < prm.zhi) peer_store4<R>(prm.peer1, zt + yy, (int)prm.nz, prm.pitch, xb, out[yy]);
            }
        }
    }
}

// ------------------------------------------------------------------ naive kernels (B8)
// One thread per point, global loads, the same canonical expression.  Debug /
// reference path: three launches per step (stencil, receiver gather, injection).
template <int R, int NDIM>
__global__ void naive_step_kernel(const StepParams prm) {
    const int64_t nx = prm.nx, ny = prm.ny, P = prm.pitch;
    const int64_t npl = nx * ny;
    const int64_t total = npl * (prm.zhi - prm.zlo);
    constexpr float c0 = tap(R, 0);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = prm.zlo + t / npl;
        const int64_t rem = t % npl;
        const int64_t y = rem / nx, x = rem % nx;
        const int64_t i = ((z + halo_planes(R)) * ny + y) * P + x;     // index in a field buffer
        const float pc = prm.p[i];
        const int64_t gz = prm.gz0 + z;
        float S = 0.f;
        {
            float s = __fmul_rn(c0, pc);
            if (x >= R && x < nx - R) {
#pragma unroll
                for (int m = 1; m <= R; ++m) s = __fmaf_rn(tap(R, m), __fadd_rn(prm.p[i - m], prm.p[i + m]), s);
                S = s;
            }
        }
        if (NDIM == 3 && y >= R && y < ny - R) {
            float s = __fmul_rn(c0, pc);
#pragma unroll
            for (int m = 1; m <= R; ++m)
                s = __fmaf_rn(tap(R, m), __fadd_rn(prm.p[i - m * P], prm.p[i + m * P]), s);
            S = __fadd_rn(S, s);
        }
        if (gz >= R && gz < prm.nzg - R) {
            const int64_t pz = ny * P;
            float s = __fmul_rn(c0, pc);
#pragma unroll
            for (int m = 1; m <= R; ++m)
                s = __fmaf_rn(tap(R, m), __fadd_rn(prm.p[i - m * pz], prm.p[i + m * pz]), s);
            S = __fadd_rn(S, s);
        }
        const int64_t ik = (z * ny + y) * P + x;
        prm.pnext[i] = time_update_rt(prm, prm.K[ik], S, pc, prm.pnext[i], (int)gz, (int)y, (int)x);
    }
}

// ------------------------------------------------------------ unfused (paper's) decomposition
// Listing 3's routines as separate kernels (the Fig. 5
// experiment): fd_pzz / [fd_pyy] / fd_pxx each write one derivative field
// (band = 0), fd_time combines them.  The derivative fields hold the
// integer-tap sums (the 1/(scale h^2) lives in K), so
//   S = (Pxx + Pyy) + Pzz  and  p_next = fma(K, S, fma(2, p, -p_prev))
// equals the fused kernel's canonical expression (a band term contributes an
// exact +0).  Fields are pitched like K (no halo planes).
// Launch geometry (r2): a 2D/3D grid of 32 x 8 threads, each thread a quad of
// 4 consecutive x points of one row (float4 loads and stores, coalesced), no
// index division; blocks run plane by plane (blockIdx.z = z in 3D), so the
// z taps of neighbouring planes hit in L2.  3D: grid (ceil(nx/128),
// ceil(ny/8), nz); 2D: grid (ceil(nx/128), ceil(nz/8), 1).  Roofline: 8 B per
// point for a derivative kernel (read p, write the field), 28 B (3D) / 24 B
// (2D) for fd_time.
struct QuadPos {
    int x, y, z;
    bool ok;
};
template <int NDIM>
__device__ __forceinline__ QuadPos quad_pos(const StepParams &prm) {
    QuadPos q;
    q.x = (blockIdx.x * 32 + threadIdx.x) * 4;
    if (NDIM == 3) { q.y = blockIdx.y * 8 + threadIdx.y; q.z = blockIdx.z; }
    else { q.y = 0; q.z = blockIdx.y * 8 + threadIdx.y; }
    q.ok = q.x < (int)prm.nx && q.y < (int)prm.ny && q.z < prm.nz;
    return q;
}
// store the in-grid elements of a quad (the pitch padding is never written)
__device__ __forceinline__ void st_quad(float *dst, const float4 v, int x, int nx) {
    if (x + 3 < nx) { *reinterpret_cast<float4 *>(dst) = v; return; }
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (x + e < nx) dst[e] = f4(v, e);
}

template <int R, int AXIS, int NDIM>   // AXIS 0 = x, 1 = y, 2 = z
__global__ void __launch_bounds__(256) d2_axis_kernel(const StepParams prm, float *__restrict__ out) {
    const QuadPos q = quad_pos<NDIM>(prm);
    if (!q.ok) return;
    const int nx = (int)prm.nx, ny = (int)prm.ny;
    const int64_t P = prm.pitch;
    const int64_t i = ((int64_t)(q.z + halo_planes(R)) * ny + q.y) * P + q.x;   // field buffer index
    const float *p = prm.p;
    constexpr float c0 = tap(R, 0);
    const float4 M = lds128(p + i);       // generic float4 load (global)
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (AXIS == 0) {
        const float4 L = lds128(p + i - 4), Rt = lds128(p + i + 4);
        const float a[12] = {L.x, L.y, L.z, L.w, M.x, M.y, M.z, M.w, Rt.x, Rt.y, Rt.z, Rt.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float d = __fmul_rn(c0, a[4 + e]);
#pragma unroll
            for (int m = 1; m <= R; ++m) d = __fmaf_rn(tap(R, m), __fadd_rn(a[4 + e - m], a[4 + e + m]), d);
            f4set(v, e, (q.x + e >= R && q.x + e < nx - R) ? d : 0.f);
        }
    } else {
        const int64_t st = AXIS == 1 ? P : (int64_t)ny * P;
        const int ia = AXIS == 1 ? q.y : (int)prm.gz0 + q.z;
        const int na = AXIS == 1 ? ny : (int)prm.nzg;
        if (ia >= R && ia < na - R) {
            float4 lo[R], hi[R];
#pragma unroll
            for (int m = 1; m <= R; ++m) { lo[m - 1] = lds128(p + i - m * st); hi[m - 1] = lds128(p + i + m * st); }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float d = __fmul_rn(c0, f4(M, e));
#pragma unroll
                for (int m = 1; m <= R; ++m) d = __fmaf_rn(tap(R, m), __fadd_rn(f4(lo[m - 1], e), f4(hi[m - 1], e)), d);
                f4set(v, e, d);
            }
        }
    }
    st_quad(out + ((int64_t)q.z * ny + q.y) * P + q.x, v, q.x, nx);
}

// fd_pzz / fd_pyy (axes with a row or plane stride): each warp owns 128
// consecutive x points (a quad per lane) at one row/plane of the other axis and
// streams ZB points along the derivative's axis with a register window of 2r+1
// float4, so every input row/plane is loaded once per warp plus 2r halo loads
// per ZB outputs (the one-point-per-thread form re-read 2r+1 rows/planes per
// output from L2: 59-62 % of the roof at order 8, profiles/fig5_r2c.md).
// Same arithmetic order as d2_axis_kernel (bitwise).  Grids:
//   3D z: (ceil(nx/128), ceil(ny/8), ceil(nz/ZB))   warp -> y
//   3D y: (ceil(nx/128), ceil(ny/ZB), ceil(nz/8))   warp -> z
//   2D z: (ceil(nx/1024), ceil(nz/ZB), 1)           warp -> 128-point x segment
template <int R, int AXIS, int NDIM, int ZB>
__global__ void __launch_bounds__(256) d2_stream_kernel(const StepParams prm, float *__restrict__ out) {
    static_assert(AXIS == 1 || AXIS == 2, "strided axes");
    const int lane = threadIdx.x, w = threadIdx.y;
    const int nx = (int)prm.nx, ny = (int)prm.ny, nz = (int)prm.nz;
    const int64_t P = prm.pitch;
    constexpr int H = halo_planes(R);
    int x, a0, n;
    int64_t b0, st, o0, ost;
    if constexpr (NDIM == 2) {
        x = (blockIdx.x * 8 + w) * 128 + 4 * lane;
        a0 = blockIdx.y * ZB; n = nz;
        b0 = (int64_t)H * P + x; st = P; o0 = x; ost = P;
    } else if constexpr (AXIS == 2) {
        x = blockIdx.x * 128 + 4 * lane;
        const int y = blockIdx.y * 8 + w;
        if (y >= ny) return;
        a0 = blockIdx.z * ZB; n = nz;
        b0 = ((int64_t)H * ny + y) * P + x; st = (int64_t)ny * P; o0 = (int64_t)y * P + x; ost = st;
    } else {
        x = blockIdx.x * 128 + 4 * lane;
        const int z = blockIdx.z * 8 + w;
        if (z >= nz) return;
        a0 = blockIdx.y * ZB; n = ny;
        b0 = (int64_t)(z + H) * ny * P + x; st = P; o0 = (int64_t)z * ny * P + x; ost = P;
    }
    if (x >= nx || a0 >= n) return;
    const int ia0 = AXIS == 2 ? (int)prm.gz0 : 0, na = AXIS == 2 ? (int)prm.nzg : ny;
    const float *p = prm.p + b0;
    constexpr float c0 = tap(R, 0);
    float4 q[2 * R + 1];
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) q[j] = lds128(p + (int64_t)(a0 - R + j) * st);
#pragma unroll
    for (int t = 0; t < ZB; ++t) {
        const int a = a0 + t;
        if (a >= n) break;
        q[2 * R] = lds128(p + (int64_t)(a + R) * st);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ia0 + a >= R && ia0 + a < na - R) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float d = __fmul_rn(c0, f4(q[R], e));
#pragma unroll
                for (int m = 1; m <= R; ++m) d = __fmaf_rn(tap(R, m), __fadd_rn(f4(q[R - m], e), f4(q[R + m], e)), d);
                f4set(v, e, d);
            }
        }
        st_quad(out + o0 + (int64_t)a * ost, v, x, nx);
#pragma unroll
        for (int j = 0; j < 2 * R; ++j) q[j] = q[j + 1];
    }
}

template <int R, int NDIM>
__global__ void __launch_bounds__(256) time_update_kernel(const StepParams prm, const float *__restrict__ pxx,
                                                          const float *__restrict__ pyy,
                                                          const float *__restrict__ pzz) {
    const QuadPos q = quad_pos<NDIM>(prm);
    if (!q.ok) return;
    const int nx = (int)prm.nx, ny = (int)prm.ny;
    const int64_t P = prm.pitch;
    const int64_t ik = ((int64_t)q.z * ny + q.y) * P + q.x;
    const int64_t i = ((int64_t)(q.z + halo_planes(R)) * ny + q.y) * P + q.x;
    const float4 dx = lds128(pxx + ik), dz = lds128(pzz + ik), k4 = lds128(prm.K + ik);
    const float4 dy = NDIM == 3 ? lds128(pyy + ik) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 pc = lds128(prm.p + i), pp = lds128(prm.pnext + i);
    float4 o;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float S = f4(dx, e);
        if (NDIM == 3) S = __fadd_rn(S, f4(dy, e));
        S = __fadd_rn(S, f4(dz, e));
        f4set(o, e, time_update_rt(prm, f4(k4, e), S, f4(pc, e), f4(pp, e), (int)prm.gz0 + q.z, q.y, q.x + e));
    }
    st_quad(prm.pnext + i, o, q.x, nx);
}

// receivers of the naive path: trace_row[id] = p_next at (z, y, x) (raw, before injection)
template <int R>
__global__ void gather_receivers_kernel(const StepParams prm) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= prm.nrec_local) return;
    const int64_t i = ((int64_t)(prm.rec.z[j] + halo_planes(R)) * prm.ny + prm.rec.y[j]) * prm.pitch + prm.rec.x[j];
    trace_row_of(prm, step_index(prm))[prm.rec.id[j]] = prm.pnext[i];
}

// K = fl32((v dt / h)^2 / scale) in fp64 (R#7), in place over the uploaded
// velocities of a pitched buffer; explicit _rn intrinsics, so the result is
// bitwise the host formula ((double)v * dt / h, squared, / scale, rounded once).
// It also validates the model on the device (fd_create): the max velocity as
// float bits (v > 0, so the bit patterns order like the values) for the CFL
// check of R#8, and the smallest host index of an entry that is not finite and
// > 0 (`bad`, initialised to ULLONG_MAX); idx0 = host index of buffer row 0.
static __global__ void velocity_to_K_kernel(float *buf, int64_t rows, int64_t nx, int64_t pitch, double dt, double h,
                                            double scale, int64_t idx0, unsigned *vmax_bits,
                                            unsigned long long *bad) {
    const int64_t total = rows * nx;
    unsigned m = 0;
    unsigned long long b = ~0ull;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = (t / nx) * pitch + t % nx;
        const float v = buf[i];
        if (v > 0.f && v <= 3.402823466e38f) m = max(m, __float_as_uint(v));
        else b = min(b, (unsigned long long)(idx0 + t));
        const double cv = __ddiv_rn(__dmul_rn((double)v, dt), h);
        buf[i] = __double2float_rn(__ddiv_rn(__dmul_rn(cv, cv), scale));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        b = min(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (m) atomicMax(vmax_bits, m);
        if (b != ~0ull) atomicMin(bad, b);
    }
}

// graph bookkeeping: the device step counter
// FD_OPT_KPLANE: table[pl] = K of K-halo-buffer plane pl (pl in [0, planes)),
// and *bad |= 1 when any in-grid point of a plane differs from its plane's
// first point (bit comparison; pitch padding excluded).
static __global__ void kplane_table_kernel(const float *Kh, int64_t planes, int64_t ny, int64_t nx, int64_t pitch,
                                           float *table, int *bad) {
    const int64_t n = planes * ny * nx;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pl = i / (ny * nx), rem = i - pl * ny * nx, y = rem / nx, x = rem - y * nx;
        const float *plane = Kh + pl * ny * pitch;
        const float ref = plane[0];
        if (__float_as_uint(plane[y * pitch + x]) != __float_as_uint(ref)) atomicOr(bad, 1);
        if (rem == 0) table[pl] = ref;
    }
}

// fd_get_traces: step-major device traces [k][nrec] -> receiver-major
// [nrec][k] through 32 x 32 shared-memory tiles (both sides coalesced); rows
// of receivers this context does not own (own[j] == 0) are written as 0.
static __global__ void traces_transpose_kernel(const float *in, float *out, int64_t nrec, int64_t k,
                                               const unsigned char *own) {
    __shared__ float tile[32][33];
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    for (int64_t k0 = (int64_t)blockIdx.y * 32; k0 < k; k0 += (int64_t)gridDim.y * 32) {
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int64_t kk = k0 + r, j = j0 + threadIdx.x;
            tile[r][threadIdx.x] = (kk < k && j < nrec) ? in[kk * nrec + j] : 0.f;
        }
        __syncthreads();
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int64_t j = j0 + r, kk = k0 + threadIdx.x;
            if (j < nrec && kk < k) out[j * k + kk] = own[j] ? tile[threadIdx.x][r] : 0.f;
        }
        __syncthreads();
    }
}

static __global__ void set_step_kernel(int64_t *kdev, int64_t k) { *kdev = k; }

// Peer transport flag sync (fd_runtime.cu peer_signal / peer_wait): the
// neighbours' flags count completed halo exchanges.  The signal runs after the
// pushing launches in stream order; the system-scope fence and release store
// publish their peer stores before the count.
static __global__ void peer_signal_kernel(int64_t *lo, int64_t *hi, int64_t v) {
    __threadfence_system();
    if (lo) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(lo), "l"(v) : "memory");
    if (hi) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(hi), "l"(v) : "memory");
}
// Spins until both neighbours have signalled exchange v.  Bounded: after
// timeout_ns (%globaltimer) it raises *err (mapped host memory; fd_step polls it
// and poisons the context) and returns, so a neighbour that died does not hang
// the stream forever; once *err is set every later wait returns at once.
static __global__ void peer_wait_kernel(const int64_t *flags, int need_lo, int need_hi, int64_t v,
                                        volatile int *err, uint64_t timeout_ns) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        int64_t a = v, b = v;
        if (need_lo) asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(a) : "l"(flags) : "memory");
        if (need_hi) asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(b) : "l"(flags + 1) : "memory");
        if (a >= v && b >= v) break;
        if (*err) return;
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) {
            *err = 1;
            __threadfence_system();
            return;
        }
        __nanosleep(200);
    }
}
static __global__ void advance_step_kernel(int64_t *kdev, int64_t n) { *kdev += n; }

// add_source on a field buffer, registration order; records the raw values.
// field = buffer base; sources with sz outside [0, nz) are skipped (other slab).
template <int R>
__global__ void inject_kernel(float *field, const StepParams prm) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const float *wn = w_next_of(prm, step_index(prm));
    for (int s = 0; s < prm.nsrc; ++s) {
        if (prm.sz[s] < 0 || prm.sz[s] >= prm.nz) continue;
        const int64_t i = ((int64_t)(prm.sz[s] + halo_planes(R)) * prm.ny + prm.sy[s]) * prm.pitch + prm.sx[s];
        const float v = field[i];
        prm.src_raw[s] = v;
        field[i] = __fadd_rn(v, wn[s]);
    }
}

}  // namespace fdk
