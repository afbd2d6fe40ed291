// fd_rs2d.cuh -- S time steps per pass on 2D grids, streamed through registers
// (temporal blocking).
//
// In 2D a "plane" of the 2.5D scheme is one row, so the x taps of a row are
// neighbouring lanes' registers and the z taps a per-thread register queue:
// no stage tile in shared memory, no producer warp, no mbarriers between
// stages.  One warp streams a column strip down z: lane l holds the quad
// x = x0 - 4 HQ + 4 l .. + 3 of every time level, 32 quads = 128 columns of
// which the middle TX = 4 (32 - 2 HQ) are its own (the HQ halo quads on each
// side are recomputed by the neighbouring strips: 4 HQ >= S r keeps the own
// quads exact after S steps).  Per row i the warp loads P^k(i), P^{k-1}(i - r),
// K(i - r) into a per-warp shared-memory ring Q rows ahead (cp.async 16-B
// copies, each lane its own quads; or, CfgRS2::TMA, three bulk tensor copies
// by one lane) and evaluates Listing 3's run() body S times,
// stage J (1..S) on row i - J r:
//   P^{k+J} = fma(K, S(P^{k+J-1}), fma(2, P^{k+J-1}, -P^{k+J-2}))
// with the eager injection of w_{k+J}; x taps by warp shuffle, z taps from
// the level-(J-1) queue (2r + 1 rows), P^{k+J-2} from the level-(J-2) queue
// (its oldest row) or, for J = 1, the P^{k-1} load.  Stages S-1 and S store
// the own quads of the run's rows to the C (P^{k+S-1}) and D (P^{k+S})
// buffers; every stage records its receivers (raw values).  Each stage
// evaluates the canonical per-point expression (fd_kernels.cuh), so a pass is
// bitwise S single steps.
//
// HBM per pass: read P^k, P^{k-1}, K, write two levels: 20 B per point for S
// updates.  Work: a persistent grid whose warps take equal row pieces of the
// column strips, then balance by work stealing (rs2d_step_kernel).
//
// Rows outside the buffers (the warm-up rows at the grid faces, the ring's
// run-out) are zero-filled and never stored; rows outside the grid never
// reach a grid row (band rule, R#3: rows r..nz-r-1 are the only ones reading
// z taps).  Halos on z-slabs: S = 2 reads 2r planes of P^k and r of P^{k-1}
// and K beyond the slab (the halo planes the runtime exchanges); S >= 3 runs
// on single-slab contexts only.
#pragma once
#include <cstdio>

#include "fd_kernels.cuh"

// Work stealing granularity defaults of CfgRS2 (A/B switches): claims of
// FD_RS_CHK * U rows; a thief cuts a word with at least FD_RS_STEALMIN
// claims' worth unclaimed
#ifndef FD_RS_CHK
#define FD_RS_CHK 2
#endif
#ifndef FD_RS_STEALMIN
#define FD_RS_STEALMIN 2
#endif

namespace fdk {

// R, S; HQ halo quads per side; W warps per CTA; Q rows in flight per warp
// (shared-memory ring); MINB CTAs per SM.
template <int R_, int S_, int HQ_, int W_, int Q_, int MINB_ = 1, bool TMA_ = true, int CHK_ = FD_RS_CHK,
          int SMIN_ = FD_RS_STEALMIN>
struct CfgRS2 {
    static constexpr int R = R_, S = S_, HQ = HQ_, W = W_, Q = Q_, MINB = MINB_;
    // work stealing: claims of CHK * U rows; a thief cuts a word with at
    // least SMIN claims' worth unclaimed (r3 A/B on C2: order 2 S = 4 best at
    // 1 / 2 -- 751 vs 722 Gpts/s at 2 / 2 --, order 4 S = 3 at 2 / 1: 641 vs 628)
    static constexpr int CHK = CHK_, SMIN = SMIN_;
    // TMA: one lane loads each row's three 512 B pieces with bulk tensor copies
    // (cp.async.bulk.tensor, out-of-grid zero fill, one mbarrier per ring
    // slot); else every lane copies its own 16 B with cp.async (LDGSTS)
    static constexpr bool TMA = TMA_;
    static constexpr int TX = 4 * (32 - 2 * HQ);          // own columns per strip
    static constexpr int NTHREADS = 32 * W;
    static constexpr int SMEM_BYTES = W * Q * 3 * 32 * 16 + W * Q * 8;   // ring + mbarriers
    static constexpr int KQ = (S - 1) * R + 1;             // K rows i - S r .. i - r
    // the K queue rounded up to a multiple of the z queues' period 2r + 1; U
    // rows per unrolled loop body = that length (no register moves)
    static constexpr int KQL = (KQ + 2 * R) / (2 * R + 1) * (2 * R + 1);
    static constexpr int U = KQL;
    static constexpr int CH = CHK * U;                     // rows per work-stealing claim
    static_assert(4 * HQ >= S * R, "the halo quads must cover S r columns");
    static_assert(S >= 2 && R >= 1 && R <= 4 && Q >= 2 && Q <= 16, "config");
};

// 16-byte asynchronous global -> shared copy (LDGSTS, L2 only); ok = false
// copies nothing and zero-fills
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Cold paths, out of line (the unrolled row loop holds S U copies of the
// stage body; keeping these out of it keeps the kernel in the instruction cache).
// Receivers of row z with x in this strip: run from rp (sorted by z), 64 per
// round (each lane loads z, x, id of two entries at once: one load latency
// per round -- a receiver line puts 120 entries of one row in every strip),
// the value of register o.e of the owning lane (lane = (x - xq0) / 4) moved by
// shuffle.  Advances rp; returns the next receiver's row (or 0x7fffffff past
// zb).  Warp-uniform call.
static __device__ __noinline__ int rs_record(float4 o, int z, int zb, int &rp, int rend, int xq0, const Receivers &rec,
                                      float *trow) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int zz[2], xx[2], id[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int ii = rp + 32 * h + lane;
            const bool in = ii < rend;
            zz[h] = in ? rec.z[ii] : 0x7fffffff;
            xx[h] = in ? rec.x[ii] : xq0;
            id[h] = in ? rec.id[ii] : 0;
        }
        int n = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool valid = zz[h] == z;
            const unsigned m = __ballot_sync(0xffffffffu, valid);
            const int dx = xx[h] - xq0;
            const int src = valid ? dx >> 2 : lane, e = dx & 3;
            const float v0 = __shfl_sync(0xffffffffu, o.x, src), v1 = __shfl_sync(0xffffffffu, o.y, src);
            const float v2 = __shfl_sync(0xffffffffu, o.z, src), v3 = __shfl_sync(0xffffffffu, o.w, src);
            if (valid && trow) trow[id[h]] = e == 0 ? v0 : (e == 1 ? v1 : (e == 2 ? v2 : v3));
            n += __popc(m);
        }
        rp += n;
        if (n < 64) break;
    }
    return (rp < rend && rec.z[rp] < zb) ? rec.z[rp] : 0x7fffffff;
}
// First index >= rp of the sorted z[] with z >= bound (or rend).  Two load
// latencies for up to 1024 entries: 32 samples at a stride, then the
// stride-long segment (a serial scan of a receiver line's 120 entries per strip
// cost ~60 k cycles of dependent loads).  Warp-uniform call.
__device__ __forceinline__ int warp_lower_bound(const int32_t *z, int rp, int rend, int bound) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int n = rend - rp;
        if (n <= 0) return rp;
        const int step = n <= 32 ? 1 : (n + 31) / 32;
        const int ii = rp + lane * step;
        const unsigned m = __ballot_sync(0xffffffffu, ii < rend && z[ii] < bound);
        const int c = __popc(m);                       // samples below bound (a prefix)
        if (step == 1) return rp + c;
        if (c == 0) return rp;
        rp += (c - 1) * step + 1;                      // sample c-1 is below: search after it
        rend = min(rend, rp - 1 + step);               // sample c (if any) is not
    }
}
// Eager injection of w at the sources of this lane's quad on row z, in
// registration order; `raw`: also store the pre-injection value (src_raw).
static __device__ __noinline__ float4 rs_inject(float4 o, int z, uint32_t smask, int xb, bool raw, const StepParams &prm,
                                         const float *wv) {
    for (int s2 = 0; s2 < prm.nsrc; ++s2) {
        if (!((smask >> s2) & 1u) || prm.sz[s2] != z) continue;
        const int dx = prm.sx[s2] - xb;
        const float vraw = f4(o, dx);
        if (raw) prm.src_raw[s2] = vraw;
        f4set(o, dx, __fadd_rn(vraw, wv[s2]));
    }
    return o;
}

// Predicated 16-byte global store without a branch (the row loop stays one
// basic block, so the compiler can overlap the stages of a row).  The
// buffers stored to are never read by the same launch: no ordering needed.
__device__ __forceinline__ void stg4_if(void *p, const float4 &v, bool ok) {
    asm volatile(
        "{\n"
        ".reg .pred q;\n"
        "setp.ne.u32 q, %5, 0;\n"
        "@q st.global.v4.f32 [%0], {%1, %2, %3, %4};\n"
        "}\n" ::"l"(p),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"((unsigned)ok));
}

// One run of a warp: output rows [za, c1) of work unit `unit`, c1 extended
// chunk by chunk while `more` (work stealing: the warp claims CH-row chunks
// from its own word of the region's work-stealing array, a thief may cut its
// end; see rs2d_step_kernel).  Rows outside the run are computed (warm-up, the
// chunk look-ahead) but never stored nor recorded.
template <class C, bool SP, bool PEER, bool KZ>
__device__ __forceinline__ int rs2d_run(const StepParams &prm, const CUtensorMap *mp, const CUtensorMap *mm,
                                        const CUtensorMap *mk, float4 *const rs_ring, uint64_t *const wbar,
                                        uint32_t *const parity_io, const int unit, const int za, int c1, bool more,
                                        unsigned long long *const myword) {
    constexpr int R = C::R, S = C::S, HQ = C::HQ, Q = C::Q, U = C::U, KQL = C::KQL, CH = C::CH;
    constexpr int H = halo_planes(R);
    constexpr unsigned FULL = 0xffffffffu;
    constexpr float c0 = tap(R, 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int colu = unit % prm.ntx;
    const int chunk = unit / prm.ntx;
    const int span = prm.zhi - prm.zlo;
    const int u1 = prm.zlo + (int)(((int64_t)span * (chunk + 1)) / prm.nchunks);   // end of the unit's rows
    const int nx = (int)prm.nx, pitch = (int)prm.pitch, nzl = (int)prm.nz;
    const int x0 = colu * C::TX, xb = x0 - 4 * HQ + 4 * lane;
    const bool xok = xb >= 0 && xb < pitch;                         // quad inside the row
    const bool own = lane >= HQ && lane < 32 - HQ && xb < pitch;   // stored by this strip
    // band rule in x as a bit mask (S = [x in] s_x is s_x & mask: the same +0.f
    // as the select, without a predicate register per point)
    uint32_t mkx[4];
    float sgx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t m = ((xb + e >= R) && (xb + e < nx - R)) ? 0xffffffffu : 0u;
        asm volatile("mov.b32 %0, %1;" : "=r"(mkx[e]) : "r"(m));   // opaque: kept, not re-derived
        sgx[e] = SP ? sponge_gx(prm, xb + e) : 1.f;
    }
    uint32_t smask = 0;                                // sources in this lane's quad
    for (int s2 = 0; s2 < prm.nsrc; ++s2)
        if (prm.sx[s2] >= xb && prm.sx[s2] < xb + 4) smask |= 1u << s2;
    const bool anysrc = __any_sync(FULL, smask != 0);
    const int64_t kk = step_index(prm);

    // addresses: buffer row (u32) x row bytes (u32) + column base (one IMAD.WIDE.U32);
    // fields hold local rows -H .. nz + H - 1 at buffer rows 0 .. nz + 2H - 1,
    // K rows -r .. nz + r - 1 at K-halo rows 0 .. nz + 2r - 1
    const int xo = xok ? xb : 0;
    const uint32_t rowB = (uint32_t)pitch * 4u;
    const char *const bP = reinterpret_cast<const char *>(prm.p + xo);
    const char *const bM = reinterpret_cast<const char *>(prm.pm + xo);
    const char *const bK = reinterpret_cast<const char *>(prm.K - (int64_t)R * pitch + xo);   // K halo row 0
    char *const bC = reinterpret_cast<char *>(prm.pnext + xb);
    char *const bD = reinterpret_cast<char *>(prm.pnext2 + xb);

    // receivers of the unit (sorted by z, x inside the strip): per stage the
    // next one and its row (0x7fffffff past the warp's rows)
    const int rbeg = prm.rec.off ? prm.rec.off[unit] : 0;
    const int rend = prm.rec.off ? prm.rec.off[unit + 1] : 0;
    const int rp0 = warp_lower_bound(prm.rec.z, rbeg, rend, za);
    const int nz0 = (rp0 < rend && prm.rec.z[rp0] < u1) ? prm.rec.z[rp0] : 0x7fffffff;
    int rpJ[S], nzJ[S];
#pragma unroll
    for (int j = 0; j < S; ++j) { rpJ[j] = rp0; nzJ[j] = nz0; }
    // Rows of events -- a receiver to record, a source to inject -- run the
    // general loop body, every other block of U rows the branch-free one (a
    // warp with receivers or a source would otherwise run every row with the
    // calls' branches and finish last).  Block [ib, ib + U) covers stage rows
    // [ib - S r, ib + U - r).  Sources: the rows of those inside the strip's
    // 128 columns (an interval: conservative for several sources).
    int src_lo = 0x7fffffff, src_hi = -0x7fffffff;
    for (int s2 = 0; s2 < prm.nsrc; ++s2)
        if (prm.sx[s2] >= x0 - 4 * HQ && prm.sx[s2] < x0 - 4 * HQ + 128) {
            src_lo = min(src_lo, prm.sz[s2]);
            src_hi = max(src_hi, prm.sz[s2]);
        }
    int rq = rp0;                                     // first receiver not yet passed by every stage
    int rz_next = rq < rend ? prm.rec.z[rq] : 0x7fffffff;

    float4 P[S][2 * R + 1];      // level j = P^{k+j}: rows newest - 2r .. newest
    float4 kq[KQL];              // K rows i - KQL r .. i - r (stage J reads row i - J r)
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
        for (int t = 0; t < 2 * R + 1; ++t) P[j][t] = zero4;
#pragma unroll
    for (int t = 0; t < KQL; ++t) kq[t] = zero4;

    // per-warp ring of Q rows in shared memory: slot q holds [P^k | P^{k-1} |
    // K] of one row, 32 lanes x 16 B each (TMA: lane 0 loads the three row
    // pieces; cp.async: every lane copies its own quads); each lane reads back
    // only its own quads
    float4 *const wr = rs_ring + warp * (Q * 3 * 32) + lane;
    const uint32_t wr_s = smem_u32(wr);
    uint32_t bpar = *parity_io;                       // TMA: phase parity bit per slot (kept across runs)
    // rows past the run's last iteration (the ring's run-out) copy nothing
    const int i0 = za - S * R;                        // P^k row of the first iteration
    auto issue_row = [&](int i, int slot) {
        const int iend = c1 + S * R + (more ? Q : 0);
        if constexpr (C::TMA) {
            // out-of-grid rows and columns are zero-filled by the tensor maps
            // (fields: buffer rows 0 .. nz + 2H - 1; K: halo rows 0 .. nz + 2r - 1)
            __syncwarp();                             // every lane has read the slot
            if (lane == 0) {
                if (i < iend) {
                    float *const d = reinterpret_cast<float *>(rs_ring + warp * (Q * 3 * 32) + slot * (3 * 32));
                    mbar_expect_tx(wbar + slot, KZ ? 1024u : 1536u);
                    tma_load_3d(d, mp, wbar + slot, x0 - 4 * HQ, 0, i + H);
                    tma_load_3d(d + 128, mm, wbar + slot, x0 - 4 * HQ, 0, i - R + H);
                    if constexpr (!KZ) tma_load_3d(d + 256, mk, wbar + slot, x0 - 4 * HQ, 0, i);
                } else {
                    mbar_arrive(wbar + slot);         // nothing to load: complete the phase
                }
            }
            return;
        }
        const uint32_t zp = (uint32_t)min(max(i + H, 0), nzl + 2 * H - 1);
        const uint32_t zm = (uint32_t)min(max(i - R + H, 0), nzl + 2 * H - 1);
        const uint32_t d = wr_s + (uint32_t)slot * (3 * 32 * 16);
        const bool ok = xok && i < iend;
        cp_async16(d, bP + (uint64_t)zp * rowB, ok);
        cp_async16(d + 512, bM + (uint64_t)zm * rowB, ok);
        if constexpr (!KZ) {
            const uint32_t zk = (uint32_t)min(max(i, 0), nzl + 2 * R - 1);   // K row i - r
            cp_async16(d + 1024, bK + (uint64_t)zk * rowB, ok);
        }
        cp_async_commit();
    };

    // one row: iteration i reads P^k(i), P^{k-1}(i - r), K(i - r) and runs
    // stage J on row i - J r, J = 1..S
    auto row = [&](int i, int &slot, auto fastc) {
        constexpr bool FAST = decltype(fastc)::value;
        if constexpr (C::TMA) {
            mbar_wait(wbar + slot, (bpar >> slot) & 1u);   // row i has landed
            bpar ^= 1u << slot;
        } else {
            cp_async_wait<Q - 1>();                   // row i has landed
        }
        const float4 *const rw = wr + slot * (3 * 32);
        const float4 nP = rw[0], nM = rw[32];
#pragma unroll
        for (int t = 0; t < 2 * R; ++t) P[0][t] = P[0][t + 1];
        P[0][2 * R] = nP;
        if constexpr (!KZ) {
#pragma unroll
            for (int t = 0; t < KQL - 1; ++t) kq[t] = kq[t + 1];
            kq[KQL - 1] = rw[64];
        }
        static_for<1, S + 1>([&](auto JJ) {
            constexpr int J = decltype(JJ)::value;
            const int z = i - J * R;                  // row of stage J
            const float4 M4 = P[J - 1][R];
            float av[12];
            av[4] = M4.x; av[5] = M4.y; av[6] = M4.z; av[7] = M4.w;
#pragma unroll
            for (int m = 1; m <= R; ++m) {
                av[4 - m] = __shfl_up_sync(FULL, f4(M4, 4 - m), 1);
                av[7 + m] = __shfl_down_sync(FULL, f4(M4, m - 1), 1);
            }
            const float4 pm4 = J == 1 ? nM : P[J >= 2 ? J - 2 : 0][0];
            const float4 k4 = KZ ? splat4(kplane(prm, z)) : kq[KQL - 1 - (J - 1) * R];
            const int gz = (int)prm.gz0 + z;
            const bool inz = (gz >= R) && (gz < (int)prm.nzg - R);
            const float sgz = SP ? sponge_gz(prm, gz) : 1.f;
            float4 o;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float pc = av[4 + e];
                float sx = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m) sx = __fmaf_rn(tap(R, m), __fadd_rn(av[4 + e - m], av[4 + e + m]), sx);
                float Sv;
                asm("and.b32 %0, %1, %2;" : "=f"(Sv) : "f"(sx), "r"(mkx[e]));
                float szz = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m)
                    szz = __fmaf_rn(tap(R, m), __fadd_rn(f4(P[J - 1][R - m], e), f4(P[J - 1][R + m], e)), szz);
                Sv = inz ? __fadd_rn(Sv, szz) : Sv;
                f4set(o, e, time_update<SP>(f4(k4, e), Sv, pc, f4(pm4, e), sgz, 1.f, sgx[e]));
            }
            if constexpr (!FAST) {
                // receivers of this stage's row (raw P^{k+J}, before the injection)
                if (z == nzJ[J - 1] && z < c1)
                    nzJ[J - 1] = rs_record(o, z, u1, rpJ[J - 1], rend, x0 - 4 * HQ, prm.rec,
                                           trace_row_of(prm, kk + J - 1));
                // w_{k+J} at every computed point (the call only on the strip's
                // source rows: an event block has S U stage rows)
                if (anysrc && z >= src_lo && z <= src_hi)
                    o = rs_inject(o, z, smask, xb, J == S && own && z >= za && z < c1, prm,
                                  w_next_of(prm, kk + J - 1));
            }
            if constexpr (J < S) {
#pragma unroll
                for (int t = 0; t < 2 * R; ++t) P[J][t] = P[J][t + 1];
                P[J][2 * R] = o;
            }
            if constexpr (J >= S - 1) {
                const bool st = own && z >= za && z < c1;
                char *const dst = (J == S ? bD : bC) + (uint64_t)(uint32_t)(z + H) * rowB;
                stg4_if(dst, o, st);
                if constexpr (PEER) {
                    if (st) peer_store4<R>(J == S ? prm.peer2 : prm.peer1, z, nzl, prm.pitch, xb, o);
                }
            }
        });
        // row i's values are consumed: its slot takes row i + Q
        issue_row(i + Q, slot);
        slot = slot + 1 == Q ? 0 : slot + 1;
    };

#pragma unroll
    for (int q = 0; q < Q; ++q) issue_row(i0 + q, q);
    int slot = 0;                                     // ring slot of row i
    unsigned long long claim = 0;                     // lane 0: pending claim (atomicAdd result)
    bool pending = false;
    for (int ib = i0;; ib += U) {
        // chunks: claim the next one a block ahead of need, resolve it when
        // the block's stage-1 rows (the most advanced) reach the claimed end,
        // so no stage computes a row past c1 while more chunks may follow
        // (rows past the final c1 are neither stored nor recorded); the ring
        // loads Q rows past c1 while more (a row issued Q iterations ahead is
        // at most Q - (S-1) r past the c1 of its issue)
        if (more) {
            const bool need = ib + U - 1 - R >= c1;
            if (!pending && (need || ib + 2 * U - 1 - R >= c1)) {
                if (lane == 0) claim = atomicAdd(myword, (unsigned long long)CH);
                pending = true;
            }
            if (need) {
                const unsigned long long w = __shfl_sync(FULL, claim, 0);
                const int nxt = prm.zlo + (int)(w & 0xfffff), end = prm.zlo + (int)((w >> 20) & 0xfffff);
                pending = false;
                if (nxt < end && nxt == c1) {
                    c1 = min(nxt + CH, end);
                    more = nxt + CH < end;
                } else {
                    more = false;
                }
            }
        }
        if (ib - S * R >= c1) break;                  // every stage-S row of the run is done
        const bool ev = PEER || rz_next < ib + U - R || (src_lo < ib + U - R && src_hi >= ib - S * R);
        if (!ev) {
#pragma unroll
            for (int u = 0; u < U; ++u) row(ib + u, slot, std::true_type{});
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) row(ib + u, slot, std::false_type{});
            rq = warp_lower_bound(prm.rec.z, max(rq, rpJ[S - 1]), rend, ib + U - S * R);
            rz_next = rq < rend ? prm.rec.z[rq] : 0x7fffffff;
        }
    }
    if constexpr (C::TMA) {
        // drain: wait for the Q copies in flight (the slots' pending phases)
        for (int q = 0; q < Q; ++q) {
            mbar_wait(wbar + slot, (bpar >> slot) & 1u);
            bpar ^= 1u << slot;
            slot = slot + 1 == Q ? 0 : slot + 1;
        }
        *parity_io = bpar;
    } else {
        cp_async_wait<0>();                           // the ring is idle when the next run starts
    }
    return c1;                                        // the run's end
}

// Work stealing (whole-launch balance).  The per-SM speed of this
// memory-bound kernel differs by up to ~1.7x across the SMs of one B200 and
// is the same launch after launch (r3 timing probe: one wave of equal runs
// ended between 34 and 72 us).  Each warp owns a 64-bit word of the region's
// array: next (claim pointer) | end | unit | epoch (rows relative to zlo).
// The owner claims CH-row chunks with atomicAdd on `next`; a warp that is
// done reads 32 words per round (one per lane), takes the one with the most
// unclaimed rows and cuts its `end` in half with atomicCAS, then runs
// [half, old end) itself (its own word republished, stealable in turn).  A
// single 64-bit word makes claim and cut race-free.  The epoch (launch
// number) keeps a thief off the words of the previous launch.
__device__ __forceinline__ unsigned long long ws_pack(int next, int end, int unit, uint32_t epoch) {
    return (unsigned long long)(uint32_t)next | ((unsigned long long)(uint32_t)end << 20) |
           ((unsigned long long)(uint32_t)unit << 40) | ((unsigned long long)epoch << 54);
}

template <class C, bool SP, bool PEER, bool KZ>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
rs2d_step_kernel(const __grid_constant__ CUtensorMap map_p0,   // P^k buffer, box (128, 1, 1) (TMA mode)
                 const __grid_constant__ CUtensorMap map_pm,   // P^{k-1} buffer, box (128, 1, 1)
                 const __grid_constant__ CUtensorMap map_k,    // K halo buffer, box (128, 1, 1)
                 const __grid_constant__ StepParams prm) {
    constexpr int S = C::S, CH = C::CH;
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    extern __shared__ __align__(128) float4 rs_ring[];
    // TMA mode: Q mbarriers per warp after the rings, initialised by the warp
    uint64_t *const wbar = reinterpret_cast<uint64_t *>(rs_ring + C::W * C::Q * 3 * 32) + warp * C::Q;
    uint32_t bpar = 0;
    if constexpr (C::TMA) {
        if (lane == 0) {
            tma_prefetch_desc(&map_p0); tma_prefetch_desc(&map_pm); tma_prefetch_desc(&map_k);
            for (int q = 0; q < C::Q; ++q) mbar_init(wbar + q, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    // Static assignment: a persistent grid (one wave of resident CTAs, or
    // fewer on small grids) of NW warps; each of the ntx column strips (work
    // units; their receivers are one CSR list each, nchunks = 1) is cut into
    // p = max(1, NW / ntx) equal row pieces, piece q (strip q / p) taken by
    // warp q mod NW; the warps without a piece start as thieves.
    const int span = prm.zhi - prm.zlo;
    const int NW = gridDim.x * C::W;
    const int pp = max(1, NW / prm.ntx), npieces = prm.ntx * pp;
    pdl_sync();
#ifdef FD_RS_CLOCK
    uint64_t clk0, clks = 0;
    int nruns = 0, nrows = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clk0));
#define FD_RS_PROBE(x) x
#else
#define FD_RS_PROBE(x)
#endif
    const int gw = blockIdx.x * C::W + warp;          // this warp's word
    unsigned long long *const ws = prm.ws;
    const uint32_t epoch = (uint32_t)((step_index(prm) / S) & 1023);
    FD_RS_PROBE(int za = -1; int zb = -1; int unit = -1;)
    if (lane == 0 && ws) atomicExch(ws + gw, ws_pack(0, 0, 0, epoch));   // nothing to steal yet
    for (int q = gw; q < npieces; q += NW) {
        const int strip = q / pp, k = q - strip * pp;
        const int a = prm.zlo + (int)(((int64_t)span * k) / pp), b = prm.zlo + (int)(((int64_t)span * (k + 1)) / pp);
        FD_RS_PROBE(if (za < 0) { za = a; zb = b; unit = strip; })
        if (b <= a) continue;
        if (ws) {
            const int c1 = min(a + CH, b);
            if (lane == 0) atomicExch(ws + gw, ws_pack(c1 - prm.zlo, b - prm.zlo, strip, epoch));
            __syncwarp();
            const int e = rs2d_run<C, SP, PEER, KZ>(prm, &map_p0, &map_pm, &map_k, rs_ring, wbar, &bpar, strip, a, c1, c1 < b, ws + gw);
            FD_RS_PROBE(++nruns; nrows += e - a; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clks));)
        } else {
            rs2d_run<C, SP, PEER, KZ>(prm, &map_p0, &map_pm, &map_k, rs_ring, wbar, &bpar, strip, a, b, false, nullptr);
        }
    }
    if (ws) {
        // steal until eight rounds in a row find nothing worth taking
        uint32_t round = 0;
        for (int miss = 0; miss < 8;) {
            const int v = (int)(((uint32_t)gw * 2654435761u + (uint32_t)(++round) * 40503u * 33u +
                                 (uint32_t)lane * 97u) % (uint32_t)prm.nws);
            const unsigned long long w = *reinterpret_cast<volatile unsigned long long *>(ws + v);
            const int nxt = (int)(w & 0xfffff), end = (int)((w >> 20) & 0xfffff);
            const bool cur = (uint32_t)(w >> 54) == epoch && v != gw;
            const int rem = cur ? end - nxt : 0;
            // the lane with the most unclaimed rows (ties: lowest lane)
            int best = rem, bl = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const int ob = __shfl_xor_sync(FULL, best, o), ol = __shfl_xor_sync(FULL, bl, o);
                if (ob > best || (ob == best && ol < bl)) { best = ob; bl = ol; }
            }
            if (best < C::SMIN * CH) { ++miss; continue; }
            int m = 0, oend = 0, vunit = 0;
            if (lane == bl) {
                m = nxt + (end - nxt) / 2;
                const unsigned long long nw = (w & ~(0xfffffull << 20)) | ((unsigned long long)m << 20);
                if (atomicCAS(ws + v, w, nw) == w) {
                    oend = end;
                    vunit = (int)((w >> 40) & 0x3fff);
                } else {
                    m = -1;                            // raced with the owner or another thief
                }
            }
            m = __shfl_sync(FULL, m, bl);
            if (m < 0) continue;
            oend = __shfl_sync(FULL, oend, bl);
            vunit = __shfl_sync(FULL, vunit, bl);
            const int c1 = min(m + CH, oend);
            if (lane == 0) atomicExch(ws + gw, ws_pack(c1, oend, vunit, epoch));
            __syncwarp();
            const int e = rs2d_run<C, SP, PEER, KZ>(prm, &map_p0, &map_pm, &map_k, rs_ring, wbar, &bpar, vunit, prm.zlo + m,
                                                    prm.zlo + c1, c1 < oend, ws + gw);
            FD_RS_PROBE(++nruns; nrows += e - prm.zlo - m;)
            miss = 0;
        }
    }
#ifdef FD_RS_CLOCK
    // timing probe (debug builds): per warp SM, unit, rows and start / end time
    uint64_t clk1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clk1));
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (lane == 0 && step_index(prm) < 4)
        printf("RSCLK %u %d %d %d %d %llu %llu %d %d %llu\n", smid, unit, warp, za, zb, (unsigned long long)clk0,
               (unsigned long long)clk1, nruns, nrows, (unsigned long long)clks);
#endif
#undef FD_RS_PROBE
}

}  // namespace fdk
