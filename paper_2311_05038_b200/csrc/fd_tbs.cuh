// fd_tbs.cuh -- S time steps per pass on 2D grids (temporal blocking of depth
// S >= 3).
//
// The two-step 2D kernel (fd_tb2.cuh, tb2d) moves 20 B per point per launch
// for 2 updates.  Reading P^k, P^{k-1}, K once and writing only the last two
// levels P^{k+S-1}, P^{k+S} (the next pass's P_prev and P) keeps the 20 B per
// launch for S updates: 6.7 B per update at S = 3.  Each of Listing 3's
// run() bodies is one pipeline stage:
//   stage J (0 <= J < S) computes P^{k+J+1} = fma(K, S(P^{k+J}), fma(2, P^{k+J}, -P^{k+J-1}))
//   with the eager injection of w_{k+J+1}, on a row block grown by
//   (S-1-J) r rows on each side (and by 4 columns per side for J < S-1, the
//   quad halo that carries the x taps of the later stages: (S-1) r <= 4);
// stage 0 reads the TMA stage (P^k box with S r halo rows and 8 columns, the
// grown P^{k-1} and K boxes); stage J >= 1 reads stage J-1's block from a
// shared-memory ring (x, z taps) and P^{k+J-1} pointwise (J = 1: the P^k box,
// J >= 2: stage J-2's ring); every stage reads K from the TMA stage.  Stage
// S-2 stores its tile interior to the C buffer (P^{k+S-1}), stage S-1 to D
// (P^{k+S}); receivers are recorded by every stage (trace rows k .. k+S-1).
// Each stage evaluates the canonical per-point expression, so a pass is
// bitwise S single steps.
//
// Validity: stage J's values are exact on its region shrunk by J r columns
// at the x edges of the 4-column quad halo (the taps of the first/last quad
// read outside the ring there); rows are exact over the whole grown block.
// Values outside the valid region are computed but never reach a valid one
// (the region shrinks by r per stage) nor memory.
//
// Warp roles: S groups of stage warps (each thread a quad x NY rows of its
// stage's block) and one TMA producer warp.  Barriers: TMA slots (full: tx
// bytes; empty: every stage's warps -- K is read by all), ring j = output of
// stage j (full: stage j's warps; empty: stage j+1 (taps) and stage j+2
// (pointwise) warps).  Single-slab 2D contexts; band rule, K field (no
// sponge / peer / per-plane-K variants).
#pragma once
#include "fd_tb2.cuh"      // role_release, kArrivalsPerWarp

namespace fdk {

template <int R_, int S_, int TX_, int TY_, int NY_, int NS_, int NR_, int MINB_ = 1>
struct CfgS2 {
    static constexpr int R = R_, S = S_, TX = TX_, TY = TY_, NY = NY_, NS = NS_, NR = NR_, MINB = MINB_;
    static_assert(S >= 2 && (S - 1) * R <= 4, "the 4-column quad halo carries (S-1) r columns");
    static constexpr int BX0 = TX + 16, BXE = TX + 8;
    static constexpr int BYP = TY + 2 * S * R;                 // P^k box rows
    static constexpr int BYA = TY + 2 * (S - 1) * R;           // P^{k-1}, K boxes = stage-0 block rows
    __host__ __device__ static constexpr int BY(int J) { return TY + 2 * (S - 1 - J) * R; }
    __host__ __device__ static constexpr int QX(int J) { return J < S - 1 ? BXE / 4 : TX / 4; }
    __host__ __device__ static constexpr int NT(int J) { return QX(J) * (BY(J) / NY); }
    __host__ __device__ static constexpr int NW(int J) { return (NT(J) + 31) / 32; }
    __host__ __device__ static constexpr int WBASE(int J) { return J == 0 ? 0 : WBASE(J - 1) + NW(J - 1); }
    static constexpr int NWALL = WBASE(S);
    static constexpr int NTHREADS = 32 * (NWALL + 1);
    static constexpr int P0F = (BX0 * BYP + 31) / 32 * 32;
    static constexpr int AF = (BXE * BYA + 31) / 32 * 32;
    static constexpr int STAGE = P0F + 2 * AF;                 // [P^k | P^{k-1} | K]
    static constexpr uint32_t STAGE_BYTES = (BX0 * BYP + 2 * BXE * BYA) * 4;
    static constexpr int RPAD = 8;                             // floats before / after a ring slot
    static constexpr int RF = (BXE * BYA + 2 * RPAD + 31) / 32 * 32;   // ring slot (rows of stage 0, max)
    static constexpr int NRINGS = S - 1;
    static constexpr int NBARS = 2 * NS + 2 * NRINGS * NR;
    static constexpr int SMEM_BYTES = (NS * STAGE + NRINGS * NR * RF) * 4 + NBARS * 8 + 16;
    // TileCfg presentation (fd_tab_tbs.cu)
    static constexpr int NY_REPORT = NY, DP = NS, DA = NR;
    static_assert(BYP <= 256 && BX0 <= 256, "TMA box");
    __host__ __device__ static constexpr bool rows_ok() {
        for (int j = 0; j < S; ++j)
            if (BY(j) % NY) return false;
        return true;
    }
    static_assert(rows_ok(), "every stage's rows must be a multiple of NY");
};

template <class C, bool SP, bool PEER, bool KZ>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
tbs2d_step_kernel(const __grid_constant__ CUtensorMap map_p0,   // P^k buffer, box (BX0, 1, BYP)
                  const __grid_constant__ CUtensorMap map_pm,   // P^{k-1} buffer, box (BXE, 1, BYA)
                  const __grid_constant__ CUtensorMap map_k,    // K halo buffer, box (BXE, 1, BYA)
                  const StepParams prm) {
    static_assert(!SP && !PEER && !KZ, "S-step kernel: band rule, K field, single slab");
    constexpr int R = C::R, S = C::S;
    extern __shared__ __align__(128) float smem[];
    float *sSt = smem;
    float *sRing = smem + C::NS * C::STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sRing + C::NRINGS * C::NR * C::RF);
    uint64_t *fullS = bars, *emptyS = fullS + C::NS;
    uint64_t *fullR = emptyS + C::NS, *emptyR = fullR + C::NRINGS * C::NR;   // [ring][slot]
    const int tid = threadIdx.x, warp = tid >> 5;
    const int unit = blockIdx.x;
    const int span = prm.zhi - prm.zlo;
    const int nb = (span + C::TY - 1) / C::TY;
    int v0, v1;                                       // blocks v = column * nb + row block (as tb2d)
    if (prm.lin > 0) {
        const int64_t V = (int64_t)prm.ntx * nb;
        v0 = (int)(V * unit / prm.lin);
        v1 = (int)(V * (unit + 1) / prm.lin);
    } else {
        const int chunk = unit / prm.ntx, colu = unit - chunk * prm.ntx;
        v0 = colu * nb + (int)(((int64_t)nb * chunk) / prm.nchunks);
        v1 = colu * nb + (int)(((int64_t)nb * (chunk + 1)) / prm.nchunks);
    }
    if (tid == 0) {
        for (int i = 0; i < C::NS; ++i) {
            mbar_init(&fullS[i], 1);
            mbar_init(&emptyS[i], kArrivalsPerWarp * C::NWALL);
        }
        static_for<0, C::NRINGS>([&](auto jj) {
            constexpr int j = decltype(jj)::value;
            constexpr int cons = C::NW(j + 1) + (j + 2 <= S - 1 ? C::NW(j + 2) : 0);
            for (int i = 0; i < C::NR; ++i) {
                mbar_init(&fullR[j * C::NR + i], kArrivalsPerWarp * C::NW(j));
                mbar_init(&emptyR[j * C::NR + i], kArrivalsPerWarp * cons);
            }
        });
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the ring slots' pads are read (never used) by the edge quads: keep them finite
    for (int i = tid; i < C::NRINGS * C::NR * C::RF; i += C::NTHREADS) sRing[i] = 0.f;
    __syncthreads();
    pdl_sync();
    if (v1 <= v0) return;
    const int nload = v1 - v0;
    const int nx = (int)prm.nx;
    const int64_t kk = step_index(prm);
    constexpr float c0 = tap(R, 0);
    const int rbeg = prm.rec.off ? prm.rec.off[unit] : 0;
    const int rend = prm.rec.off ? prm.rec.off[unit + 1] : 0;
    auto rec_block = [&](int i) { return (prm.rec.x[i] / C::TX) * nb + (prm.rec.z[i] - prm.zlo) / C::TY; };

    if (warp == C::NWALL) {
        // ---------------------------------------------------------------- producer
        if ((tid & 31) == 0) {
            tma_prefetch_desc(&map_p0); tma_prefetch_desc(&map_pm); tma_prefetch_desc(&map_k);
            for (int l = 0; l < nload; ++l) {
                const int v = v0 + l, colu = v / nb;
                const int s = l % C::NS, rb = prm.zlo + (v - colu * nb) * C::TY, x0 = colu * C::TX;
                mbar_wait_producer(&emptyS[s], ((l / C::NS) & 1) ^ 1);
                mbar_expect_tx(&fullS[s], C::STAGE_BYTES);
                float *st = sSt + s * C::STAGE;
                // buffer row of local row z is z + 2r; the K halo buffer's is z + r
                tma_load_3d(st, &map_p0, &fullS[s], x0 - 8, 0, rb - S * R + halo_planes(R));
                tma_load_3d(st + C::P0F, &map_pm, &fullS[s], x0 - 4, 0, rb - (S - 1) * R + halo_planes(R));
                tma_load_3d(st + C::P0F + C::AF, &map_k, &fullS[s], x0 - 4, 0, rb - (S - 1) * R + R);
            }
        }
        return;
    }

    // ------------------------------------------------------------------ stages
    static_for<0, S>([&](auto jj) {
        constexpr int J = decltype(jj)::value;
        if (warp < C::WBASE(J) || warp >= C::WBASE(J) + C::NW(J)) return;
        constexpr bool LAST = J == S - 1;
        constexpr int QX = C::QX(J), NY = C::NY, BYJ = C::BY(J);
        constexpr int GR = (S - 1 - J) * R;            // rows of growth on each side
        const int t = tid - 32 * C::WBASE(J);
        const bool act = t < C::NT(J);
        const int q = act ? t % QX : 0, re0 = act ? (t / QX) * NY : 0;
        // x of the quad: grown stages start 4 columns left of the tile
        const int xoff = LAST ? 0 : -4;
        // columns of this quad inside each source array (offset of the quad's first float)
        const int c_p0 = 4 * q + (LAST ? 8 : 4);     // P^k box (starts at x0 - 8)
        const int c_e = 4 * q + (LAST ? 4 : 0);      // grown arrays (start at x0 - 4)
        const bool qint = LAST || (q >= 1 && q <= C::TX / 4);
        int colc = -1, x0 = 0, xb = 0;
        bool inx[4];
        uint32_t smask = 0;
        float *const trow = trace_row_of(prm, kk + J);
        const float *const wv = w_next_of(prm, kk + J);
        int rp = rbeg;
        RingPos<C::NS> ps;
        RingPos<C::NR> pr;
        for (int l = 0; l < nload; ++l) {
            const int v = v0 + l, colu = v / nb;
            const int rb = prm.zlo + (v - colu * nb) * C::TY;
            if (colu != colc) {
                colc = colu;
                x0 = colu * C::TX;
                xb = x0 + xoff + 4 * q;
#pragma unroll
                for (int e = 0; e < 4; ++e) inx[e] = (xb + e >= R) && (xb + e < nx - R);
                smask = 0;
                for (int s2 = 0; s2 < prm.nsrc; ++s2)
                    if (act && prm.sx[s2] >= xb && prm.sx[s2] < xb + 4) smask |= 1u << s2;
            }
            mbar_wait(&fullS[ps.slot], ps.par);
            const float *tp = sSt + ps.slot * C::STAGE, *tpm = tp + C::P0F, *tk = tpm + C::AF;
            // cur = P^{k+J} (x / z taps), prev = P^{k+J-1} (pointwise), rows relative to this stage's row 0
            const float *cur;
            int cur_w, cur_c, cur_r;                  // row pitch, quad column, row offset (= r)
            if constexpr (J == 0) { cur = tp; cur_w = C::BX0; cur_c = c_p0; cur_r = R; }
            else {
                mbar_wait(&fullR[(J - 1) * C::NR + pr.slot], pr.par);
                cur = sRing + ((J - 1) * C::NR + pr.slot) * C::RF + C::RPAD;
                cur_w = C::BXE; cur_c = c_e; cur_r = R;
            }
            const float *prv;
            int prv_w, prv_c, prv_r;
            if constexpr (J == 0) { prv = tpm; prv_w = C::BXE; prv_c = c_e; prv_r = 0; }
            else if constexpr (J == 1) { prv = tp; prv_w = C::BX0; prv_c = c_p0; prv_r = 2 * R; }
            else { prv = sRing + ((J - 2) * C::NR + pr.slot) * C::RF + C::RPAD; prv_w = C::BXE; prv_c = c_e; prv_r = 2 * R; }
            const int krow = J * R;                   // this stage's row 0 inside the K box
            float *outp = nullptr;
            if constexpr (!LAST) {
                mbar_wait(&emptyR[J * C::NR + pr.slot], pr.par ^ 1u);
                outp = sRing + (J * C::NR + pr.slot) * C::RF + C::RPAD;
            }
            float4 out[NY];
            float4 col[NY + 2 * R];
#pragma unroll
            for (int i = 0; i < NY + 2 * R; ++i) col[i] = lds128(cur + (re0 + cur_r - R + i) * cur_w + cur_c);
#pragma unroll
            for (int yy = 0; yy < NY; ++yy) {
                const int re = re0 + yy;
                const float *row = cur + (re + cur_r) * cur_w + cur_c;
                const float4 L4 = lds128(row - 4), M4 = col[yy + R], R4 = lds128(row + 4);
                const float av[12] = {L4.x, L4.y, L4.z, L4.w, M4.x, M4.y, M4.z, M4.w, R4.x, R4.y, R4.z, R4.w};
                const float4 pp4 = lds128(prv + (re + prv_r) * prv_w + prv_c);
                const float4 k4 = lds128(tk + (re + krow) * C::BXE + c_e);
                const int z = rb - GR + re;
                const int gz = (int)prm.gz0 + z;
                const bool inz = (gz >= R) && (gz < (int)prm.nzg - R);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float pc = av[4 + e];
                    float sx = __fmul_rn(c0, pc);
#pragma unroll
                    for (int m = 1; m <= R; ++m) sx = __fmaf_rn(tap(R, m), __fadd_rn(av[4 + e - m], av[4 + e + m]), sx);
                    float Sv = inx[e] ? sx : 0.f;
                    float szz = __fmul_rn(c0, pc);
#pragma unroll
                    for (int m = 1; m <= R; ++m)
                        szz = __fmaf_rn(tap(R, m), __fadd_rn(f4(col[yy + R - m], e), f4(col[yy + R + m], e)), szz);
                    Sv = inz ? __fadd_rn(Sv, szz) : Sv;
                    f4set(out[yy], e, time_update<false>(f4(k4, e), Sv, pc, f4(pp4, e), 1.f, 1.f, 1.f));
                }
            }
            // release what this stage read: the TMA slot (all stages), ring J-1
            // (taps) and ring J-2 (pointwise) -- after the last shared-memory read
            if constexpr (J >= 1) role_release(&emptyR[(J - 1) * C::NR + pr.slot]);
            if constexpr (J >= 2) role_release(&emptyR[(J - 2) * C::NR + pr.slot]);
            role_release(&emptyS[ps.slot]);
            // receivers (raw P^{k+J+1}, tile interior) -- before the injection
            if (rp < rend && rec_block(rp) == v)
                rp = warp_record<NY>(out, prm.rec.z, prm.rec.id, rp, rend, rb, rb + C::TY, trow,
                                     [&](int i, int &ln, int &yy, int &e) {
                                         const int re = prm.rec.z[i] - (rb - GR), dx = prm.rec.x[i] - (x0 + xoff);
                                         const int tt = (re / NY) * QX + dx / 4;
                                         if (C::WBASE(J) + (tt >> 5) != warp) return false;
                                         ln = tt & 31; yy = re % NY; e = dx & 3;
                                         return true;
                                     }, prm.rec.x, x0, x0 + C::TX);
            if (act) {
                if (smask) {                              // w_{k+J+1} wherever in this stage's block
#pragma unroll
                    for (int yy = 0; yy < NY; ++yy) {
                        const int z = rb - GR + re0 + yy;
                        for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                            if (!((smask >> s2) & 1u) || prm.sz[s2] != z) continue;
                            const int dx = prm.sx[s2] - xb;
                            const float vraw = f4(out[yy], dx);
                            if (LAST && z >= rb && z < rb + C::TY && z < prm.zhi) prm.src_raw[s2] = vraw;
                            f4set(out[yy], dx, __fadd_rn(vraw, wv[s2]));
                        }
                    }
                }
                if constexpr (!LAST) {
#pragma unroll
                    for (int yy = 0; yy < NY; ++yy)
                        *reinterpret_cast<float4 *>(outp + (re0 + yy) * C::BXE + c_e) = out[yy];
                }
                // global stores: stage S-2 -> C (P^{k+S-1}), stage S-1 -> D (P^{k+S}); tile interior
                if constexpr (J >= S - 2) {
                    float *dstb = J == S - 1 ? prm.pnext2 : prm.pnext;
                    if (qint && xb < (int)prm.pitch) {
#pragma unroll
                        for (int yy = 0; yy < NY; ++yy) {
                            const int z = rb - GR + re0 + yy;
                            if (z >= rb && z < rb + C::TY && z < prm.zhi)
                                *reinterpret_cast<float4 *>(dstb + (int64_t)(z + halo_planes(R)) * prm.pitch + xb) =
                                    out[yy];
                        }
                    }
                }
            }
            if constexpr (!LAST) role_release(&fullR[J * C::NR + pr.slot]);
            ps.next();
            pr.next();
        }
    });
}

}  // namespace fdk
