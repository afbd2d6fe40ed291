// fd_tb2.cuh -- two time steps per pass (temporal blocking).
//
// One launch performs steps k and k+1 of Listing 3's run() body
// over the 3D grid:
//   stage A: P^{k+1} = fma(K, S(P^k), fma(2, P^k, -P^{k-1})) on the tile grown
//            by r in x and y (the halo the second step needs), plus the eager
//            injection of w_{k+1}; kept in a shared-memory plane ring and
//            written (tile interior) to the C buffer;
//   stage B: P^{k+2} = fma(K, S(P^{k+1}), fma(2, P^{k+1}, -P^k)) on the tile,
//            injection of w_{k+2}, written to the D buffer.
// Both evaluate the canonical per-point expression of fd_kernels.cuh, so a
// pass is bitwise two single steps.  HBM traffic per pair of updates: read
// P^k, P^{k-1}, K once, write P^{k+1}, P^{k+2}: 20 B, i.e. 10 B per update
// instead of 16.  The x-y halo ring of stage A is recomputed by neighbouring
// tiles (redundant compute instead of communication).
//
// Buffers: four field buffers rotate (cur, prev) -> (C, D); none is written
// while another CTA may still read it (P^k and P^{k-1} are read with halos).
// Single-slab contexts only (slabs would need 2r-deep halos).
#pragma once
#include "fd_kernels.cuh"

namespace fdk {

template <int R_, int TX_, int TY_, int NYA_, int NYB_, int DP_, int DA_, int NCONS_>
struct CfgTB {
    static constexpr int R = R_, TX = TX_, TY = TY_, NYA = NYA_, NYB = NYB_, DP = DP_, DA = DA_;
    static constexpr int NCONS = NCONS_, NWC = NCONS / 32, NTHREADS = NCONS + 32;
    // P^k tile: x halo 8 (4-float aligned, covers 2r <= 8), y halo 2r
    static constexpr int BX0 = TX + 16, BY0 = TY + 4 * R;
    // grown tile E (stage A region, P^{k-1}/K/P^{k+1} tiles): x halo 4, y halo r
    static constexpr int BXE = TX + 8, BYE = TY + 2 * R;
    static constexpr int QXE = BXE / 4, QXI = TX / 4;
    static constexpr int P0F = (BX0 * BY0 + 31) / 32 * 32;
    static constexpr int EF = (BXE * BYE + 31) / 32 * 32;
    static constexpr int NSP = 2 * R + 1 + DP;   // P^k planes z1-r .. z1+r (+ prefetch)
    static constexpr int NSA = R + 1 + DA;       // (P^{k-1}, K) planes z1-r .. z1 (+ prefetch)
    static constexpr int NS1 = 2 * R + 2;        // P^{k+1} planes z2-r .. z2+r, +1 (one barrier/plane)
    static constexpr int ITEMS_A = QXE * (BYE / NYA), ITEMS_B = QXI * (TY / NYB);
    static constexpr uint32_t P0_BYTES = BX0 * BY0 * 4, AUX_BYTES = 2 * BXE * BYE * 4;
    static constexpr int SMEM_FLOATS = NSP * P0F + NSA * 2 * EF + NS1 * EF;
    static constexpr int SMEM_BYTES = SMEM_FLOATS * 4 + (2 * NSP + 2 * NSA) * 8 + 16;
    static_assert(BYE % NYA == 0 && TY % NYB == 0 && NCONS % 32 == 0, "tile");
    static_assert(BX0 <= 256 && BY0 <= 256 && R <= 4, "TMA box");
};

__device__ __forceinline__ void consumer_barrier(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <class C>
__global__ void __launch_bounds__(C::NTHREADS)
tb2_step_kernel(const __grid_constant__ CUtensorMap map_p0,   // P^k buffer, box (BX0, BY0, 1)
                const __grid_constant__ CUtensorMap map_pm,   // P^{k-1} buffer, box (BXE, BYE, 1)
                const __grid_constant__ CUtensorMap map_k,    // K, box (BXE, BYE, 1)
                const StepParams prm) {                       // pnext = C, pnext2 = D
    constexpr int R = C::R;
    extern __shared__ __align__(128) float smem[];
    float *sP0 = smem;
    float *sAux = sP0 + C::NSP * C::P0F;       // slot: [P^{k-1} tile | K tile]
    float *sP1 = sAux + C::NSA * 2 * C::EF;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sP1 + C::NS1 * C::EF);
    uint64_t *fullP = bars, *emptyP = bars + C::NSP, *fullA = bars + 2 * C::NSP, *emptyA = fullA + C::NSA;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntiles = prm.ntx * prm.nty;
    const int unit = blockIdx.x;
    const int chunk = unit / ntiles, tile = unit - chunk * ntiles;
    const int x0 = (tile % prm.ntx) * C::TX, y0 = (tile / prm.ntx) * C::TY;
    const int span = prm.zhi - prm.zlo;
    const int z0 = prm.zlo + (int)(((int64_t)span * chunk) / prm.nchunks);
    const int z1e = prm.zlo + (int)(((int64_t)span * (chunk + 1)) / prm.nchunks);
    if (tid == 0) {
        for (int i = 0; i < C::NSP; ++i) { mbar_init(&fullP[i], 1); mbar_init(&emptyP[i], C::NWC); }
        for (int i = 0; i < C::NSA; ++i) { mbar_init(&fullA[i], 1); mbar_init(&emptyA[i], C::NWC); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (z1e <= z0) return;
    // load l: P^k plane j = z0 - 2r + l;  for l >= 2r also the aux planes of
    // z1 = j - r (stage A of z1 at iteration l; stage B of z2 = z1 - r when l >= 4r)
    const int nload = (z1e - z0) + 4 * R;

    if (warp == C::NWC) {
        if (lane == 0) {
            tma_prefetch_desc(&map_p0); tma_prefetch_desc(&map_pm); tma_prefetch_desc(&map_k);
            for (int l = 0; l < nload; ++l) {
                const int j = z0 - 2 * R + l, s = l % C::NSP;
                mbar_wait(&emptyP[s], ((l / C::NSP) & 1) ^ 1);
                mbar_expect_tx(&fullP[s], C::P0_BYTES);
                tma_load_3d(sP0 + s * C::P0F, &map_p0, &fullP[s], x0 - 8, y0 - 2 * R, j + R);
                if (l >= 2 * R) {
                    const int a = l - 2 * R, z1 = j - R, sa = a % C::NSA;
                    mbar_wait(&emptyA[sa], ((a / C::NSA) & 1) ^ 1);
                    mbar_expect_tx(&fullA[sa], C::AUX_BYTES);
                    float *dst = sAux + sa * 2 * C::EF;
                    tma_load_3d(dst, &map_pm, &fullA[sa], x0 - 4, y0 - R, z1 + R);
                    tma_load_3d(dst + C::EF, &map_k, &fullA[sa], x0 - 4, y0 - R, z1);
                }
            }
        }
        return;
    }

    const int64_t nx = prm.nx, ny = prm.ny;
    const int64_t kk = step_index(prm);
    float *const trow1 = trace_row_of(prm, kk), *const trow2 = trace_row_of(prm, kk + 1);
    const float *const w1 = w_next_of(prm, kk), *const w2 = w_next_of(prm, kk + 1);
    int rpA = prm.rec.off ? prm.rec.off[unit] : 0, rpB = rpA;
    const int rend = prm.rec.off ? prm.rec.off[unit + 1] : 0;
    int rzA = rpA < rend ? prm.rec.z[rpA] : INT32_MAX, rzB = rzA;
    // sources whose (y, x) lies in the grown tile E (stage A injects there)
    uint32_t smask = 0;
    for (int q = 0; q < prm.nsrc; ++q)
        if (prm.sx[q] >= x0 - 4 && prm.sx[q] < x0 + C::TX + 4 && prm.sy[q] >= y0 - R && prm.sy[q] < y0 + C::TY + R)
            smask |= 1u << q;
    constexpr float c0 = tap(R, 0);
    // this thread's work items (fixed for every plane)
    constexpr int NIA = (C::ITEMS_A + C::NCONS - 1) / C::NCONS;
    constexpr int NIB = (C::ITEMS_B + C::NCONS - 1) / C::NCONS;
    int qA[NIA], reA[NIA], xbA[NIA];
    uint32_t inxA[NIA];                  // bit e: x term included for point e
#pragma unroll
    for (int ii = 0; ii < NIA; ++ii) {
        const int it = min(tid + ii * C::NCONS, C::ITEMS_A - 1);
        qA[ii] = it % C::QXE;
        reA[ii] = (it / C::QXE) * C::NYA;
        xbA[ii] = x0 - 4 + 4 * qA[ii];
        inxA[ii] = 0;
        for (int e = 0; e < 4; ++e) inxA[ii] |= (uint32_t)((xbA[ii] + e >= R) && (xbA[ii] + e < nx - R)) << e;
    }
    int qB[NIB], riB[NIB], xbB[NIB];
    uint32_t inxB[NIB];
#pragma unroll
    for (int ii = 0; ii < NIB; ++ii) {
        const int it = min(tid + ii * C::NCONS, C::ITEMS_B - 1);
        qB[ii] = it % C::QXI + 1;
        riB[ii] = (it / C::QXI) * C::NYB;
        xbB[ii] = x0 + 4 * (qB[ii] - 1);
        inxB[ii] = 0;
        for (int e = 0; e < 4; ++e) inxB[ii] |= (uint32_t)((xbB[ii] + e >= R) && (xbB[ii] + e < nx - R)) << e;
    }

    for (int l = 2 * R; l < nload; ++l) {
        const int j = z0 - 2 * R + l, z1 = j - R, a = l - 2 * R;
        mbar_wait(&fullP[l % C::NSP], (l / C::NSP) & 1);
        mbar_wait(&fullA[a % C::NSA], (a / C::NSA) & 1);
        // ------------------------------------------------ stage A: P^{k+1}(z1) on E
        {
            const float *pz[2 * R + 1];                     // P^k planes z1-r .. z1+r
#pragma unroll
            for (int m = 0; m <= 2 * R; ++m) pz[m] = sP0 + ((l - 2 * R + m) % C::NSP) * C::P0F;
            const float *tc = pz[R];
            const float *tpm = sAux + (a % C::NSA) * 2 * C::EF, *tk = tpm + C::EF;
            float *t1 = sP1 + (a % C::NS1) * C::EF;
            const int64_t gz = prm.gz0 + z1;
            const bool inz = (gz >= R) && (gz < prm.nzg - R);
            const bool store = (z1 >= z0) && (z1 < z1e);
            const bool recs_here = store && trow1 && rzA == z1;
            bool srcs_here = false;
            if (smask)
                for (int q = 0; q < prm.nsrc; ++q) srcs_here |= ((smask >> q) & 1u) && prm.sz[q] == z1;
#pragma unroll
            for (int ii = 0; ii < NIA; ++ii) {
                if (tid + ii * C::NCONS >= C::ITEMS_A) break;
                const int q = qA[ii], re0 = reA[ii], xb = xbA[ii];   // quad, first E row, first x
                bool inx[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) inx[e] = (inxA[ii] >> e) & 1u;
                float4 col[C::NYA + 2 * R];
#pragma unroll
                for (int i = 0; i < C::NYA + 2 * R; ++i) col[i] = lds128(tc + (re0 + i) * C::BX0 + 4 * q + 4);
#pragma unroll
                for (int yy = 0; yy < C::NYA; ++yy) {
                    const int re = re0 + yy, r0 = re + R, y = y0 - R + re;
                    const int off0 = r0 * C::BX0 + 4 * q;
                    const float4 L4 = lds128(tc + off0), M4 = col[yy + R], R4 = lds128(tc + off0 + 8);
                    const float av[12] = {L4.x, L4.y, L4.z, L4.w, M4.x, M4.y, M4.z, M4.w, R4.x, R4.y, R4.z, R4.w};
                    float4 zl[R], zh[R];
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        zl[m - 1] = lds128(pz[R - m] + off0 + 4);
                        zh[m - 1] = lds128(pz[R + m] + off0 + 4);
                    }
                    const int offe = re * C::BXE + 4 * q;
                    const float4 pm4 = lds128(tpm + offe);
                    const float4 k4 = lds128(tk + offe);
                    const bool iny = (y >= R) && (y < ny - R);
                    float4 o;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float pc = av[4 + e];
                        float sx = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m) sx = __fmaf_rn(tap(R, m), __fadd_rn(av[4 + e - m], av[4 + e + m]), sx);
                        float S = inx[e] ? sx : 0.f;
                        float sy = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            sy = __fmaf_rn(tap(R, m), __fadd_rn(f4(col[yy + R - m], e), f4(col[yy + R + m], e)), sy);
                        S = iny ? __fadd_rn(S, sy) : S;
                        float sz = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            sz = __fmaf_rn(tap(R, m), __fadd_rn(f4(zl[m - 1], e), f4(zh[m - 1], e)), sz);
                        S = inz ? __fadd_rn(S, sz) : S;
                        f4set(o, e, __fmaf_rn(f4(k4, e), S, __fmaf_rn(2.f, pc, -f4(pm4, e))));
                    }
                    const bool interior = q >= 1 && q <= C::QXI && re >= R && re < R + C::TY && y < ny;
                    if (recs_here && interior) {                   // raw P^{k+1}, owner only
                        for (int rp = rpA; rp < rend && prm.rec.z[rp] == z1; ++rp) {
                            if (prm.rec.y[rp] != y) continue;
                            const int dx = prm.rec.x[rp] - xb;
                            if (dx >= 0 && dx < 4) trow1[prm.rec.id[rp]] = f4(o, dx);
                        }
                    }
                    if (srcs_here) {                               // w_{k+1} wherever in E
                        for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                            if (prm.sz[s2] != z1 || prm.sy[s2] != y) continue;
                            const int dx = prm.sx[s2] - xb;
                            if (dx >= 0 && dx < 4) f4set(o, dx, __fadd_rn(f4(o, dx), w1[s2]));
                        }
                    }
                    *reinterpret_cast<float4 *>(t1 + offe) = o;
                    if (store && interior && xb < prm.pitch)
                        *reinterpret_cast<float4 *>(prm.pnext + ((int64_t)(z1 + R) * ny + y) * prm.pitch + xb) = o;
                }
            }
            // aux planes below z0 are not needed by stage B: release now
            __syncwarp();
            if (lane == 0 && a < R) mbar_arrive(&emptyA[a % C::NSA]);
        }
        if (rzA == z1) {
            while (rpA < rend && prm.rec.z[rpA] <= z1) ++rpA;
            rzA = rpA < rend ? prm.rec.z[rpA] : INT32_MAX;
        }
        consumer_barrier(C::NCONS);
        // ------------------------------------------------ stage B: P^{k+2}(z2) on the tile
        if (l >= 4 * R) {
            const int z2 = z1 - R, b = a - R;                        // aux index of plane z2
            const float *tpk = sP0 + ((l - 2 * R) % C::NSP) * C::P0F;  // P^k plane z2
            const float *tk = sAux + (b % C::NSA) * 2 * C::EF + C::EF;
            const float *p1[2 * R + 1];                              // P^{k+1} planes z2-r .. z2+r
#pragma unroll
            for (int m = 0; m <= 2 * R; ++m) p1[m] = sP1 + ((b - R + m) % C::NS1) * C::EF;
            const float *t1c = p1[R];
            const int64_t gz = prm.gz0 + z2;
            const bool inz = (gz >= R) && (gz < prm.nzg - R);
            const bool recs_here = trow2 && rzB == z2;
            bool srcs_here = false;
            if (smask)
                for (int q = 0; q < prm.nsrc; ++q) srcs_here |= ((smask >> q) & 1u) && prm.sz[q] == z2;
#pragma unroll
            for (int ii = 0; ii < NIB; ++ii) {
                if (tid + ii * C::NCONS >= C::ITEMS_B) break;
                const int q = qB[ii], ri0 = riB[ii], xb = xbB[ii];
                bool inx[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) inx[e] = (inxB[ii] >> e) & 1u;
                float4 col[C::NYB + 2 * R];
#pragma unroll
                for (int i = 0; i < C::NYB + 2 * R; ++i) col[i] = lds128(t1c + (ri0 + i) * C::BXE + 4 * q);
#pragma unroll
                for (int yy = 0; yy < C::NYB; ++yy) {
                    const int re = ri0 + yy + R, y = y0 + ri0 + yy;
                    const int offe = re * C::BXE + 4 * q;
                    const float4 L4 = lds128(t1c + offe - 4), M4 = col[yy + R], R4 = lds128(t1c + offe + 4);
                    const float av[12] = {L4.x, L4.y, L4.z, L4.w, M4.x, M4.y, M4.z, M4.w, R4.x, R4.y, R4.z, R4.w};
                    float4 zl[R], zh[R];
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        zl[m - 1] = lds128(p1[R - m] + offe);
                        zh[m - 1] = lds128(p1[R + m] + offe);
                    }
                    const float4 pk4 = lds128(tpk + (re + R) * C::BX0 + 4 * q + 4);
                    const float4 k4 = lds128(tk + offe);
                    const bool iny = (y >= R) && (y < ny - R);
                    float4 out;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float pc = av[4 + e];
                        float sx = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m) sx = __fmaf_rn(tap(R, m), __fadd_rn(av[4 + e - m], av[4 + e + m]), sx);
                        float S = inx[e] ? sx : 0.f;
                        float sy = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            sy = __fmaf_rn(tap(R, m), __fadd_rn(f4(col[yy + R - m], e), f4(col[yy + R + m], e)), sy);
                        S = iny ? __fadd_rn(S, sy) : S;
                        float sz = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            sz = __fmaf_rn(tap(R, m), __fadd_rn(f4(zl[m - 1], e), f4(zh[m - 1], e)), sz);
                        S = inz ? __fadd_rn(S, sz) : S;
                        f4set(out, e, __fmaf_rn(f4(k4, e), S, __fmaf_rn(2.f, pc, -f4(pk4, e))));
                    }
                    if (recs_here) {
                        for (int rp = rpB; rp < rend && prm.rec.z[rp] == z2; ++rp) {
                            if (prm.rec.y[rp] != y) continue;
                            const int dx = prm.rec.x[rp] - xb;
                            if (dx >= 0 && dx < 4) trow2[prm.rec.id[rp]] = f4(out, dx);
                        }
                    }
                    if (srcs_here) {
                        for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                            if (prm.sz[s2] != z2 || prm.sy[s2] != y) continue;
                            const int dx = prm.sx[s2] - xb;
                            if (dx >= 0 && dx < 4) {
                                const float v = f4(out, dx);
                                prm.src_raw[s2] = v;
                                f4set(out, dx, __fadd_rn(v, w2[s2]));
                            }
                        }
                    }
                    if (y < ny && xb < prm.pitch)
                        *reinterpret_cast<float4 *>(prm.pnext2 + ((int64_t)(z2 + R) * ny + y) * prm.pitch + xb) = out;
                }
            }
            if (rzB == z2) {
                while (rpB < rend && prm.rec.z[rpB] <= z2) ++rpB;
                rzB = rpB < rend ? prm.rec.z[rpB] : INT32_MAX;
            }
            // release: aux plane z2 (its K tile was the last use)
            __syncwarp();
            if (lane == 0) mbar_arrive(&emptyA[b % C::NSA]);
        }
        // release P^k plane j - 2r: last used by this iteration (stage A z taps,
        // stage B pointwise)
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyP[(l - 2 * R) % C::NSP]);
    }
}

}  // namespace fdk
