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
// pass is bitwise two single steps.  (A first version ran both stages on all
// warps with a CTA barrier per plane and z taps from shared memory: 2.3x the
// instructions of the single-step kernel, 339 Gpts/s on C3 -- replaced.)  HBM traffic per pair of updates: read
// P^k, P^{k-1}, K once, write P^{k+1}, P^{k+2}: 20 B, i.e. 10 B per update
// instead of 16.  The x-y halo ring of stage A is recomputed by neighbouring
// tiles (redundant compute instead of communication).
//
// Buffers: four field buffers rotate (cur, prev) -> (C, D); none is written
// while another CTA may still read it (P^k and P^{k-1} are read with halos).
// On z-slabs the halos are 2r planes of P^k and r of P^{k-1} (fd_runtime.cu).
#pragma once
#include "fd_kernels.cuh"

namespace fdk {

// Role-barrier arrivals of the A / B warps.  Default: every thread arrives
// (each thread releases its own shared-memory accesses -- the form
// compute-sanitizer racecheck can follow).  FD_TB2_THREAD_ARRIVE=0: one
// arrival per warp after __syncwarp (which orders the lanes' accesses before
// lane 0's release-arrive); same speed (r05 A/B: 581.6 vs 581.5 Gpts/s, the
// same 12.2 M re-polls of stage A on empty P1 slots), but racecheck reports
// the per-warp form as hazards between A's P1 stores and B's loads.
#ifndef FD_TB2_THREAD_ARRIVE
#define FD_TB2_THREAD_ARRIVE 1
#endif
#ifndef FD_TB2_ROTATE
#define FD_TB2_ROTATE 0
#endif
constexpr int kArrivalsPerWarp = FD_TB2_THREAD_ARRIVE ? 32 : 1;

template <class... B>
__device__ __forceinline__ void role_release(B *...bars) {
#if FD_TB2_THREAD_ARRIVE
    (mbar_arrive(bars), ...);
#else
    __syncwarp();
    if ((threadIdx.x & 31) == 0) (mbar_arrive(bars), ...);
#endif
}

// x taps of a thread's quad: av[0..3] = the left quad, av[4..7] = M4 (the
// thread's own 4 points), av[8..11] = the right quad; only av[4-R..3] and
// av[8..7+R] are read.  For R <= 2 the halo values are the neighbouring lanes'
// own quads (lane - 1 / lane + 1 own x - 4 .. x - 1 / x + 4 .. x + 7): taken by
// warp shuffles, and from shared memory (`lq` = the left quad's address, the
// right quad at lq + 8) only by the lanes whose neighbour in x is not the
// adjacent lane (needL / needR: warp edge or row-group edge).  The scalar
// halo loads they replace read 4 B at a 16 B lane stride -- 4-way bank
// conflicts, 76 % of the excess shared wavefronts of the r05f profile.  Every
// lane of the warp must execute this (full-mask shuffles).
// FD_XSHFL_3D: 0 (default) the halo quads from shared memory; 1 shuffles in
// both stages of tb2ws, 2 stage B only, 3 stage A only.  r2 A/B on B200
// (scripts/ab.sh, C3 order 2, 200-step runs): shared-memory halos 622.8 Gpts/s,
// shuffles in both stages 599.5 -- the shuffles sit on the dependent chain
// after the z-queue value and add the edge-lane branches; the 2D kernel lost
// 4 % (C2 order 2) and 12 % (order 4) with them, so it keeps its loads.
#ifndef FD_XSHFL_3D
#define FD_XSHFL_3D 0
#endif
// FD_TB2_COLQ: the y-tap column takes the thread's own rows from its z queue
// instead of re-reading them from shared memory -- bit 0: stage A, bit 1:
// stage B (3: both)
#ifndef FD_TB2_COLQ
#define FD_TB2_COLQ 3
#endif
template <int R, bool SHFL>
__device__ __forceinline__ void quad_xtaps(float (&av)[12], const float4 M4, const float *lq, bool needL, bool needR) {
    av[4] = M4.x; av[5] = M4.y; av[6] = M4.z; av[7] = M4.w;
    if constexpr (SHFL && R <= 2) {
#pragma unroll
        for (int m = 1; m <= R; ++m) {
            av[4 - m] = __shfl_up_sync(0xffffffffu, f4(M4, 4 - m), 1);
            av[7 + m] = __shfl_down_sync(0xffffffffu, f4(M4, m - 1), 1);
        }
        if (needL) {
            const float4 L4 = lds128(lq);
            av[0] = L4.x; av[1] = L4.y; av[2] = L4.z; av[3] = L4.w;
        }
        if (needR) {
            const float4 R4 = lds128(lq + 8);
            av[8] = R4.x; av[9] = R4.y; av[10] = R4.z; av[11] = R4.w;
        }
    } else {
        const float4 L4 = lds128(lq), R4 = lds128(lq + 8);
        av[0] = L4.x; av[1] = L4.y; av[2] = L4.z; av[3] = L4.w;
        av[8] = R4.x; av[9] = R4.y; av[10] = R4.z; av[11] = R4.w;
    }
}

// ------------------------------------------------------------------ warp-specialised variant
// Same two-step pass, but stage A and stage B run on separate warp groups that
// overlap (no CTA barrier per plane) and both keep their z taps in a register
// queue like the single-step kernel:
//   warp 0..NWA-1   : stage A, threads own a quad column x NYA rows of the grown
//                     tile E; queue of 2r+1 planes of P^k; write P^{k+1} to the
//                     shared ring P1 (and C for the tile interior)
//   warp NWA..+NWB-1: stage B, threads own a quad column x NYB rows of the tile;
//                     queue of 2r+1 planes of P^{k+1}; write P^{k+2} to D
//   last warp       : TMA producer
// Rings (mbarrier full/empty): P^k planes (released by A after its x-y taps
// and by B after its pointwise read), (P^{k-1}, K) planes (A: stage A, B: K of
// stage B), P1 planes (full: A -> B, empty: B -> A).
template <int R_, int TX_, int TY_, int NYA_, int NYB_, int DP_, int DA_, int D1_, int MINB_ = 1>
struct CfgWS {
    static constexpr int R = R_, TX = TX_, TY = TY_, NYA = NYA_, NYB = NYB_, DP = DP_, DA = DA_, D1 = D1_;
    static constexpr int MINB = MINB_;          // __launch_bounds__ min blocks per SM (register cap)
    static constexpr int BX0 = TX + 16, BY0 = TY + 4 * R;         // P^k tile (x halo 8, y halo 2r)
    static constexpr int BXE = TX + 8, BYE = TY + 2 * R;          // grown tile E
    static constexpr int QXE = BXE / 4, QXI = TX / 4;
    static constexpr int NTA = QXE * (BYE / NYA), NTB = QXI * (TY / NYB);   // active threads per role
    static constexpr int NWA = (NTA + 31) / 32, NWB = (NTB + 31) / 32;
    static constexpr int NTHREADS = 32 * (NWA + NWB + 1);
    static constexpr int P0F = (BX0 * BY0 + 31) / 32 * 32;
    static constexpr int EF = (BXE * BYE + 31) / 32 * 32;
    static constexpr int NSP = 2 * R + 1 + DP;    // P^k planes z2 .. z1+r (A reads z1+r newest, B reads z2)
    static constexpr int NSA = R + 1 + DA;        // aux planes z2 .. z1
    static constexpr int NS1 = R + 1 + D1;        // P1 planes z2 .. z1
    static constexpr uint32_t P0_BYTES = BX0 * BY0 * 4, AUX_BYTES = 2 * BXE * BYE * 4;
    static constexpr int SMEM_FLOATS = NSP * P0F + NSA * 2 * EF + NS1 * EF;
    static constexpr int SMEM_BYTES = SMEM_FLOATS * 4 + (2 * NSP + 2 * NSA + 2 * NS1) * 8 + 16;
    static constexpr int NY = NYB;
    static_assert(BYE % NYA == 0 && TY % NYB == 0, "tile");
    static_assert(BX0 <= 256 && BY0 <= 256 && R <= 4, "TMA box");
};

template <class C, bool SP, bool PEER, bool KZ>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
tb2ws_step_kernel(const __grid_constant__ CUtensorMap map_p0, const __grid_constant__ CUtensorMap map_pm,
                  const __grid_constant__ CUtensorMap map_k, const StepParams prm) {
    constexpr int R = C::R;
    extern __shared__ __align__(128) float smem[];
    float *sP0 = smem;
    float *sAux = sP0 + C::NSP * C::P0F;
    float *sP1 = sAux + C::NSA * 2 * C::EF;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sP1 + C::NS1 * C::EF);
    uint64_t *fullP = bars, *emptyP = fullP + C::NSP;
    uint64_t *fullA = emptyP + C::NSP, *emptyA = fullA + C::NSA;
    uint64_t *full1 = emptyA + C::NSA, *empty1 = full1 + C::NS1;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntiles = prm.ntx * prm.nty;
    const int unit = blockIdx.x;
    const int chunk = unit / ntiles, tile = unit - chunk * ntiles;
    const int x0 = (tile % prm.ntx) * C::TX, y0 = (tile / prm.ntx) * C::TY;
    const int span = prm.zhi - prm.zlo;
    const int z0 = prm.zlo + (int)(((int64_t)span * chunk) / prm.nchunks);
    const int z1e = prm.zlo + (int)(((int64_t)span * (chunk + 1)) / prm.nchunks);
    if (tid == 0) {
        // role barriers count the arriving warps (or threads, see role_release)
        for (int i = 0; i < C::NSP; ++i) { mbar_init(&fullP[i], 1); mbar_init(&emptyP[i], kArrivalsPerWarp * (C::NWA + C::NWB)); }
        for (int i = 0; i < C::NSA; ++i) { mbar_init(&fullA[i], 1); mbar_init(&emptyA[i], kArrivalsPerWarp * (C::NWA + C::NWB)); }
        for (int i = 0; i < C::NS1; ++i) { mbar_init(&full1[i], kArrivalsPerWarp * C::NWA); mbar_init(&empty1[i], kArrivalsPerWarp * C::NWB); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_sync();
    if (z1e <= z0) return;
    // P^k load l: plane j = z0 - 2r + l (l < nload); aux load a (a = l - 2r >= 0):
    // plane z1 = z0 - r + a.  Stage A iteration a (l = a + 2r) computes P^{k+1}(z1);
    // stage B iteration a (a >= 2r) computes P^{k+2}(z2 = z1 - r).
    const int nload = (z1e - z0) + 4 * R, na = nload - 2 * R;
    const int nx = (int)prm.nx, ny = (int)prm.ny;   // 32-bit index math (dims <= 2^30)
    const int64_t kk = step_index(prm);
    constexpr float c0 = tap(R, 0);
    int rp = prm.rec.off ? prm.rec.off[unit] : 0;
    const int rend = prm.rec.off ? prm.rec.off[unit + 1] : 0;
    int rz = rp < rend ? prm.rec.z[rp] : INT32_MAX;

    if (warp == C::NWA + C::NWB) {
        // -------------------------------------------------------------- producer
        if (lane == 0) {
            tma_prefetch_desc(&map_p0); tma_prefetch_desc(&map_pm); tma_prefetch_desc(&map_k);
            for (int l = 0; l < nload; ++l) {
                const int j = z0 - 2 * R + l, s = l % C::NSP;
                mbar_wait_producer(&emptyP[s], ((l / C::NSP) & 1) ^ 1);
                mbar_expect_tx(&fullP[s], C::P0_BYTES);
                tma_load_3d(sP0 + s * C::P0F, &map_p0, &fullP[s], x0 - 8, y0 - 2 * R, j + halo_planes(R));
                if (l >= 2 * R) {
                    const int a = l - 2 * R, z1 = j - R, sa = a % C::NSA;
                    mbar_wait_producer(&emptyA[sa], ((a / C::NSA) & 1) ^ 1);
                    mbar_expect_tx(&fullA[sa], KZ ? C::AUX_BYTES / 2 : C::AUX_BYTES);
                    float *dst = sAux + sa * 2 * C::EF;
                    tma_load_3d(dst, &map_pm, &fullA[sa], x0 - 4, y0 - R, z1 + halo_planes(R));
                    if constexpr (!KZ)
                        tma_load_3d(dst + C::EF, &map_k, &fullA[sa], x0 - 4, y0 - R, z1 + R);   // K halo buffer
                }
            }
        }
        return;
    }

    constexpr int Q = 2 * R + 1;
    const int64_t plane = (int64_t)ny * prm.pitch;   // floats per buffer plane
    const int pitch = (int)prm.pitch;
    // The z-tap queues shift by 2r float4 moves per plane (FD_TB2_ROTATE=1
    // instead unrolls the loops by Q = 2r+1 so that at phase PH = iteration mod
    // Q the entry of logical position i (plane j - 2r + i) lives in
    // qz[(PH + i) % Q] -- no moves, but ncu r05: 19 % fewer instructions and
    // 1.4x the time, instruction-cache misses (no_instruction stalls) and
    // spills at the 128-register cap).  Ring slots and parities advance
    // incrementally (RingPos) instead of by divisions, and the per-row
    // predicates and store offsets are loop invariants.

    if (warp < C::NWA) {
        // -------------------------------------------------------------- stage A
        const bool act = tid < C::NTA;
        const int q = act ? tid % C::QXE : 0, re0 = act ? (tid / C::QXE) * C::NYA : 0;
        const int xb = x0 - 4 + 4 * q;                 // first x of the quad (E coordinates 4q)
        bool inx[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) inx[e] = (xb + e >= R) && (xb + e < nx - R);
        float sgx[4], sgy[C::NYA];                     // sponge factors (SP only)
#pragma unroll
        for (int e = 0; e < 4; ++e) sgx[e] = SP ? sponge_gx(prm, xb + e) : 1.f;
#pragma unroll
        for (int yy = 0; yy < C::NYA; ++yy) sgy[yy] = SP ? sponge_gy(prm, y0 - R + re0 + yy) : 1.f;
        const bool qint = q >= 1 && q <= C::QXI;
        const bool needL = lane == 0 || q == 0, needR = lane == 31 || q == C::QXE - 1;
        // per row: band rule along y, stored to C (tile interior), offset in a plane
        uint32_t ymask = 0, stmask = 0;
        int roff[C::NYA];
#pragma unroll
        for (int yy = 0; yy < C::NYA; ++yy) {
            const int re = re0 + yy, y = y0 - R + re;
            if (y >= R && y < ny - R) ymask |= 1u << yy;
            if (act && qint && re >= R && re < R + C::TY && y < ny && xb < pitch) stmask |= 1u << yy;
            roff[yy] = y * pitch + xb;
        }
        uint32_t smask = 0;                            // sources in this thread's columns/rows of E
        for (int s2 = 0; s2 < prm.nsrc; ++s2)
            if (act && prm.sx[s2] >= xb && prm.sx[s2] < xb + 4 && prm.sy[s2] >= y0 - R + re0 &&
                prm.sy[s2] < y0 - R + re0 + C::NYA)
                smask |= 1u << s2;
        float *const trow = trace_row_of(prm, kk);
        const float *const wv = w_next_of(prm, kk);
        float4 qz[Q][C::NYA];
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
            for (int yy = 0; yy < C::NYA; ++yy) qz[i][yy] = make_float4(0.f, 0.f, 0.f, 0.f);
        RingPos<C::NSP> pl;                            // P^k load l (full wait)
        RingPos<C::NSP> pz{C::NSP - R, 0u};            // P^k load l - r (plane z1: x-y taps)
        RingPos<C::NSA> pa;                            // aux plane a
        RingPos<C::NS1> p1;                            // P1 plane a
        auto body = [&](const int l, auto ph) {
            constexpr int PH = decltype(ph)::value;
            mbar_wait(&fullP[pl.slot], pl.par);
            const float *tp = sP0 + pl.slot * C::P0F;
#pragma unroll
            for (int yy = 0; yy < C::NYA; ++yy)
                qz[(PH + 2 * R) % Q][yy] = lds128(tp + (re0 + yy + R) * C::BX0 + 4 * q + 4);
            if (l < 2 * R) {
                // planes below z0 - r are z taps only: A is done with them now;
                // planes z0 - r .. z0 - 1 still serve A's x-y taps (released there)
                if (l < R) role_release(&emptyP[pl.slot]);
                pl.next(); pz.next();
                return;
            }
            const int a = l - 2 * R, z1 = z0 - R + a;
            const float *tc = sP0 + pz.slot * C::P0F;      // P^k plane z1 (x-y taps)
            mbar_wait(&fullA[pa.slot], pa.par);
            const float *tpm = sAux + pa.slot * 2 * C::EF, *tk = tpm + C::EF;
            mbar_wait(&empty1[p1.slot], p1.par ^ 1u);
            float *t1 = sP1 + p1.slot * C::EF;
            const int gz = (int)prm.gz0 + z1;
            const bool inz = (gz >= R) && (gz < (int)prm.nzg - R);
            const float sgz = SP ? sponge_gz(prm, gz) : 1.f;
            const float kza = KZ ? kplane(prm, z1) : 0.f;
            const bool store = (z1 >= z0) && (z1 < z1e);
            const bool push1 = PEER && peer_plane(prm.peer1, z1, (int)prm.nz);
            float *const cpl = prm.pnext + (int64_t)(z1 + halo_planes(R)) * plane;
            float4 oraw[C::NYA];                                  // raw P^{k+1} (receivers)
#pragma unroll
            for (int yy = 0; yy < C::NYA; ++yy) oraw[yy] = make_float4(0.f, 0.f, 0.f, 0.f);
            // shuffled x taps need every lane (inactive ones compute on row 0 / quad 0 and store nothing)
            if (FD_XSHFL_3D == 1 || FD_XSHFL_3D == 3 || act) {
                float4 col[C::NYA + 2 * R];       // y taps; the thread's own rows are its z-queue centre
#pragma unroll
                for (int i = 0; i < C::NYA + 2 * R; ++i)
                    col[i] = ((FD_TB2_COLQ & 1) && i >= R && i < R + C::NYA) ? qz[(PH + R) % Q][i - R]
                                                                      : lds128(tc + (re0 + i) * C::BX0 + 4 * q + 4);
#pragma unroll
                for (int yy = 0; yy < C::NYA; ++yy) {
                    const int re = re0 + yy;
                    float av[12];
                    quad_xtaps<R, FD_XSHFL_3D == 1 || FD_XSHFL_3D == 3>(av, qz[(PH + R) % Q][yy], tc + (re + R) * C::BX0 + 4 * q, needL, needR);
                    const int offe = re * C::BXE + 4 * q;
                    const float4 pm4 = lds128(tpm + offe), k4 = KZ ? splat4(kza) : lds128(tk + offe);
                    const bool iny = (ymask >> yy) & 1u;
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
                        float szz = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            szz = __fmaf_rn(tap(R, m), __fadd_rn(f4(qz[(PH + R - m) % Q][yy], e),
                                                                  f4(qz[(PH + R + m) % Q][yy], e)), szz);
                        S = inz ? __fadd_rn(S, szz) : S;
                        f4set(o, e, time_update<SP>(f4(k4, e), S, pc, f4(pm4, e), sgz, sgy[yy], sgx[e]));
                    }
                    oraw[yy] = o;
                    if (smask) {                                      // w_{k+1} wherever in E
                        const int y = y0 - R + re;
                        for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                            if (!((smask >> s2) & 1u) || prm.sz[s2] != z1 || prm.sy[s2] != y) continue;
                            const int dx = prm.sx[s2] - xb;
                            f4set(o, dx, __fadd_rn(f4(o, dx), wv[s2]));
                        }
                    }
                    if (act) *reinterpret_cast<float4 *>(t1 + offe) = o;
                    if (store && ((stmask >> yy) & 1u)) {
                        *reinterpret_cast<float4 *>(cpl + roff[yy]) = o;
                        if (push1) peer_store4<R>(prm.peer1, z1, (int)prm.nz, plane, (int64_t)roff[yy], o);
                    }
                }
            }
            if (store && rz == z1) {                              // owners: tile-interior A threads
                rp = warp_record<C::NYA>(oraw, prm.rec.z, prm.rec.id, rp, rend, z1, z1 + 1, trow,
                                         [&](int i, int &ln, int &yy, int &e) {
                                             const int re = prm.rec.y[i] - (y0 - R), dx = prm.rec.x[i] - (x0 - 4);
                                             const int t = (re / C::NYA) * C::QXE + dx / 4;
                                             if ((t >> 5) != warp) return false;
                                             ln = t & 31; yy = re % C::NYA; e = dx & 3;
                                             return true;
                                         });
                rz = rp < rend ? prm.rec.z[rp] : INT32_MAX;
            }
            // P1 plane z1 ready; P^k plane z1 done for A (x-y taps); aux plane z1
            // done for A; planes of P^k below the window are A-done at their read
            role_release(&full1[p1.slot], &emptyP[pz.slot], &emptyA[pa.slot]);
            pl.next(); pz.next(); pa.next(); p1.next();
        };
#if FD_TB2_ROTATE
        for (int l0 = 0; l0 < nload; l0 += Q)
            static_for<0, Q>([&](auto ph) {
                if (l0 + decltype(ph)::value < nload) body(l0 + decltype(ph)::value, ph);
            });
#else
        for (int l = 0; l < nload; ++l) {
#pragma unroll
            for (int i = 0; i < 2 * R; ++i)
#pragma unroll
                for (int yy = 0; yy < C::NYA; ++yy) qz[i][yy] = qz[i + 1][yy];
            body(l, std::integral_constant<int, 0>{});
        }
#endif
        // P^k planes z1e + r .. z1e + 2r - 1 (the last r loads) were only z taps: A-done
        // (released when read? they are released by B too); nothing else to release
        return;
    }

    // ------------------------------------------------------------------ stage B
    const int tb = tid - 32 * C::NWA;
    const bool act = tb < C::NTB;
    const int qi = act ? tb % C::QXI : 0, ri0 = act ? (tb / C::QXI) * C::NYB : 0;
    const int q = qi + 1, xb = x0 + 4 * qi;
    const bool needL = lane == 0 || qi == 0, needR = lane == 31 || qi == C::QXI - 1;
    bool inx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) inx[e] = (xb + e >= R) && (xb + e < nx - R);
    float sgx[4], sgy[C::NYB];                         // sponge factors (SP only)
#pragma unroll
    for (int e = 0; e < 4; ++e) sgx[e] = SP ? sponge_gx(prm, xb + e) : 1.f;
#pragma unroll
    for (int yy = 0; yy < C::NYB; ++yy) sgy[yy] = SP ? sponge_gy(prm, y0 + ri0 + yy) : 1.f;
    uint32_t ymask = 0, vmask = 0;                     // band rule along y; rows inside the grid
#pragma unroll
    for (int yy = 0; yy < C::NYB; ++yy) {
        const int y = y0 + ri0 + yy;
        if (y >= R && y < ny - R) ymask |= 1u << yy;
        if (y < ny) vmask |= 1u << yy;
    }
    const int boff = (y0 + ri0) * pitch + xb;          // row ri0 of this thread within a plane
    uint32_t smask = 0;
    for (int s2 = 0; s2 < prm.nsrc; ++s2)
        if (act && prm.sx[s2] >= xb && prm.sx[s2] < xb + 4 && prm.sy[s2] >= y0 + ri0 && prm.sy[s2] < y0 + ri0 + C::NYB)
            smask |= 1u << s2;
    float *const trow = trace_row_of(prm, kk + 1);
    const float *const wv = w_next_of(prm, kk + 1);
    float4 qz[Q][C::NYB];
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int yy = 0; yy < C::NYB; ++yy) qz[i][yy] = make_float4(0.f, 0.f, 0.f, 0.f);
    // B's releases run in plane order on every ring: P^k load a, aux plane and
    // P1 plane 0, 1, ... (warm-up planes as they pass, then plane z2's)
    RingPos<C::NS1> f1;                                // P1 plane a (full wait)
    RingPos<C::NSP> rP;                                // P^k load a (= plane z2 for a >= 2r)
    RingPos<C::NSA> rA;                                // next aux plane to release
    RingPos<C::NS1> r1;                                // next P1 plane to release
    auto body = [&](const int a, auto ph) {
        constexpr int PH = decltype(ph)::value;
        mbar_wait(&full1[f1.slot], f1.par);
        const float *t1n = sP1 + f1.slot * C::EF;
#pragma unroll
        for (int yy = 0; yy < C::NYB; ++yy) qz[(PH + 2 * R) % Q][yy] = lds128(t1n + (ri0 + yy + R) * C::BXE + 4 * q);
        f1.next();
        if (a < 2 * R) {
            // warm-up: B never reads P^k loads 0 .. 2r-1 (it reads P^k at z2 >= z0,
            // load b + r >= 2r) nor aux planes 0 .. r-1; P1 planes 0 .. r-1 are z
            // taps only.  Release them as this iteration passes.
            if (a < R) {
                role_release(&emptyP[rP.slot], &empty1[r1.slot], &emptyA[rA.slot]);
                r1.next(); rA.next();
            } else {
                role_release(&emptyP[rP.slot]);
            }
            rP.next();
            return;
        }
        const int b = a - R, z2 = z0 - R + b;               // plane computed now (>= z0)
        const float *t1c = sP1 + r1.slot * C::EF;           // P1 plane z2 (x-y taps)
        const float *tpk = sP0 + rP.slot * C::P0F;          // P^k plane z2 = load b + r
        const float *tk = sAux + rA.slot * 2 * C::EF + C::EF;   // aux plane z2 (K)
        const int gz = (int)prm.gz0 + z2;
        const bool inz = (gz >= R) && (gz < (int)prm.nzg - R);
        const float sgz = SP ? sponge_gz(prm, gz) : 1.f;
        const float kzb = KZ ? kplane(prm, z2) : 0.f;
        float4 out[C::NYB];
        if (FD_XSHFL_3D == 1 || FD_XSHFL_3D == 2 || act) {   // (shuffles: every lane)
            float4 col[C::NYB + 2 * R];           // y taps; the thread's own rows are its z-queue centre
#pragma unroll
            for (int i = 0; i < C::NYB + 2 * R; ++i)
                col[i] = ((FD_TB2_COLQ & 2) && i >= R && i < R + C::NYB) ? qz[(PH + R) % Q][i - R]
                                                                  : lds128(t1c + (ri0 + i) * C::BXE + 4 * q);
#pragma unroll
            for (int yy = 0; yy < C::NYB; ++yy) {
                const int re = ri0 + yy + R;
                const int offe = re * C::BXE + 4 * q;
                float av[12];
                quad_xtaps<R, FD_XSHFL_3D == 1 || FD_XSHFL_3D == 2>(av, qz[(PH + R) % Q][yy], t1c + offe - 4, needL, needR);
                const float4 pk4 = lds128(tpk + (re + R) * C::BX0 + 4 * q + 4);
                const float4 k4 = KZ ? splat4(kzb) : lds128(tk + offe);
                const bool iny = (ymask >> yy) & 1u;
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
                    float szz = __fmul_rn(c0, pc);
#pragma unroll
                    for (int m = 1; m <= R; ++m)
                        szz = __fmaf_rn(tap(R, m), __fadd_rn(f4(qz[(PH + R - m) % Q][yy], e),
                                                              f4(qz[(PH + R + m) % Q][yy], e)), szz);
                    S = inz ? __fadd_rn(S, szz) : S;
                    f4set(out[yy], e, time_update<SP>(f4(k4, e), S, pc, f4(pk4, e), sgz, sgy[yy], sgx[e]));
                }
            }
        }
        // release: P1 plane z2 (x-y taps done; its column is in the queue), P^k
        // plane z2 (pointwise), aux plane z2 (K)
        role_release(&empty1[r1.slot], &emptyP[rP.slot], &emptyA[rA.slot]);
        r1.next(); rP.next(); rA.next();
        if (rz == z2) {                                           // owners: B threads
            rp = warp_record<C::NYB>(out, prm.rec.z, prm.rec.id, rp, rend, z2, z2 + 1, trow,
                                     [&](int i, int &ln, int &yy, int &e) {
                                         const int dy = prm.rec.y[i] - y0, dx = prm.rec.x[i] - x0;
                                         const int t = (dy / C::NYB) * C::QXI + dx / 4;
                                         if (C::NWA + (t >> 5) != warp) return false;
                                         ln = t & 31; yy = dy % C::NYB; e = dx & 3;
                                         return true;
                                     });
            rz = rp < rend ? prm.rec.z[rp] : INT32_MAX;
        }
        if (!act) return;
        if (smask) {
            for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                if (!((smask >> s2) & 1u) || prm.sz[s2] != z2) continue;
                const int dy = prm.sy[s2] - (y0 + ri0), dx = prm.sx[s2] - xb;
#pragma unroll
                for (int yy = 0; yy < C::NYB; ++yy)
                    if (yy == dy) {
                        const float v = f4(out[yy], dx);
                        prm.src_raw[s2] = v;
                        f4set(out[yy], dx, __fadd_rn(v, wv[s2]));
                    }
            }
        }
        if (xb < pitch) {
            float *dst = prm.pnext2 + (int64_t)(z2 + halo_planes(R)) * plane + boff;
#pragma unroll
            for (int yy = 0; yy < C::NYB; ++yy)
                if ((vmask >> yy) & 1u) *reinterpret_cast<float4 *>(dst + yy * pitch) = out[yy];
            if (PEER && peer_plane(prm.peer2, z2, (int)prm.nz)) {
#pragma unroll
                for (int yy = 0; yy < C::NYB; ++yy)
                    if ((vmask >> yy) & 1u)
                        peer_store4<R>(prm.peer2, z2, (int)prm.nz, plane, (int64_t)(boff + yy * pitch), out[yy]);
            }
        }
    };
#if FD_TB2_ROTATE
    for (int a0 = 0; a0 < na; a0 += Q)
        static_for<0, Q>([&](auto ph) {
            if (a0 + decltype(ph)::value < na) body(a0 + decltype(ph)::value, ph);
        });
#else
    for (int a = 0; a < na; ++a) {
#pragma unroll
        for (int i = 0; i < 2 * R; ++i)
#pragma unroll
            for (int yy = 0; yy < C::NYB; ++yy) qz[i][yy] = qz[i + 1][yy];
        body(a, std::integral_constant<int, 0>{});
    }
#endif
}


// ------------------------------------------------------------------ 2D two-step kernel
// 2D grids stream TY-row blocks down z (as tile2d_step_kernel).  Per block the
// producer loads ONE stage: the P^k box (TX+16) x (TY+4r) rows and the grown
// (P^{k-1}, K) boxes (TX+8) x (TY+2r); stage-A warps compute P^{k+1} on the
// grown block into a shared P1 tile (interior rows to C), stage-B warps
// compute P^{k+2} on the block from it (to D), one block behind.  Blocks are
// self-contained (their z halo rows come with the box), so the P1 ring only
// decouples A from B.  20 B per point per launch = 10 B per update.
template <int R_, int TX_, int TY_, int NYA_, int NYB_, int NS_, int N1_, int MINB_ = 1>
struct CfgWS2 {
    static constexpr int R = R_, TX = TX_, TY = TY_, NYA = NYA_, NYB = NYB_, NS = NS_, N1 = N1_, MINB = MINB_;
    static constexpr int BX0 = TX + 16, BY0 = TY + 4 * R;         // P^k block (x halo 8, z halo 2r)
    static constexpr int BXE = TX + 8, BYE = TY + 2 * R;          // grown block E
    static constexpr int QXE = BXE / 4, QXI = TX / 4;
    static constexpr int NTA = QXE * (BYE / NYA), NTB = QXI * (TY / NYB);
    static constexpr int NWA = (NTA + 31) / 32, NWB = (NTB + 31) / 32;
    static constexpr int NTHREADS = 32 * (NWA + NWB + 1);
    static constexpr int P0F = (BX0 * BY0 + 31) / 32 * 32;
    static constexpr int EF = (BXE * BYE + 31) / 32 * 32;
    static constexpr int STAGE = P0F + 2 * EF;                    // [P^k | P^{k-1} | K]
    static constexpr uint32_t STAGE_BYTES = (BX0 * BY0 + 2 * BXE * BYE) * 4;
    static constexpr int SMEM_BYTES = (NS * STAGE + N1 * EF) * 4 + (2 * NS + 2 * N1) * 8 + 16;
    static constexpr int NY = NYB, DP = NS, DA = N1;
    static_assert(BYE % NYA == 0 && TY % NYB == 0, "tile");
    static_assert(BX0 <= 256 && BY0 <= 256 && R <= 4, "TMA box");
};

template <class C, bool SP, bool PEER, bool KZ>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
tb2d_step_kernel(const __grid_constant__ CUtensorMap map_p0,   // P^k buffer, box (BX0, 1, BY0)
                 const __grid_constant__ CUtensorMap map_pm,   // P^{k-1} buffer, box (BXE, 1, BYE)
                 const __grid_constant__ CUtensorMap map_k,    // K, box (BXE, 1, BYE)
                 const StepParams prm) {
    constexpr int R = C::R;
    extern __shared__ __align__(128) float smem[];
    float *sSt = smem;
    float *sP1 = smem + C::NS * C::STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sP1 + C::N1 * C::EF);
    uint64_t *fullS = bars, *emptyS = fullS + C::NS, *full1 = emptyS + C::NS, *empty1 = full1 + C::N1;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr bool anyp = PEER;                          // in-kernel halo pushes (boundary launches)
    // Work: blocks v = column * nb + block row, taken in order.  Chunked mode
    // (prm.lin == 0): unit = chunk * ntx + column, a z-range of one column.
    // Linear mode (prm.lin = G units, one wave): unit u takes the contiguous
    // range [V u / G, V (u+1) / G) of the V = ntx * nb blocks, crossing column
    // boundaries -- balanced to one block, one pipeline warm-up per CTA (blocks
    // are self-contained: their z halo rows come with the box).
    const int unit = blockIdx.x;
    const int span = prm.zhi - prm.zlo;
    const int nb = (span + C::TY - 1) / C::TY;
    int v0, v1;
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
        for (int i = 0; i < C::NS; ++i) { mbar_init(&fullS[i], 1); mbar_init(&emptyS[i], kArrivalsPerWarp * (C::NWA + C::NWB)); }
        for (int i = 0; i < C::N1; ++i) { mbar_init(&full1[i], kArrivalsPerWarp * C::NWA); mbar_init(&empty1[i], kArrivalsPerWarp * C::NWB); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_sync();
    if (v1 <= v0) return;
    const int nload = v1 - v0;
    // receiver i belongs to block v (receivers are sorted by (unit, v, z))
    auto rec_block = [&](int i) { return (prm.rec.x[i] / C::TX) * nb + (prm.rec.z[i] - prm.zlo) / C::TY; };
    const int nx = (int)prm.nx;
    const int64_t kk = step_index(prm);
    constexpr float c0 = tap(R, 0);
    int rp = prm.rec.off ? prm.rec.off[unit] : 0;
    const int rend = prm.rec.off ? prm.rec.off[unit + 1] : 0;

    if (warp == C::NWA + C::NWB) {
        if (lane == 0) {
            tma_prefetch_desc(&map_p0); tma_prefetch_desc(&map_pm); tma_prefetch_desc(&map_k);
            for (int l = 0; l < nload; ++l) {
                const int v = v0 + l, colu = v / nb;
                const int s = l % C::NS, rb = prm.zlo + (v - colu * nb) * C::TY, x0 = colu * C::TX;
                mbar_wait_producer(&emptyS[s], ((l / C::NS) & 1) ^ 1);
                mbar_expect_tx(&fullS[s], C::STAGE_BYTES - (KZ ? C::BXE * C::BYE * 4 : 0));
                float *st = sSt + s * C::STAGE;
                tma_load_3d(st, &map_p0, &fullS[s], x0 - 8, 0, rb - 2 * R + halo_planes(R));        // rows rb-2r.. (+r halo)
                tma_load_3d(st + C::P0F, &map_pm, &fullS[s], x0 - 4, 0, rb - R + halo_planes(R));   // rows rb-r..
                if constexpr (!KZ)
                    tma_load_3d(st + C::P0F + C::EF, &map_k, &fullS[s], x0 - 4, 0, rb);   // K halo buffer: rows rb - r ..
            }
        }
        return;
    }

    if (warp < C::NWA) {
        // ---------------------------------------------------------------- stage A
        const bool act = tid < C::NTA;
        const int q = act ? tid % C::QXE : 0, re0 = act ? (tid / C::QXE) * C::NYA : 0;
        const bool qint = q >= 1 && q <= C::QXI;
        // per-column state (recomputed when the block moves to another column)
        int colc = -1, x0 = 0, xb = 0;
        bool inx[4];
        float sgx[4];                                  // sponge factors (SP only)
        uint32_t smask = 0;
        float *const trow = trace_row_of(prm, kk);
        const float *const wv = w_next_of(prm, kk);
        for (int l = 0; l < nload; ++l) {
            const int s = l % C::NS, s1 = l % C::N1;
            const int v = v0 + l, colu = v / nb;
            const int rb = prm.zlo + (v - colu * nb) * C::TY;
            if (colu != colc) {
                colc = colu;
                x0 = colu * C::TX;
                xb = x0 - 4 + 4 * q;
#pragma unroll
                for (int e = 0; e < 4; ++e) inx[e] = (xb + e >= R) && (xb + e < nx - R);
#pragma unroll
                for (int e = 0; e < 4; ++e) sgx[e] = SP ? sponge_gx(prm, xb + e) : 1.f;
                smask = 0;
                for (int s2 = 0; s2 < prm.nsrc; ++s2)
                    if (act && prm.sx[s2] >= xb && prm.sx[s2] < xb + 4) smask |= 1u << s2;
            }
            mbar_wait(&fullS[s], (l / C::NS) & 1);
            mbar_wait(&empty1[s1], ((l / C::N1) & 1) ^ 1);
            const float *tp = sSt + s * C::STAGE, *tpm = tp + C::P0F, *tk = tpm + C::EF;
            float *t1 = sP1 + s1 * C::EF;
            float4 oraw[C::NYA];                                   // raw P^{k+1} (receivers)
#pragma unroll
            for (int yy = 0; yy < C::NYA; ++yy) oraw[yy] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (act) {
                float4 col[C::NYA + 2 * R];
#pragma unroll
                for (int i = 0; i < C::NYA + 2 * R; ++i) col[i] = lds128(tp + (re0 + i) * C::BX0 + 4 * q + 4);
#pragma unroll
                for (int yy = 0; yy < C::NYA; ++yy) {
                    const int re = re0 + yy, z = rb - R + re;
                    const float *row = tp + (re + R) * C::BX0 + 4 * q;
                    const float4 L4 = lds128(row), M4 = col[yy + R], R4 = lds128(row + 8);
                    const float av[12] = {L4.x, L4.y, L4.z, L4.w, M4.x, M4.y, M4.z, M4.w, R4.x, R4.y, R4.z, R4.w};
                    const int offe = re * C::BXE + 4 * q;
                    const float4 pm4 = lds128(tpm + offe), k4 = KZ ? splat4(kplane(prm, z)) : lds128(tk + offe);
                    const int gz = (int)prm.gz0 + z;
                    const bool inz = (gz >= R) && (gz < (int)prm.nzg - R);
                    float4 o;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float pc = av[4 + e];
                        float sx = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m) sx = __fmaf_rn(tap(R, m), __fadd_rn(av[4 + e - m], av[4 + e + m]), sx);
                        float S = inx[e] ? sx : 0.f;
                        float szz = __fmul_rn(c0, pc);
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            szz = __fmaf_rn(tap(R, m), __fadd_rn(f4(col[yy + R - m], e), f4(col[yy + R + m], e)), szz);
                        S = inz ? __fadd_rn(S, szz) : S;
                        f4set(o, e, time_update<SP>(f4(k4, e), S, pc, f4(pm4, e), SP ? sponge_gz(prm, gz) : 1.f,
                                                    1.f, sgx[e]));
                    }
                    const bool interior = qint && re >= R && re < R + C::TY && z < prm.zhi;
                    oraw[yy] = o;
                    if (smask) {                                       // w_{k+1} wherever in E
                        for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                            if (!((smask >> s2) & 1u) || prm.sz[s2] != z) continue;
                            const int dx = prm.sx[s2] - xb;
                            f4set(o, dx, __fadd_rn(f4(o, dx), wv[s2]));
                        }
                    }
                    *reinterpret_cast<float4 *>(t1 + offe) = o;
                    if (interior && xb < (int)prm.pitch) {
                        *reinterpret_cast<float4 *>(prm.pnext + (int64_t)(z + halo_planes(R)) * prm.pitch + xb) = o;
                        if (anyp) peer_store4<R>(prm.peer1, z, (int)prm.nz, prm.pitch, xb, o);
                    }
                }
            }
            if (rp < rend && rec_block(rp) == v)                      // owners: block-interior A threads
                rp = warp_record<C::NYA>(oraw, prm.rec.z, prm.rec.id, rp, rend, rb, rb + C::TY, trow,
                                         [&](int i, int &ln, int &yy, int &e) {
                                             const int re = prm.rec.z[i] - (rb - R), dx = prm.rec.x[i] - (x0 - 4);
                                             const int t = (re / C::NYA) * C::QXE + dx / 4;
                                             if ((t >> 5) != warp) return false;
                                             ln = t & 31; yy = re % C::NYA; e = dx & 3;
                                             return true;
                                         }, prm.rec.x, x0, x0 + C::TX);
            role_release(&full1[s1], &emptyS[s]);
        }
        return;
    }

    // -------------------------------------------------------------------- stage B
    const int tb = tid - 32 * C::NWA;
    const bool act = tb < C::NTB;
    const int qi = act ? tb % C::QXI : 0, ri0 = act ? (tb / C::QXI) * C::NYB : 0;
    const int q = qi + 1;
    int colc = -1, x0 = 0, xb = 0;                     // per-column state
    bool inx[4];
    float sgx[4];                                      // sponge factors (SP only)
    uint32_t smask = 0;
    float *const trow = trace_row_of(prm, kk + 1);
    const float *const wv = w_next_of(prm, kk + 1);
    for (int l = 0; l < nload; ++l) {
        const int s = l % C::NS, s1 = l % C::N1;
        const int v = v0 + l, colu = v / nb;
        const int rb = prm.zlo + (v - colu * nb) * C::TY;
        if (colu != colc) {
            colc = colu;
            x0 = colu * C::TX;
            xb = x0 + 4 * qi;
#pragma unroll
            for (int e = 0; e < 4; ++e) inx[e] = (xb + e >= R) && (xb + e < nx - R);
#pragma unroll
            for (int e = 0; e < 4; ++e) sgx[e] = SP ? sponge_gx(prm, xb + e) : 1.f;
            smask = 0;
            for (int s2 = 0; s2 < prm.nsrc; ++s2)
                if (act && prm.sx[s2] >= xb && prm.sx[s2] < xb + 4) smask |= 1u << s2;
        }
        mbar_wait(&full1[s1], (l / C::N1) & 1);
        const float *tp = sSt + s * C::STAGE, *tk = tp + C::P0F + C::EF;
        const float *t1 = sP1 + s1 * C::EF;
        const int zt = rb + ri0;
        float4 out[C::NYB];
        if (act) {
            float4 col[C::NYB + 2 * R];
#pragma unroll
            for (int i = 0; i < C::NYB + 2 * R; ++i) col[i] = lds128(t1 + (ri0 + i) * C::BXE + 4 * q);
#pragma unroll
            for (int yy = 0; yy < C::NYB; ++yy) {
                const int re = ri0 + yy + R;
                const int offe = re * C::BXE + 4 * q;
                const float4 L4 = lds128(t1 + offe - 4), M4 = col[yy + R], R4 = lds128(t1 + offe + 4);
                const float av[12] = {L4.x, L4.y, L4.z, L4.w, M4.x, M4.y, M4.z, M4.w, R4.x, R4.y, R4.z, R4.w};
                const float4 pk4 = lds128(tp + (re + R) * C::BX0 + 4 * q + 4);
                const float4 k4 = KZ ? splat4(kplane(prm, zt + yy)) : lds128(tk + offe);
                const int gz = (int)prm.gz0 + zt + yy;
                const bool inz = (gz >= R) && (gz < (int)prm.nzg - R);
                const float sgz = SP ? sponge_gz(prm, gz) : 1.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float pc = av[4 + e];
                    float sx = __fmul_rn(c0, pc);
#pragma unroll
                    for (int m = 1; m <= R; ++m) sx = __fmaf_rn(tap(R, m), __fadd_rn(av[4 + e - m], av[4 + e + m]), sx);
                    float S = inx[e] ? sx : 0.f;
                    float szz = __fmul_rn(c0, pc);
#pragma unroll
                    for (int m = 1; m <= R; ++m)
                        szz = __fmaf_rn(tap(R, m), __fadd_rn(f4(col[yy + R - m], e), f4(col[yy + R + m], e)), szz);
                    S = inz ? __fadd_rn(S, szz) : S;
                    f4set(out[yy], e, time_update<SP>(f4(k4, e), S, pc, f4(pk4, e), sgz, 1.f, sgx[e]));
                }
            }
        }
        role_release(&empty1[s1], &emptyS[s]);
        if (rp < rend && rec_block(rp) == v)                          // owners: B threads
            rp = warp_record<C::NYB>(out, prm.rec.z, prm.rec.id, rp, rend, rb, rb + C::TY, trow,
                                     [&](int i, int &ln, int &yy, int &e) {
                                         const int dz = prm.rec.z[i] - rb, dx = prm.rec.x[i] - x0;
                                         const int t = (dz / C::NYB) * C::QXI + dx / 4;
                                         if (C::NWA + (t >> 5) != warp) return false;
                                         ln = t & 31; yy = dz % C::NYB; e = dx & 3;
                                         return true;
                                     }, prm.rec.x, x0, x0 + C::TX);
        if (!act) continue;
        if (smask) {
            for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                if (!((smask >> s2) & 1u)) continue;
                const int dz = prm.sz[s2] - zt, dx = prm.sx[s2] - xb;
                if (dz < 0 || dz >= C::NYB) continue;
#pragma unroll
                for (int yy = 0; yy < C::NYB; ++yy)
                    if (yy == dz) {
                        const float v = f4(out[yy], dx);
                        prm.src_raw[s2] = v;
                        f4set(out[yy], dx, __fadd_rn(v, wv[s2]));
                    }
            }
        }
        if (xb < (int)prm.pitch) {
            float *dst = prm.pnext2 + (int64_t)(zt + halo_planes(R)) * prm.pitch + xb;
#pragma unroll
            for (int yy = 0; yy < C::NYB; ++yy)
                if (zt + yy < prm.zhi) *reinterpret_cast<float4 *>(dst + (int64_t)yy * prm.pitch) = out[yy];
            if (PEER) {
#pragma unroll
                for (int yy = 0; yy < C::NYB; ++yy)
                    if (zt + yy < prm.zhi)
                        peer_store4<R>(prm.peer2, zt + yy, (int)prm.nz, prm.pitch, xb, out[yy]);
            }
        }
    }
}

}  // namespace fdk
