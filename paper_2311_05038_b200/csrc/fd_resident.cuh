// fd_resident.cuh -- the whole run of one fd_step(n) call in ONE launch of one
// thread-block cluster, for grids small enough to live in the cluster's
// shared memory ("C1-size grids: a whole run in one cluster
// with DSMEM and cluster barriers").
//
// Why: at C1 (256 x 256) a step moves 1 MB, ~0.15 us at HBM speed, but a
// launch (even replayed from a CUDA graph) costs ~3.5 us: the run is
// launch-bound.  Here the NC CTAs of one cluster (8 portable / 16 non-portable)
// each hold a z-slab of planes of p, p_prev and K in shared memory for all n
// steps; per step each CTA
//   1. computes P^{k+1} on its planes (the canonical fp32 expression of
//      fd_kernels.cuh, so results are bitwise those of every other kernel),
//      writing it over p_prev in place, and PUSHES its r boundary planes into
//      the neighbouring CTAs' halo planes of the same buffer (DSMEM stores,
//      st.shared::cluster through cluster.map_shared_rank);
//   2. after __syncthreads: records its receivers (raw P^{k+1}), then the
//      sources' w_{k+1} in registration order (eager injection, including the
//      pushed copy when the source sits on a boundary plane);
//   3. cluster.sync() (barrier.cluster arrive.release / wait.acquire): every
//      CTA's P^{k+1} and pushed halos are complete and visible.
// Buffer hazards: step k reads the halo planes of the CUR buffer and the
// pushes of step k write the halo planes of the other buffer, so one cluster
// barrier per step suffices.  HBM sees the fields twice per fd_step call (load
// at the start, store at the end) plus the trace rows.
#pragma once
#include <cooperative_groups.h>

#include "fd_kernels.cuh"

namespace fdk {

struct ResidentArgs {
    const float *in_cur, *in_prev;   // field buffers (halo_planes(r) halo planes) at the start
    float *out_cur, *out_prev;       // where the final P and P_prev go (may alias the inputs)
    int32_t nsteps;                  // steps of this launch
    int32_t npmax;                   // max planes per CTA (shared-memory layout)
    const int32_t *rec;              // receivers sorted by CTA: z, y, x, id arrays of nrec, then off[NC+1]
    int32_t nrec;
};

template <int R, int NDIM>
__global__ void __launch_bounds__(1024, 1) resident_kernel(const StepParams prm, const ResidentArgs ra) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int nc = (int)cl.num_blocks(), c = (int)cl.block_rank();
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int nz = (int)prm.nz, ny = (int)prm.ny, nx = (int)prm.nx, pitch = (int)prm.pitch;
    const int PS = ny * nx;                                       // floats per plane (compact rows)
    const int pz0 = (int)((int64_t)nz * c / nc), pz1 = (int)((int64_t)nz * (c + 1) / nc), np = pz1 - pz0;
    const int nplo = c > 0 ? pz0 - (int)((int64_t)nz * (c - 1) / nc) : 0;   // planes of CTA c - 1
    extern __shared__ __align__(16) float sm[];
    const int BUF = (ra.npmax + 2 * R) * PS;
    float *const B0 = sm, *const B1 = sm + BUF, *const Ks = sm + 2 * BUF;
    constexpr float c0 = tap(R, 0);
    // The CTA's np * PS points are swept flat with stride nthr.  A thread's
    // point (z, y, x) advances by the fixed (dz, dy, dx) per iteration, so no
    // division happens in the loops.
    struct Pt { int z, y, x; };
    const int W = np * PS;
    Pt t0;
    t0.z = tid / PS;
    t0.y = (tid - t0.z * PS) / nx;
    t0.x = tid - t0.z * PS - t0.y * nx;
    const int dz = nthr / PS, dyy = (nthr - dz * PS) / nx, dxx = nthr - dz * PS - dyy * nx;
    auto advance = [&](Pt &p) {
        p.x += dxx; p.y += dyy; p.z += dz;
        if (p.x >= nx) { p.x -= nx; ++p.y; }
        if (p.y >= ny) { p.y -= ny; ++p.z; }
    };

    // load own planes (plane z at buffer plane z + r); zero the halo planes
    // that face the global z faces (never read: the z band skips them)
    {
        Pt p = t0;
        for (int idx = tid; idx < W; idx += nthr, advance(p)) {
            const int i = p.y * nx + p.x;
            const int64_t g = ((int64_t)(pz0 + p.z + halo_planes(R)) * ny + p.y) * pitch + p.x;
            B0[(p.z + R) * PS + i] = ra.in_cur[g];
            B1[(p.z + R) * PS + i] = ra.in_prev[g];
            Ks[p.z * PS + i] = prm.K[((int64_t)(pz0 + p.z) * ny + p.y) * pitch + p.x];
        }
    }
    for (int i = tid; i < R * PS; i += nthr) {
        if (c == 0) { B0[i] = 0.f; B1[i] = 0.f; }
        if (c == nc - 1) { B0[(np + R) * PS + i] = 0.f; B1[(np + R) * PS + i] = 0.f; }
    }
    cl.sync();
    // initial halos of P: pull the neighbours' boundary planes once
    if (c > 0) {
        const float *lo = cl.map_shared_rank(B0, c - 1);
        for (int i = tid; i < R * PS; i += nthr) B0[i] = lo[nplo * PS + i];        // its planes nplo-r .. nplo-1
    }
    if (c < nc - 1) {
        const float *hi = cl.map_shared_rank(B0, c + 1);
        for (int i = tid; i < R * PS; i += nthr) B0[(np + R) * PS + i] = hi[R * PS + i];   // its planes 0 .. r-1
    }
    __syncthreads();

    const int rb = ra.rec ? ra.rec[4 * ra.nrec + c] : 0, re = ra.rec ? ra.rec[4 * ra.nrec + c + 1] : 0;
    bool own_src = false;
    for (int s2 = 0; s2 < prm.nsrc; ++s2) own_src |= prm.sz[s2] >= pz0 && prm.sz[s2] < pz1;
    float *P = B0, *Q = B1;
    for (int s = 0; s < ra.nsteps; ++s) {
        const int64_t k = prm.k + s;
        // Q (p_prev) becomes P^{k+1}; the neighbours' Q halos receive our
        // boundary planes: our plane z is plane nplo + z of CTA c - 1 (its
        // buffer plane nplo + z + r, an upper halo plane when z < r) and plane
        // z - np of CTA c + 1 (buffer plane z - np + r)
        float *const qlo = c > 0 ? cl.map_shared_rank(Q, c - 1) : nullptr;
        float *const qhi = c < nc - 1 ? cl.map_shared_rank(Q, c + 1) : nullptr;
        const float *__restrict__ const Pr = P;
        float *__restrict__ const Qr = Q;
        Pt p = t0;
#pragma unroll 4
        for (int idx = tid; idx < W; idx += nthr) {
            const int z = p.z, i = p.y * nx + p.x;
            const int gz = pz0 + z;
            const float *pp = Pr + (z + R) * PS + i;
            const float pc = pp[0];
            float S = 0.f;
            if (p.x >= R && p.x < nx - R) {
                float sx = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m) sx = __fmaf_rn(tap(R, m), __fadd_rn(pp[-m], pp[m]), sx);
                S = sx;
            }
            if (NDIM == 3 && p.y >= R && p.y < ny - R) {
                float sy = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m) sy = __fmaf_rn(tap(R, m), __fadd_rn(pp[-m * nx], pp[m * nx]), sy);
                S = __fadd_rn(S, sy);
            }
            if (gz >= R && gz < (int)prm.nzg - R) {
                float sz = __fmul_rn(c0, pc);
#pragma unroll
                for (int m = 1; m <= R; ++m) sz = __fmaf_rn(tap(R, m), __fadd_rn(pp[-m * PS], pp[m * PS]), sz);
                S = __fadd_rn(S, sz);
            }
            float *const qq = Qr + (z + R) * PS + i;
            const float v = time_update_rt(prm, Ks[z * PS + i], S, pc, qq[0], gz, p.y, p.x);
            qq[0] = v;
            if (z < R && qlo) qlo[(nplo + z + R) * PS + i] = v;
            if (z >= np - R && qhi) qhi[(z - np + R) * PS + i] = v;
            advance(p);
        }
        __syncthreads();
        // receivers: raw P^{k+1}
        float *const trow = trace_row_of(prm, k);
        for (int j = rb + tid; j < re; j += nthr) {
            const int z = ra.rec[j] - pz0, y = ra.rec[ra.nrec + j], x = ra.rec[2 * ra.nrec + j];
            trow[ra.rec[3 * ra.nrec + j]] = Q[(z + R) * PS + y * nx + x];
        }
        if (own_src) {
            // eager injection of w_{k+1}, registration order (after the receivers)
            __syncthreads();
            if (tid == 0) {
                const float *wn = w_next_of(prm, k);
                for (int s2 = 0; s2 < prm.nsrc; ++s2) {
                    const int z = prm.sz[s2] - pz0;
                    if (z < 0 || z >= np) continue;
                    const int i = prm.sy[s2] * nx + prm.sx[s2];
                    const float v = Q[(z + R) * PS + i];
                    prm.src_raw[s2] = v;
                    const float w = __fadd_rn(v, wn[s2]);
                    Q[(z + R) * PS + i] = w;
                    if (z < R && qlo) qlo[(nplo + z + R) * PS + i] = w;
                    if (z >= np - R && qhi) qhi[(z - np + R) * PS + i] = w;
                }
            }
        }
        cl.sync();
        float *const t = P; P = Q; Q = t;
    }
    // store own planes: P -> out_cur, Q -> out_prev
    {
        Pt p = t0;
        for (int idx = tid; idx < W; idx += nthr, advance(p)) {
            const int i = p.y * nx + p.x;
            const int64_t g = ((int64_t)(pz0 + p.z + halo_planes(R)) * ny + p.y) * pitch + p.x;
            ra.out_cur[g] = P[(p.z + R) * PS + i];
            ra.out_prev[g] = Q[(p.z + R) * PS + i];
        }
    }
}

}  // namespace fdk
