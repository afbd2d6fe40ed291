// fd_tables.cuh -- compiled configurations of the tiled step kernels.
//
// Each tiled kernel (fused_step_kernel, tile2d_step_kernel, tb2ws_step_kernel,
// tb2d_step_kernel) is a template over its tile configuration and three
// switches, compiled as variant v = SP | 2 * PEER | 4 * KZ:
//   SP   the absorbing sponge frame (R#18),
//   PEER the in-kernel halo pushes of the peer transport (section 7),
//   KZ   K read from the per-plane table instead of the K field
//        (FD_OPT_KPLANE, section 5.10; exact: the same fp32 K values).
// Tuning-only entries carry variant 0 alone; the configurations the auto
// policy picks ("full") carry all eight.  The tables are split over several
// translation units (fd_tab_*.cu) so nvcc compiles them in parallel.
#pragma once
#include <vector>

#include "fd_kernels.cuh"

using namespace fdk;

typedef void (*launch_fused_t)(dim3, int, cudaStream_t, const CUtensorMap &, const CUtensorMap &,
                               const CUtensorMap &, const StepParams &, bool pdl);

constexpr int kVariants = 8;
enum { kVarSponge = 1, kVarPeer = 2, kVarKPlane = 4 };

struct TileCfg {
    int ndim, r, tx, ty, ny, dp, dk;
    int pbw, tbw;        // TMA box widths (halo'd p row piece, p_prev/K row piece)
    int pbz, tbz;        // TMA box depths in z (2D row blocks; 1 in 3D)
    int threads, smem;
    const void *kernel[kVariants];
    launch_fused_t launch[kVariants];
    int steps = 2;       // time steps per launch (temporal-blocking table: 2, or S of tbs2d / rs2d)
    int kind = 0;        // 0: TMA-staged tiles; 1: register-streamed 2D strips (rs2d_step_kernel, no
                         // shared memory; tx = own columns per strip, ty = 1, ny = warps per CTA)
    bool full() const { return kernel[kVariants - 1] != nullptr; }
};

namespace fdtab {
std::vector<TileCfg> tiles3d_r12();   // fused_step_kernel, r = 1, 2   (fd_tab_3d12.cu)
std::vector<TileCfg> tiles3d_r34();   // fused_step_kernel, r = 3, 4   (fd_tab_3d34.cu)
std::vector<TileCfg> tiles2d();       // tile2d_step_kernel           (fd_tab_2d.cu)
std::vector<TileCfg> tb2ws();         // tb2ws_step_kernel, 3D r <= 2  (fd_tab_tb2ws.cu)
std::vector<TileCfg> tb2d();          // tb2d_step_kernel, 2D          (fd_tab_tb2d.cu)
std::vector<TileCfg> tbs2d();         // tbs2d_step_kernel, 2D, S >= 3 (fd_tab_tbs.cu)
std::vector<TileCfg> rs2d();          // rs2d_step_kernel, 2D, defaults (fd_tab_rs2d.cu)
std::vector<TileCfg> rs2d_x();        // rs2d_step_kernel, 2D, tuning   (fd_tab_rs2d_x.cu)
}  // namespace fdtab

#ifdef FD_TABLE_TU
// pdl: launch with programmatic stream serialization (the kernels call
// pdl_sync() after their prologue; fd_kernels.cuh)
#define FD_LAUNCHER(NAME, KERNEL)                                                                            \
    template <class C, int V>                                                                                \
    static void NAME(dim3 grid, int smem, cudaStream_t st, const CUtensorMap &a, const CUtensorMap &b,       \
                     const CUtensorMap &c, const StepParams &p, bool pdl) {                                  \
        if (!pdl) {                                                                                          \
            KERNEL<C, (V & 1) != 0, (V & 2) != 0, (V & 4) != 0><<<grid, C::NTHREADS, smem, st>>>(a, b, c, p); \
            return;                                                                                          \
        }                                                                                                    \
        cudaLaunchConfig_t cfg = {};                                                                         \
        cudaLaunchAttribute at[1];                                                                           \
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                       \
        at[0].val.programmaticStreamSerializationAllowed = 1;                                                \
        cfg.gridDim = grid; cfg.blockDim = dim3(C::NTHREADS); cfg.dynamicSmemBytes = (size_t)smem;           \
        cfg.stream = st; cfg.attrs = at; cfg.numAttrs = 1;                                                   \
        cudaLaunchKernelEx(&cfg, KERNEL<C, (V & 1) != 0, (V & 2) != 0, (V & 4) != 0>, a, b, c, p);           \
    }

#define FD_VARIANT(T, C, KERNEL, LAUNCH, V)                                                                  \
    do {                                                                                                     \
        T.kernel[V] = (const void *)KERNEL<C, ((V) & 1) != 0, ((V) & 2) != 0, ((V) & 4) != 0>;               \
        T.launch[V] = LAUNCH<C, V>;                                                                          \
    } while (0)
#define FD_VARIANTS(T, C, FULL, KERNEL, LAUNCH)                                                              \
    do {                                                                                                     \
        FD_VARIANT(T, C, KERNEL, LAUNCH, 0);                                                                 \
        if constexpr (FULL) {                                                                                \
            FD_VARIANT(T, C, KERNEL, LAUNCH, 1);                                                             \
            FD_VARIANT(T, C, KERNEL, LAUNCH, 2);                                                             \
            FD_VARIANT(T, C, KERNEL, LAUNCH, 3);                                                             \
            FD_VARIANT(T, C, KERNEL, LAUNCH, 4);                                                             \
            FD_VARIANT(T, C, KERNEL, LAUNCH, 5);                                                             \
            FD_VARIANT(T, C, KERNEL, LAUNCH, 6);                                                             \
            FD_VARIANT(T, C, KERNEL, LAUNCH, 7);                                                             \
        }                                                                                                    \
    } while (0)
#endif
