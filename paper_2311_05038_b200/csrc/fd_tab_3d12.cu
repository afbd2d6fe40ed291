// fd_tab_3d12.cu -- 3D single-step tiles, r = 1, 2 (see fd_tables.cuh).
#define FD_TABLE_TU
#include "fd_tables.cuh"

FD_LAUNCHER(launch_fused, fused_step_kernel)

template <int R, int NDIM, int TX, int TY, int NY, int DP, int DK, bool FULL = false>
static TileCfg make_cfg() {
    using C = Cfg<R, NDIM, TX, TY, NY, DP, DK>;
    TileCfg t{NDIM, R, TX, TY, NY, DP, DK, C::PBW, C::TBW, 1, 1, C::NTHREADS, C::SMEM_BYTES, {}, {}};
    FD_VARIANTS(t, C, FULL, fused_step_kernel, launch_fused);
    return t;
}

// Compiled tiles (index = position in tile_table(); FD_OPT_TILE selects one).
// 3D (fused_step_kernel): x-y tiles with rows per thread NY (4 for r <= 2, 2
// or 1 above, to bound the register queue), p-ring prefetch DP, (p_prev, K)
// ring prefetch DK.  scripts/tune.py sweeps them; choose_tile() encodes the
// result (the preferred entry per (ndim, r) is the "full" one).
#define CFG3(R, NY, F1, F2) make_cfg<R, 3, 64, 32, NY, 2, 2>(), make_cfg<R, 3, 128, 32, NY, 2, 2, F2>(), \
                    make_cfg<R, 3, 64, 16, NY, 2, 2>(), make_cfg<R, 3, 128, 16, NY, 2, 2, F1>(), \
                    make_cfg<R, 3, 64, 32, NY, 1, 1>(), make_cfg<R, 3, 32, 32, NY, 2, 2>()
#define CFG3W(R) make_cfg<R, 3, 64, 32, 2, 2, 2>(), make_cfg<R, 3, 32, 32, 2, 2, 2>(), \
                 make_cfg<R, 3, 64, 16, 2, 2, 2, true>(), make_cfg<R, 3, 128, 16, 2, 2, 2>(), \
                 make_cfg<R, 3, 64, 16, 1, 2, 2>(), make_cfg<R, 3, 64, 16, 2, 1, 1>()

std::vector<TileCfg> fdtab::tiles3d_r12() { return {CFG3(1, 4, true, false), CFG3(2, 4, false, true)}; }
