// fd_tab_2d.cu -- 2D single-step tiles (see fd_tables.cuh).
#define FD_TABLE_TU
#include "fd_tables.cuh"

FD_LAUNCHER(launch_tile2d, tile2d_step_kernel)

template <int R, int TX, int TY, int NY, int NS, bool FULL = false>
static TileCfg make_cfg2() {
    using C = Cfg2<R, TX, TY, NY, NS>;
    TileCfg t{2, R, TX, TY, NY, NS, 0, C::PBW, C::TBW, C::PBZ, C::TBZ, C::NTHREADS, C::SMEM_BYTES, {}, {}};
    FD_VARIANTS(t, C, FULL, tile2d_step_kernel, launch_tile2d);
    return t;
}

// 2D (tile2d_step_kernel): TX columns x TY-row blocks, NS ring slots.
#define CFG2(R) make_cfg2<R, 128, 32, 4, 3>(), make_cfg2<R, 128, 16, 4, 4>(), \
                make_cfg2<R, 64, 32, 4, 4>(), make_cfg2<R, 128, 64, 8, 2>(), \
                make_cfg2<R, 64, 16, 2, 4>(), make_cfg2<R, 64, 32, 4, 3, true>(), make_cfg2<R, 64, 32, 2, 3>()
std::vector<TileCfg> fdtab::tiles2d() { return {CFG2(1), CFG2(2), CFG2(3), CFG2(4)}; }
