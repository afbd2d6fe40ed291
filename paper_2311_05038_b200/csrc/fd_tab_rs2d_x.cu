// fd_tab_rs2d_x.cu -- register-streamed 2D strips: tuning entries (and the
// two-step configurations that carry every variant, for the bitwise tests of
// slabs, sponge and peer pushes); defaults in fd_tab_rs2d.cu.
#define FD_TABLE_TU
#include "fd_rs2d.cuh"
#include "fd_tables.cuh"

FD_LAUNCHER(launch_rs2d, rs2d_step_kernel)

// VARS: 0 = the band-rule kernel only, 1 = also the per-plane-K variant (the
// S >= 3 defaults: single-slab contexts never run the sponge / peer
// variants), 2 = all eight variants
template <int R, int S, int HQ, int W, int Q, int MINB, int VARS, bool TMA, int CHK = FD_RS_CHK,
          int SMIN = FD_RS_STEALMIN>
static TileCfg make_rs2d() {
    using C = CfgRS2<R, S, HQ, W, Q, MINB, TMA, CHK, SMIN>;
    TileCfg t{2, R, C::TX, 1, W, Q, C::U, 128, 128, 1, 1, C::NTHREADS, C::SMEM_BYTES, {}, {}};
    if constexpr (VARS == 2) {
        FD_VARIANTS(t, C, true, rs2d_step_kernel, launch_rs2d);
    } else {
        FD_VARIANT(t, C, rs2d_step_kernel, launch_rs2d, 0);
        if constexpr (VARS == 1) FD_VARIANT(t, C, rs2d_step_kernel, launch_rs2d, 4);
    }
    t.steps = S;
    t.kind = 1;
    return t;
}

std::vector<TileCfg> fdtab::rs2d_x() {
    return {
        // TMA rows (one lane, three bulk tensor copies per row): r3 C2 order 2
        // S = 4 629 vs 723 with cp.async rows
        make_rs2d<1, 4, 1, 4, 16, 2, 0, true>(), make_rs2d<1, 3, 1, 4, 16, 2, 0, true>(),
        make_rs2d<2, 3, 2, 4, 16, 2, 0, true>(), make_rs2d<2, 4, 2, 4, 16, 2, 0, false>(),
        // two steps per pass (behind tb2d: C2 order 2 478 vs 562)
        make_rs2d<1, 2, 1, 4, 16, 2, 2, true>(), make_rs2d<1, 2, 1, 4, 16, 2, 0, false>(),
        make_rs2d<2, 2, 1, 4, 16, 2, 2, true>(),
        make_rs2d<3, 2, 2, 4, 8, 4, 0, true>(), make_rs2d<4, 2, 2, 4, 8, 4, 0, true>(),
        // orders 6 / 8, two steps, cp.async rows (r3: 419 / 319)
        make_rs2d<3, 2, 2, 4, 16, 2, 0, false>(), make_rs2d<4, 2, 2, 4, 16, 2, 0, false>(),
        // more warps per SM with shallower rings (12 / 16 warps per SM)
        make_rs2d<1, 4, 1, 4, 12, 3, 0, false>(), make_rs2d<1, 4, 1, 4, 8, 4, 0, false>(),
        make_rs2d<1, 3, 1, 4, 12, 3, 0, false>(), make_rs2d<2, 3, 2, 4, 12, 3, 0, false>()};
}
