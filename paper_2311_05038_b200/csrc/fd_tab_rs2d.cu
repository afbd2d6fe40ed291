// fd_tab_rs2d.cu -- register-streamed S-steps-per-pass strips, 2D: the
// default configurations (fd_rs2d.cuh; see fd_tables.cuh; tuning entries in
// fd_tab_rs2d_x.cu).  tx = own columns per strip, ty = 1, ny = warps per CTA,
// dp = rows in flight per warp, dk = rows per unrolled loop body; TMA boxes of
// one 128-float row piece (pbw / tbw 128, pbz / tbz 1).
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

std::vector<TileCfg> fdtab::rs2d() {
    return {
        // three / four steps per pass (single slab, band rule, K field or
        // per-plane K); 4 warps per CTA, 16 rows in flight per warp (cp.async
        // rows), 2 CTAs per SM.  r3 on C2 with work stealing: order 2 S = 4
        // 723 Gpts/s (751 with 6-row claims; S = 3 681), order 4 S = 3 622, order 6 S = 3 441
        // (two-step tb2d: 562 / 500, single-step order 6: 390)
        // (stealing granularity per entry: r3 A/B, CfgRS2)
        make_rs2d<1, 4, 1, 4, 16, 2, 1, false, 1, 2>(), make_rs2d<1, 3, 1, 4, 16, 2, 1, false, 1, 2>(),
        make_rs2d<2, 3, 2, 4, 16, 2, 1, false, 2, 1>(),
        // order 6: 3 halo quads per side (104 own columns)
        make_rs2d<3, 3, 3, 4, 16, 2, 1, false, 2, 2>()};   // (1 / 2: 432 vs 441)
}
