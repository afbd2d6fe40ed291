// fd_tab_rs2d.cu -- register-streamed S-steps-per-pass strips, 2D
// (fd_rs2d.cuh; see fd_tables.cuh).  tx = own columns per strip, ty = 1 (the
// chunk split is by rows), ny = warps per CTA, dp = rows in flight per warp
// (cp.async ring), dk = rows per unrolled loop body; TMA boxes of one 128-float row piece (pbw / tbw 128, pbz / tbz 1).
#define FD_TABLE_TU
#include "fd_rs2d.cuh"
#include "fd_tables.cuh"

FD_LAUNCHER(launch_rs2d, rs2d_step_kernel)

template <int R, int S, int HQ, int W, int Q, int MINB = 1, bool FULL = false, bool TMA = true>
static TileCfg make_rs2d() {
    using C = CfgRS2<R, S, HQ, W, Q, MINB, TMA>;
    TileCfg t{2, R, C::TX, 1, W, Q, C::U, 128, 128, 1, 1, C::NTHREADS, C::SMEM_BYTES, {}, {}};
    FD_VARIANTS(t, C, FULL, rs2d_step_kernel, launch_rs2d);
    t.steps = S;
    t.kind = 1;
    return t;
}

std::vector<TileCfg> fdtab::rs2d() {
    return {
        // three / four steps per pass (single slab, band rule, K field or
        // per-plane K): the 2D defaults are the first entry of each (r, S) --
        // r3 on C2 with work stealing: order 2 S = 4 723 Gpts/s (S = 3 681),
        // order 4 S = 3 622 (two-step tb2d: 562 / 500); cp.async rows beat TMA
        // rows here (S = 4: 723 vs 629); 4 warps per CTA, 16 rows in flight
        // per warp, 2 CTAs per SM
        make_rs2d<1, 4, 1, 4, 16, 2, true, false>(), make_rs2d<1, 4, 1, 4, 16, 2>(),
        make_rs2d<1, 3, 1, 4, 16, 2, true, false>(), make_rs2d<1, 3, 1, 4, 16, 2>(),
        make_rs2d<2, 3, 2, 4, 16, 2, true, false>(), make_rs2d<2, 3, 2, 4, 16, 2>(),
        make_rs2d<2, 4, 2, 4, 16, 2, false, false>(),
        // two steps per pass (tuning-only behind tb2d: C2 order 2 478 vs 562)
        make_rs2d<1, 2, 1, 4, 16, 2, true>(), make_rs2d<1, 2, 1, 4, 16, 2, false, false>(),
        make_rs2d<2, 2, 1, 4, 16, 2, true>(),
        make_rs2d<3, 2, 2, 4, 8, 4, true>(),
        make_rs2d<4, 2, 2, 4, 8, 4, true>()};
}
