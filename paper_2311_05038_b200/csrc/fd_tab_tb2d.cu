// fd_tab_tb2d.cu -- two-steps-per-pass (temporal blocking) tiles, 2D
// (fd_tb2.cuh; see fd_tables.cuh).
#define FD_TABLE_TU
#include "fd_tb2.cuh"
#include "fd_tables.cuh"

FD_LAUNCHER(launch_tb2d, tb2d_step_kernel)

template <int R, int TX, int TY, int NYA, int NYB, int NS, int N1, int MINB = 1, bool FULL = false>
static TileCfg make_tb2d() {
    using C = CfgWS2<R, TX, TY, NYA, NYB, NS, N1, MINB>;
    TileCfg t{2, R, TX, TY, NYB, NS, N1, C::BX0, C::BXE, C::BY0, C::BYE, C::NTHREADS, C::SMEM_BYTES, {}, {}};
    FD_VARIANTS(t, C, FULL, tb2d_step_kernel, launch_tb2d);
    return t;
}

std::vector<TileCfg> fdtab::tb2d() {
    return {
        // 2D: blocks of 32 - 2r rows, so the grown block is 32 rows.  r04 sweep
        // (C2): order 2 554 Gpts/s (3 stages, two CTAs per SM; 518 with 2) vs
        // 400 single-step; order 4 486 vs 397; order 6 391 vs 392; order 8 328 vs 385
        make_tb2d<1, 64, 30, 2, 3, 3, 2, 2, true>(), make_tb2d<1, 64, 30, 2, 3, 2, 2, 2>(),
        make_tb2d<1, 64, 30, 4, 3, 3, 2>(), make_tb2d<1, 64, 30, 4, 2, 3, 2>(),
        // order 4 (r05): 40-row blocks, 2 stages, two CTAs per SM 499 vs 490
        // (28-row blocks, 3 stages: 1.29x vs 1.24x stage-A recomputation)
        make_tb2d<2, 64, 40, 4, 4, 2, 2, 2, true>(), make_tb2d<2, 64, 28, 4, 4, 3, 2, 1>(),
        make_tb2d<2, 64, 28, 4, 2, 3, 2>(),
        make_tb2d<3, 64, 26, 4, 2, 3, 2, 1, true>(), make_tb2d<3, 64, 26, 2, 2, 3, 2>(),
        make_tb2d<4, 64, 24, 4, 4, 3, 2, 1, true>(), make_tb2d<4, 64, 24, 4, 3, 3, 2>(),
        make_tb2d<1, 128, 30, 2, 3, 3, 2, 1>(),
        // r2: 56-column tiles (4096 = 73.1 columns of 56: 74 x 4 chunks = 296
        // CTAs = one wave of two CTAs per SM on C2, vs 64 x 9 = 576 = 1.95 waves)
        make_tb2d<1, 56, 30, 2, 3, 3, 2, 2>(), make_tb2d<1, 56, 30, 2, 2, 3, 2, 2>(),
        make_tb2d<2, 56, 40, 4, 4, 2, 2, 2>(), make_tb2d<2, 56, 40, 4, 2, 2, 2, 2>()};
        // (r2, removed: one CTA per SM with 5-6-stage rings, 4 stages in flight
        // per SM instead of 2 -- C2 order 2 418-436 vs 556 Gpts/s, order 4
        // 281-372 vs 501: 15 warps per SM do not hide the stage latency)
}
