// fd_tab_tb2ws.cu -- two-steps-per-pass (temporal blocking) tiles, 3D
// (fd_tb2.cuh; see fd_tables.cuh).  Presented as TileCfg so the chunking /
// receiver code is shared: pbw/pbz hold the P^k box (BX0, BY0), tbw/tbz the
// grown-tile box (BXE, BYE).
#define FD_TABLE_TU
#include "fd_tb2.cuh"
#include "fd_tables.cuh"

FD_LAUNCHER(launch_tb2ws, tb2ws_step_kernel)

template <int R, int TX, int TY, int NYA, int NYB, int DP, int DA, int D1, int MINB = 1, bool FULL = false>
static TileCfg make_tb2ws() {
    using C = CfgWS<R, TX, TY, NYA, NYB, DP, DA, D1, MINB>;
    TileCfg t{3, R, TX, TY, NYB, DP, DA, C::BX0, C::BXE, C::BY0, C::BYE, C::NTHREADS, C::SMEM_BYTES, {}, {}};
    FD_VARIANTS(t, C, FULL, tb2ws_step_kernel, launch_tb2ws);
    return t;
}

std::vector<TileCfg> fdtab::tb2ws() {
    return {
        // 3D r=1, r04 sweep (C3 order 2, scripts/tune.py --tsteps 2): one
        // 128 x 16 CTA per SM with 6-slot P^k / 5-slot aux rings 581-584 Gpts/s;
        // the r03 choice (64 x 16, two CTAs per SM, 5/4 slots) 518; 64 x 16 with
        // 6/5 slots 542; 128 x 16 with 5/4 slots 534; more stage-B warps
        // (NYB = 2) 481-551.  r05 (after the instruction cuts): 7-slot P^k ring
        // 605 vs 602 (6 slots) -- the default
        make_tb2ws<1, 128, 16, 2, 4, 4, 3, 2, 1, true>(), make_tb2ws<1, 128, 16, 2, 4, 3, 3, 2, 1>(),
        make_tb2ws<1, 128, 16, 2, 4, 3, 3, 3, 1>(), make_tb2ws<1, 64, 16, 2, 4, 3, 3, 1, 2>(),
        make_tb2ws<1, 64, 16, 2, 4, 2, 2, 2, 2>(), make_tb2ws<1, 128, 8, 2, 2, 2, 2, 2, 2>(),
        // 3D r=2 (order 4 stays on single steps by default: 421 vs <= 320 Gpts/s in r03)
        make_tb2ws<2, 64, 16, 4, 4, 1, 1, 1, 1, true>(), make_tb2ws<2, 64, 16, 2, 4, 1, 1, 1, 2>(),
        make_tb2ws<2, 64, 16, 2, 4, 3, 3, 2, 1>(), make_tb2ws<2, 128, 8, 2, 2, 3, 3, 2, 1>(),
        make_tb2ws<2, 64, 16, 2, 4, 2, 2, 2, 1>(),
        // r05 role-balance sweep (3D r=1, 128 x 16): stage-A rows per thread
        // NYA / stage-B rows NYB -> warps 7+4, 10+8, 7+8, 4+4
        make_tb2ws<1, 128, 16, 3, 4, 3, 3, 2, 1>(), make_tb2ws<1, 128, 16, 2, 2, 3, 3, 2, 1>(),
        make_tb2ws<1, 128, 16, 3, 2, 3, 3, 2, 1>(), make_tb2ws<1, 128, 16, 6, 4, 3, 3, 2, 1>(),
        // r2: 3D r = 3, 4 (orders 6, 8), tuning-only (FD_OPT_TSTEPS=2): 64 x 16
        // tiles, stage A on the 72 x (16 + 2r) grown tile (1.6-1.7x the points)
        make_tb2ws<3, 64, 16, 2, 2, 1, 1, 1>(), make_tb2ws<4, 64, 16, 2, 2, 0, 0, 0>(),
        make_tb2ws<4, 64, 16, 1, 2, 0, 0, 0>(),
        // r2: 3D r = 2 on 128 x 16 tiles (stage A recomputes 1.33x instead of
        // 1.41x): C3 order 4 415.7 vs 419 single-step, C4 428.4 vs 421.4 --
        // a wash; order 4 keeps single steps by default
        make_tb2ws<2, 128, 16, 2, 4, 2, 1, 1, 1>()};
}
