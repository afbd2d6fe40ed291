// fd_tab_tbs.cu -- S-steps-per-pass tiles, 2D (fd_tbs.cuh; see fd_tables.cuh).
// Band rule, K field, single slab: variant 0 only.  pbw/pbz: the P^k box
// (BX0, BYP), tbw/tbz: the grown boxes (BXE, BYA); dp/dk: TMA / ring slots.
#define FD_TABLE_TU
#include "fd_tbs.cuh"
#include "fd_tables.cuh"

FD_LAUNCHER(launch_tbs2d, tbs2d_step_kernel)

template <int R, int S, int TX, int TY, int NY, int NS, int NR, int MINB = 1>
static TileCfg make_tbs2d() {
    using C = CfgS2<R, S, TX, TY, NY, NS, NR, MINB>;
    TileCfg t{2, R, TX, TY, NY, NS, NR, C::BX0, C::BXE, C::BYP, C::BYA, C::NTHREADS, C::SMEM_BYTES, {}, {}};
    FD_VARIANT(t, C, tbs2d_step_kernel, launch_tbs2d, 0);
    t.steps = S;
    return t;
}

std::vector<TileCfg> fdtab::tbs2d() {
    return {
        // order 2, three steps per pass: 64 x 30 tiles, 2 rows per thread
        // (stages of 34 / 32 / 30 rows: 10 + 9 + 8 warps), 4-5 TMA slots
        make_tbs2d<1, 3, 64, 30, 2, 5, 3>(), make_tbs2d<1, 3, 64, 30, 2, 4, 3>(),
        // four steps per pass (38 / 36 / 34 / 32 rows... 24-row tiles to fit)
        make_tbs2d<1, 4, 64, 20, 2, 5, 3>(),
        // order 4, three steps: 28-row tiles, 4 rows per thread
        make_tbs2d<2, 3, 64, 28, 4, 4, 3>()};
}
