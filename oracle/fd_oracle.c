/*
 * fd_oracle.c -- fp64 CPU oracle for the acoustic finite-difference time step
 * of Hadjigeorgiou et al., "An approach to performance portability through
 * generic programming" (arXiv 2311.05038).
 *
 * *** TEST INFRASTRUCTURE ONLY. ***
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2311_05038_b200/, libfd.so) never calls, links or includes it, and it
 * shares no code, header, table or helper with the CUDA path.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n (both under the
 * paper's reference directory); "R#n" = reading n of DESIGN.md section 3 (the
 * readings taken where the paper is silent).
 *
 * What it computes (Eq. 1, Listing 3, run() body P:154-161):
 *
 *   for k = 0 .. nt-1
 *     add_source : P[idx_s] += amp_s * R(k*dt)      (R#4,R#5)
 *     fd_pzz     : Pzz = d2P/dz2  (band rows = 0)   (R#3)
 *     [fd_pyy]   : Pyy = d2P/dy2  (3D only)          (R#10)
 *     fd_pxx     : Pxx = d2P/dx2  (band cols = 0)
 *     fd_time    : Pnew = 2P - Pold + dt^2 V^2 (Pxx+[Pyy+]Pzz)
 *     swap(Pold,P); swap(P,Pnew)
 *     receivers  : T[j][k] = P[idx_j]                (R#6)
 *
 * All arithmetic is IEEE fp64, evaluated in the written order; the library is
 * compiled with -ffp-contract=off so no FMA contraction changes it.  Each
 * point of each field is an independent expression, so the result does not
 * depend on the OpenMP thread count (used only to time the oracle).
 *
 * Layout (R#11): row-major, slowest axis first: 2D (nz, nx), 3D (nz, ny, nx);
 * x is the fastest axis.  Axis ids used below: 0 = x, 1 = y, 2 = z.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_ARG (-1)
#define ORC_ERR_RANGE (-2)
#define ORC_ERR_NOMEM (-4)

/* ------------------------------------------------------------------------ */
/* Central second-derivative coefficients (R#1, R#2).                        */
/* The standard central-difference weights of order 2r for d2/dx2 on a       */
/* uniform grid (Fornberg 1988, Table 1), written as exact rationals and     */
/* rounded once to fp64.  c[0] is the centre tap, c[m] the tap at +-m.        */
/* S:225-230 fixes symmetry and sum-to-zero; the order is the paper's gap.   */
/* ------------------------------------------------------------------------ */
int oracle_coefficients(int r, double *c)
{
    if (!c) return ORC_ERR_ARG;
    switch (r) {
    case 1:
        c[0] = -2.0;          c[1] = 1.0;
        return ORC_OK;
    case 2:
        c[0] = -5.0 / 2.0;    c[1] = 4.0 / 3.0;   c[2] = -1.0 / 12.0;
        return ORC_OK;
    case 3:
        c[0] = -49.0 / 18.0;  c[1] = 3.0 / 2.0;   c[2] = -3.0 / 20.0;
        c[3] = 1.0 / 90.0;
        return ORC_OK;
    case 4:
        c[0] = -205.0 / 72.0; c[1] = 8.0 / 5.0;   c[2] = -1.0 / 5.0;
        c[3] = 8.0 / 315.0;   c[4] = -1.0 / 560.0;
        return ORC_OK;
    default:
        return ORC_ERR_ARG;
    }
}

/* Stability limit of the leapfrog scheme (R#8): von Neumann analysis of
 * Pnew = 2P - Pold + C^2 * sum_a S(theta_a) P with C = v*dt/h and symbol
 * S(theta) = c0 + 2 sum_m c_m cos(m theta).  Stable iff C^2 * D * |S(pi)| <= 4,
 * i.e. C <= 2 / sqrt(D |S(pi)|).  Reproduces S:338 (2D: 1/sqrt2, sqrt(3/8)). */
double oracle_cfl_max(int ndim, int order)
{
    double c[5];
    int r = order / 2;
    if ((ndim != 2 && ndim != 3) || order % 2 || oracle_coefficients(r, c))
        return -1.0;
    double s_pi = c[0];
    for (int m = 1; m <= r; ++m)
        s_pi += 2.0 * c[m] * ((m % 2) ? -1.0 : 1.0);
    return 2.0 / sqrt((double)ndim * fabs(s_pi));
}

/* Ricker wavelet, the source time function S(t) (R#5):
 * R(t) = (1 - 2 pi^2 f^2 (t-t0)^2) exp(-pi^2 f^2 (t-t0)^2). */
double oracle_ricker(double t, double f, double t0)
{
    const double pi = 3.14159265358979323846;
    double a = pi * pi * f * f * (t - t0) * (t - t0);
    return (1.0 - 2.0 * a) * exp(-a);
}

/* ------------------------------------------------------------------------ */
/* Grid helpers                                                              */
/* ------------------------------------------------------------------------ */
typedef struct {
    int ndim;
    int64_t n[3];      /* extents by axis id: n[0]=nx, n[1]=ny (1 in 2D), n[2]=nz */
    int64_t stride[3]; /* linear stride of one step along each axis */
    int64_t npts;
} grid_t;

static int make_grid(int ndim, const int64_t *dims, grid_t *g)
{
    if (ndim != 2 && ndim != 3) return ORC_ERR_ARG;
    if (ndim == 2) { g->n[2] = dims[0]; g->n[1] = 1;       g->n[0] = dims[1]; }
    else           { g->n[2] = dims[0]; g->n[1] = dims[1]; g->n[0] = dims[2]; }
    for (int a = 0; a < 3; ++a)
        if (g->n[a] < 1) return ORC_ERR_ARG;
    g->ndim = ndim;
    g->stride[0] = 1;
    g->stride[1] = g->n[0];
    g->stride[2] = g->n[0] * g->n[1];
    g->npts = g->n[0] * g->n[1] * g->n[2];
    return ORC_OK;
}

/* Linear index of a point given slow->fast indices (ndim of them). */
static int lin_index(const grid_t *g, const int64_t *idx, int64_t *out)
{
    int64_t iz = idx[0], iy = 0, ix;
    if (g->ndim == 2) ix = idx[1];
    else { iy = idx[1]; ix = idx[2]; }
    if (iz < 0 || iz >= g->n[2] || iy < 0 || iy >= g->n[1] || ix < 0 || ix >= g->n[0])
        return ORC_ERR_RANGE;
    *out = (iz * g->n[1] + iy) * g->n[0] + ix;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* fd_pxx / fd_pyy / fd_pzz.                          */
/* out_i = (c0*P_i + sum_{m=1..r} c_m*(P_{i-m e_a} + P_{i+m e_a})) / h^2     */
/* for r <= i_a < n_a - r, and out_i = 0 in the band (R#3).  Taps are  */
/* pair-grouped with m ascending (R#13).                                      */
/* ------------------------------------------------------------------------ */
static void second_derivative(const grid_t *g, int axis, int r, const double *c,
                              double h, const double *P, double *out, int nthreads)
{
    const int64_t n_a = g->n[axis], s = g->stride[axis];
    const double h2 = h * h;
    const int64_t nz = g->n[2], plane = g->n[0] * g->n[1];
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(static)
#endif
    for (int64_t iz = 0; iz < nz; ++iz) {
        for (int64_t q = 0; q < plane; ++q) {
            const int64_t i = iz * plane + q;
            int64_t i_a;
            if (axis == 2) i_a = iz;
            else if (axis == 1) i_a = q / g->n[0];
            else i_a = q % g->n[0];
            if (i_a < r || i_a >= n_a - r) { out[i] = 0.0; continue; }
            double acc = c[0] * P[i];
            for (int m = 1; m <= r; ++m)
                acc += c[m] * (P[i - m * s] + P[i + m * s]);
            out[i] = acc / h2;
        }
    }
    (void)nthreads;
}

/* Public single-axis derivative (operator pins). axis: 0=x, 1=y (3D), 2=z. */
int oracle_second_derivative(int ndim, const int64_t *dims, double h, int order,
                             int axis, const double *P, double *out)
{
    grid_t g;
    double c[5];
    int r = order / 2;
    if (!P || !out || h <= 0.0 || order % 2 || make_grid(ndim, dims, &g) ||
        oracle_coefficients(r, c) || axis < 0 || axis > 2 || (ndim == 2 && axis == 1))
        return ORC_ERR_ARG;
    second_derivative(&g, axis, r, c, h, P, out, 1);
    return ORC_OK;
}

/* fd_time: Pnew = 2P - Pold + dt^2 V^2 (sum of the
 * per-axis second derivatives), summed x, then y, then z.  (Pyy may be NULL.) */
static void time_update(int64_t npts, double dt, const double *P, const double *Pold,
                        const double *V, const double *Pxx, const double *Pyy,
                        const double *Pzz, double *Pnew, int nthreads)
{
    const double dt2 = dt * dt;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(static)
#endif
    for (int64_t i = 0; i < npts; ++i) {
        double lap = Pyy ? (Pxx[i] + Pyy[i]) + Pzz[i] : Pxx[i] + Pzz[i];
        Pnew[i] = 2.0 * P[i] - Pold[i] + dt2 * V[i] * V[i] * lap;
    }
    (void)nthreads;
}

/* Public fd_time (S:270-272 worked example).  Pyy may be NULL (2D). */
int oracle_time_update(int64_t npts, double dt, const double *P, const double *Pold,
                       const double *V, const double *Pxx, const double *Pyy,
                       const double *Pzz, double *Pnew)
{
    if (npts < 0 || !P || !Pold || !V || !Pxx || !Pzz || !Pnew) return ORC_ERR_ARG;
    time_update(npts, dt, P, Pold, V, Pxx, Pyy, Pzz, Pnew, 1);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* The simulation: nt repetitions of the run() body (R#15).       */
/*   P    in: P^0 (R#12),  out: P^nt                                          */
/*   Pold in: P^-1,        out: P_mod^{nt-1} (includes that step's source)    */
/*   T    out: T[j*nt + k] = P^{k+1}[rec_j]   (R#6), may be NULL if nrec == 0 */
/* Sources are added in registration order (R#17).                           */
/* ------------------------------------------------------------------------ */
int oracle_run(int ndim, const int64_t *dims, double h, double dt, int order,
               const double *V,
               int nsrc, const int64_t *src_idx, const double *src_f,
               const double *src_t0, const double *src_amp,
               int nrec, const int64_t *rec_idx,
               int64_t nt, double *P, double *Pold, double *T, int nthreads)
{
    grid_t g;
    double c[5];
    const int r = order / 2;
    if (!V || !P || !Pold || nt < 0 || h <= 0.0 || dt <= 0.0 || order % 2 ||
        make_grid(ndim, dims, &g) || oracle_coefficients(r, c) || nsrc < 0 || nrec < 0)
        return ORC_ERR_ARG;
    if (nthreads < 1) nthreads = 1;

    int64_t *sl = calloc((size_t)(nsrc + 1), sizeof(int64_t));
    int64_t *rl = calloc((size_t)(nrec + 1), sizeof(int64_t));
    if (!sl || !rl) { free(sl); free(rl); return ORC_ERR_NOMEM; }
    for (int s = 0; s < nsrc; ++s)
        if (lin_index(&g, src_idx + (int64_t)s * ndim, &sl[s])) { free(sl); free(rl); return ORC_ERR_RANGE; }
    for (int j = 0; j < nrec; ++j)
        if (lin_index(&g, rec_idx + (int64_t)j * ndim, &rl[j])) { free(sl); free(rl); return ORC_ERR_RANGE; }

    const size_t bytes = (size_t)g.npts * sizeof(double);
    double *Pxx = malloc(bytes), *Pzz = malloc(bytes);
    double *Pyy = (ndim == 3) ? malloc(bytes) : NULL;
    double *Pnew = malloc(bytes);
    if (!Pxx || !Pzz || !Pnew || (ndim == 3 && !Pyy)) {
        free(Pxx); free(Pzz); free(Pyy); free(Pnew); free(sl); free(rl);
        return ORC_ERR_NOMEM;
    }
    double *cur = P, *old = Pold, *nxt = Pnew;

    for (int64_t k = 0; k < nt; ++k) {
        /* 1. add_source (before the derivatives) */
        for (int s = 0; s < nsrc; ++s)
            cur[sl[s]] += src_amp[s] * oracle_ricker((double)k * dt, src_f[s], src_t0[s]);
        /* 2. fd_pzz, [fd_pyy], fd_pxx */
        second_derivative(&g, 2, r, c, h, cur, Pzz, nthreads);
        if (ndim == 3) second_derivative(&g, 1, r, c, h, cur, Pyy, nthreads);
        second_derivative(&g, 0, r, c, h, cur, Pxx, nthreads);
        /* 3. fd_time */
        time_update(g.npts, dt, cur, old, V, Pxx, Pyy, Pzz, nxt, nthreads);
        /* 4. swap(Pold, P); swap(P, Pnew) */
        double *t = old; old = cur; cur = nxt; nxt = t;
        /* 5. receivers sample the newest field (R#6) */
        for (int j = 0; j < nrec; ++j)
            T[(int64_t)j * nt + k] = cur[rl[j]];
    }
    /* Hand the rotated buffers back in the caller's arrays.  cur/old may alias
     * P, Pold or the scratch Pnew in any rotation, so stage through scratch
     * (Pxx, Pzz are free now). */
    memcpy(Pxx, cur, bytes);
    memcpy(Pzz, old, bytes);
    memcpy(P, Pxx, bytes);
    memcpy(Pold, Pzz, bytes);

    free(Pxx); free(Pzz); free(Pyy); free(Pnew); free(sl); free(rl);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Absorbing sponge boundary (reading R#18).  The paper is    */
/* silent on boundaries (R#3) and SPEC lists absorbing boundaries as a         */
/* non-goal; this is the optional alternative to the band rule alone. */
/* Cerjan et al. (1985, Geophysics 50:705): after each step, multiply the new */
/* and the current field by G inside a frame of nb cells, with                */
/*   g(j) = exp(-(alpha * (nb - d))^2),  d = min(j, n-1-j) < nb; else 1       */
/* per axis and G(i) = g_z(i_z) * g_y(i_y) * g_x(i_x).  Written for the       */
/* STORED fields (P as it enters the next step, i.e. Cerjan's damped P^{k+1}  */
/* plus the next injection; Pold = P^{k-1} as stored one step earlier):       */
/* Cerjan's Pold for step k is G * (stored P^{k-1}), so the step is            */
/*   Pnew = G * (2 P - G * Pold + dt^2 V^2 (Pxx [+ Pyy] + Pzz))               */
/* and the stored Pnew is Cerjan's damped P^{k+1} (equivalence checked in      */
/* tests/test_oracle_pins.py against the damp-after-step form).  The band rule */
/* still applies to the derivatives.  nb = 0 gives G = 1: the plain scheme.   */
/* ------------------------------------------------------------------------ */
int oracle_sponge_profile(int64_t n, int nb, double alpha, double *g)
{
    if (n < 1 || nb < 0 || !g) return ORC_ERR_ARG;
    for (int64_t j = 0; j < n; ++j) {
        const int64_t d = j < n - 1 - j ? j : n - 1 - j;
        if (d < nb) {
            const double a = alpha * (double)(nb - d);
            g[j] = exp(-(a * a));
        } else {
            g[j] = 1.0;
        }
    }
    return ORC_OK;
}

int oracle_run_sponge(int ndim, const int64_t *dims, double h, double dt, int order,
                      const double *V,
                      int nsrc, const int64_t *src_idx, const double *src_f,
                      const double *src_t0, const double *src_amp,
                      int nrec, const int64_t *rec_idx,
                      int64_t nt, double *P, double *Pold, double *T, int nthreads,
                      int nb, double alpha)
{
    grid_t g;
    double c[5];
    const int r = order / 2;
    if (!V || !P || !Pold || nt < 0 || h <= 0.0 || dt <= 0.0 || order % 2 || nb < 0 ||
        make_grid(ndim, dims, &g) || oracle_coefficients(r, c) || nsrc < 0 || nrec < 0)
        return ORC_ERR_ARG;
    if (nthreads < 1) nthreads = 1;
    int64_t *sl = calloc((size_t)(nsrc + 1), sizeof(int64_t));
    int64_t *rl = calloc((size_t)(nrec + 1), sizeof(int64_t));
    if (!sl || !rl) { free(sl); free(rl); return ORC_ERR_NOMEM; }
    for (int s = 0; s < nsrc; ++s)
        if (lin_index(&g, src_idx + (int64_t)s * ndim, &sl[s])) { free(sl); free(rl); return ORC_ERR_RANGE; }
    for (int j = 0; j < nrec; ++j)
        if (lin_index(&g, rec_idx + (int64_t)j * ndim, &rl[j])) { free(sl); free(rl); return ORC_ERR_RANGE; }

    const size_t bytes = (size_t)g.npts * sizeof(double);
    double *Pxx = malloc(bytes), *Pzz = malloc(bytes);
    double *Pyy = (ndim == 3) ? malloc(bytes) : NULL;
    double *Pnew = malloc(bytes), *G = malloc(bytes);
    double *gx = malloc((size_t)g.n[0] * sizeof(double)), *gy = malloc((size_t)g.n[1] * sizeof(double));
    double *gz = malloc((size_t)g.n[2] * sizeof(double));
    if (!Pxx || !Pzz || !Pnew || !G || !gx || !gy || !gz || (ndim == 3 && !Pyy)) {
        free(Pxx); free(Pzz); free(Pyy); free(Pnew); free(G); free(gx); free(gy); free(gz); free(sl); free(rl);
        return ORC_ERR_NOMEM;
    }
    /* the damping factor per point: the product of the per-axis profiles */
    oracle_sponge_profile(g.n[0], nb, alpha, gx);
    oracle_sponge_profile(g.n[2], nb, alpha, gz);
    if (ndim == 3) oracle_sponge_profile(g.n[1], nb, alpha, gy);
    else gy[0] = 1.0;
    for (int64_t iz = 0; iz < g.n[2]; ++iz)
        for (int64_t iy = 0; iy < g.n[1]; ++iy)
            for (int64_t ix = 0; ix < g.n[0]; ++ix)
                G[(iz * g.n[1] + iy) * g.n[0] + ix] = gz[iz] * gy[iy] * gx[ix];

    double *cur = P, *old = Pold, *nxt = Pnew;
    const double dt2 = dt * dt;
    for (int64_t k = 0; k < nt; ++k) {
        for (int s = 0; s < nsrc; ++s)
            cur[sl[s]] += src_amp[s] * oracle_ricker((double)k * dt, src_f[s], src_t0[s]);
        second_derivative(&g, 2, r, c, h, cur, Pzz, nthreads);
        if (ndim == 3) second_derivative(&g, 1, r, c, h, cur, Pyy, nthreads);
        second_derivative(&g, 0, r, c, h, cur, Pxx, nthreads);
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(static)
#endif
        for (int64_t i = 0; i < g.npts; ++i) {
            const double lap = Pyy ? (Pxx[i] + Pyy[i]) + Pzz[i] : Pxx[i] + Pzz[i];
            nxt[i] = G[i] * (2.0 * cur[i] - G[i] * old[i] + dt2 * V[i] * V[i] * lap);
        }
        double *t = old; old = cur; cur = nxt; nxt = t;
        for (int j = 0; j < nrec; ++j)
            T[(int64_t)j * nt + k] = cur[rl[j]];
    }
    memcpy(Pxx, cur, bytes);
    memcpy(Pzz, old, bytes);
    memcpy(P, Pxx, bytes);
    memcpy(Pold, Pzz, bytes);
    free(Pxx); free(Pzz); free(Pyy); free(Pnew); free(G); free(gx); free(gy); free(gz); free(sl); free(rl);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Slab mode: the same recursion on nranks z-slabs,    */
/* each holding its own planes plus r halo planes per side, the halos         */
/* refreshed by plain memcpy from the neighbour slab after every step.  Used   */
/* to check the decomposition logic (partition, halo placement, source and    */
/* receiver ownership) on the CPU; must be bitwise equal to oracle_run.       */
/* Partition: nz split evenly, the first nz mod nranks slabs one plane more.  */
/* ------------------------------------------------------------------------ */
int oracle_partition(int64_t nz, int nranks, int rank, int64_t *z0, int64_t *z1)
{
    if (nranks < 1 || rank < 0 || rank >= nranks || nz < nranks || !z0 || !z1)
        return ORC_ERR_ARG;
    int64_t base = nz / nranks, extra = nz % nranks;
    *z0 = rank * base + (rank < extra ? rank : extra);
    *z1 = *z0 + base + (rank < extra ? 1 : 0);
    return ORC_OK;
}

int oracle_run_slabs(int ndim, const int64_t *dims, double h, double dt, int order,
                     const double *V,
                     int nsrc, const int64_t *src_idx, const double *src_f,
                     const double *src_t0, const double *src_amp,
                     int nrec, const int64_t *rec_idx,
                     int64_t nt, double *P, double *Pold, double *T, int nranks)
{
    grid_t g;
    double c[5];
    const int r = order / 2;
    if (!V || !P || !Pold || nt < 0 || h <= 0.0 || dt <= 0.0 || order % 2 ||
        make_grid(ndim, dims, &g) || oracle_coefficients(r, c) || nranks < 1 ||
        g.n[2] < (int64_t)nranks * r || nsrc < 0 || nrec < 0)
        return ORC_ERR_ARG;
    const int64_t plane = g.n[0] * g.n[1], nz = g.n[2];
    int64_t *sl = calloc((size_t)(nsrc + 1), sizeof(int64_t));
    int64_t *rl = calloc((size_t)(nrec + 1), sizeof(int64_t));
    for (int s = 0; s < nsrc; ++s)
        if (lin_index(&g, src_idx + (int64_t)s * ndim, &sl[s])) { free(sl); free(rl); return ORC_ERR_RANGE; }
    for (int j = 0; j < nrec; ++j)
        if (lin_index(&g, rec_idx + (int64_t)j * ndim, &rl[j])) { free(sl); free(rl); return ORC_ERR_RANGE; }

    /* Per-slab state: planes [z0-r, z1+r) of P; [z0, z1) of Pold, V. */
    typedef struct { int64_t z0, z1, nloc; double *p, *old, *nxt, *v, *dxx, *dyy, *dzz; } slab_t;
    slab_t *sb = calloc((size_t)nranks, sizeof(slab_t));
    int err = ORC_OK;
    for (int q = 0; q < nranks && !err; ++q) {
        oracle_partition(nz, nranks, q, &sb[q].z0, &sb[q].z1);
        int64_t nh = sb[q].z1 - sb[q].z0 + 2 * r;   /* planes incl. halos */
        sb[q].nloc = nh;
        size_t bh = (size_t)(nh * plane) * sizeof(double);
        sb[q].p = calloc(1, bh);  sb[q].old = calloc(1, bh);  sb[q].nxt = calloc(1, bh);
        sb[q].v = calloc(1, bh);  sb[q].dxx = calloc(1, bh);  sb[q].dzz = calloc(1, bh);
        sb[q].dyy = calloc(1, bh);
        if (!sb[q].p || !sb[q].old || !sb[q].nxt || !sb[q].v || !sb[q].dxx || !sb[q].dzz || !sb[q].dyy)
            err = ORC_ERR_NOMEM;
        else {
            /* Fill owned + halo planes that exist globally. */
            for (int64_t lz = 0; lz < nh; ++lz) {
                int64_t gz = sb[q].z0 - r + lz;
                if (gz < 0 || gz >= nz) continue;
                memcpy(sb[q].p + lz * plane, P + gz * plane, (size_t)plane * sizeof(double));
                memcpy(sb[q].old + lz * plane, Pold + gz * plane, (size_t)plane * sizeof(double));
                memcpy(sb[q].v + lz * plane, V + gz * plane, (size_t)plane * sizeof(double));
            }
        }
    }
    if (err) goto done;

    for (int64_t k = 0; k < nt; ++k) {
        for (int q = 0; q < nranks; ++q) {
            slab_t *S = &sb[q];
            /* 1. add_source on every slab copy (owned or halo) of the point */
            for (int s = 0; s < nsrc; ++s) {
                int64_t gz = sl[s] / plane, lz = gz - S->z0 + r;
                if (lz < 0 || lz >= S->nloc) continue;
                S->p[lz * plane + sl[s] % plane] +=
                    src_amp[s] * oracle_ricker((double)k * dt, src_f[s], src_t0[s]);
            }
            /* 2. derivatives on owned planes; the z band uses the global z index */
            for (int64_t lz = r; lz < S->nloc - r; ++lz) {
                int64_t gz = S->z0 - r + lz;
                for (int64_t qq = 0; qq < plane; ++qq) {
                    int64_t i = lz * plane + qq;
                    int64_t ix = qq % g.n[0], iy = qq / g.n[0];
                    const int64_t sa[3] = {1, g.n[0], plane};
                    const int64_t ia[3] = {ix, iy, gz};
                    double *outs[3] = {S->dxx, S->dyy, S->dzz};
                    for (int a = 0; a < 3; ++a) {
                        if (ndim == 2 && a == 1) { outs[a][i] = 0.0; continue; }
                        if (ia[a] < r || ia[a] >= g.n[a] - r) { outs[a][i] = 0.0; continue; }
                        double acc = c[0] * S->p[i];
                        for (int m = 1; m <= r; ++m)
                            acc += c[m] * (S->p[i - m * sa[a]] + S->p[i + m * sa[a]]);
                        outs[a][i] = acc / (h * h);
                    }
                    double lap = (ndim == 3) ? (S->dxx[i] + S->dyy[i]) + S->dzz[i]
                                             : S->dxx[i] + S->dzz[i];
                    S->nxt[i] = 2.0 * S->p[i] - S->old[i] + dt * dt * S->v[i] * S->v[i] * lap;
                }
            }
        }
        /* 4. rotation, owned planes (halo planes of nxt refreshed below) */
        for (int q = 0; q < nranks; ++q) {
            slab_t *S = &sb[q];
            double *t = S->old; S->old = S->p; S->p = S->nxt; S->nxt = t;
        }
        /* halo exchange: r planes from each neighbour's owned edge */
        for (int q = 0; q < nranks; ++q) {
            slab_t *S = &sb[q];
            for (int hz = 0; hz < r; ++hz) {
                if (q > 0) {  /* low halo <- rank q-1's top owned planes */
                    slab_t *L = &sb[q - 1];
                    int64_t src_lz = L->nloc - 2 * r + hz;
                    memcpy(S->p + (int64_t)hz * plane, L->p + src_lz * plane, (size_t)plane * sizeof(double));
                }
                if (q < nranks - 1) {  /* high halo <- rank q+1's bottom owned planes */
                    slab_t *U = &sb[q + 1];
                    memcpy(S->p + (S->nloc - r + hz) * plane, U->p + (int64_t)(r + hz) * plane,
                           (size_t)plane * sizeof(double));
                }
            }
        }
        /* 5. receivers: the owner records */
        for (int j = 0; j < nrec; ++j) {
            int64_t gz = rl[j] / plane;
            for (int q = 0; q < nranks; ++q)
                if (gz >= sb[q].z0 && gz < sb[q].z1)
                    T[(int64_t)j * nt + k] = sb[q].p[(gz - sb[q].z0 + r) * plane + rl[j] % plane];
        }
    }
    /* gather owned planes */
    for (int q = 0; q < nranks; ++q)
        for (int64_t gz = sb[q].z0; gz < sb[q].z1; ++gz) {
            int64_t lz = gz - sb[q].z0 + r;
            memcpy(P + gz * plane, sb[q].p + lz * plane, (size_t)plane * sizeof(double));
            memcpy(Pold + gz * plane, sb[q].old + lz * plane, (size_t)plane * sizeof(double));
        }
done:
    for (int q = 0; q < nranks; ++q) {
        free(sb[q].p); free(sb[q].old); free(sb[q].nxt); free(sb[q].v);
        free(sb[q].dxx); free(sb[q].dyy); free(sb[q].dzz);
    }
    free(sb); free(sl); free(rl);
    return err;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
