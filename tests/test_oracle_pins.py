"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Each test names the oracle part it pins and the passage / closed form it uses.
None of the expected values comes from the oracle itself or from the CUDA path:
they are textbook rationals (tests/golden/), closed forms (polynomial
exactness and its leading error term, exact discrete standing and plane waves,
the 3D Green's function, the one-step closed form, the von Neumann limit),
invariants (discrete energy, weighted reciprocity, mirror symmetry, the light
cone, band zeros) and refinement ratios.  See DESIGN.md section 4.

P:n = PAPER.md line n, S:n = SPEC.md line n, R#n = DESIGN.md reading n.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ORDERS = (2, 4, 6, 8)


def _golden_coeffs():
    out = {}
    with open(os.path.join(GOLDEN, "fd_coefficients.txt")) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            out[int(parts[0])] = [Fraction(p) for p in parts[1:]]
    return out


GOLD = _golden_coeffs()


# ---------------------------------------------------------------------------
# Coefficients (R#1, R#2) -- textbook table + polynomial exactness
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("order", ORDERS)
def test_coefficients_match_textbook_rationals(order):
    c = oracle.coefficients(order)
    gold = GOLD[order]
    assert len(c) == len(gold)
    for cm, gm in zip(c, gold):
        assert cm == float(gm)          # exact rational rounded once to fp64
    # symmetric with sum zero; second moment 2 (consistency)
    assert sum(gold[0:1]) + 2 * sum(gold[1:]) == 0
    assert 2 * sum(m * m * gm for m, gm in enumerate(gold)) == 2


def _poly_field(shape, axis, p, h, x0):
    """Field (x)^p varying along ``axis`` ('x','y','z') only; x = x0 + i*h."""
    nd = len(shape)
    ax = {"x": nd - 1, "y": nd - 2, "z": 0}[axis]
    i = np.arange(shape[ax], dtype=np.float64)
    x = x0 + i * h
    bshape = [1] * nd
    bshape[ax] = shape[ax]
    return np.broadcast_to((x ** p).reshape(bshape), shape).copy(), x, ax


@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("ndim,axis", [(2, "x"), (2, "z"), (3, "x"), (3, "y"), (3, "z")])
def test_derivative_polynomial_exactness_and_leading_error(order, ndim, axis):
    """d2/dx2 of x^p is exact for p <= 2r+1; at p = 2r+2 the error is the
    closed form (-1)^(r+1) 2 (r!)^2 h^(2r) (Taylor remainder of the
    central formula); the band is exactly 0; the other axes see a
    field constant along them (S:252 -> ~0)."""
    r = order // 2
    h = 0.25
    shape = (2 * r + 7,) * ndim if ndim == 3 else (2 * r + 9, 2 * r + 11)
    for p in range(0, 2 * r + 3):
        P, x, ax = _poly_field(shape, axis, p, h, x0=-1.0)
        d = oracle.second_derivative(P, h, order, axis)
        n = shape[ax]
        sl_int = [slice(None)] * ndim
        sl_int[ax] = slice(r, n - r)
        xi = x[r:n - r]
        exact = p * (p - 1) * xi ** (p - 2) if p >= 2 else np.zeros_like(xi)
        if p == 2 * r + 2:
            exact = exact + (-1) ** (r + 1) * 2 * math.factorial(r) ** 2 * h ** (2 * r)
        bshape = [1] * ndim
        bshape[ax] = n - 2 * r
        want = np.broadcast_to(exact.reshape(bshape), d[tuple(sl_int)].shape)
        scale = max(1.0, np.max(np.abs(P)) / h ** 2)
        assert np.max(np.abs(d[tuple(sl_int)] - want)) <= 1e-12 * scale, (p, axis)
        # band: exactly zero
        for band in (slice(0, r), slice(n - r, n)):
            sl_b = [slice(None)] * ndim
            sl_b[ax] = band
            assert np.all(d[tuple(sl_b)] == 0.0)
        # a perpendicular axis sees a constant field: zero up to coefficient rounding
        other = [a for a in (("x", "z") if ndim == 2 else ("x", "y", "z")) if a != axis][0]
        d2 = oracle.second_derivative(P, h, order, other)
        tol = 0.0 if r == 1 else 1e-13 * scale    # r=1 taps are exact integers
        assert np.max(np.abs(d2)) <= tol


def test_spec_examples_constant_quadratic_transpose():
    """S:252 constant -> 0 everywhere; S:253 (j*dh)^2 -> interior 2 exactly
    (2nd order); S:260 fd_pzz(P) == transpose(fd_pxx(P^T))."""
    P = np.full((5, 7), 5.0)
    assert np.all(oracle.second_derivative(P, 0.5, 2, "x") == 0.0)
    assert np.all(oracle.second_derivative(P, 0.5, 2, "z") == 0.0)
    dh = 0.5
    j = np.arange(7) * dh
    Q = np.tile(j ** 2, (5, 1))
    d = oracle.second_derivative(Q, dh, 2, "x")
    assert np.all(d[:, 1:-1] == 2.0) and np.all(d[:, [0, -1]] == 0.0)
    rng = np.random.default_rng(1)
    R = rng.standard_normal((9, 13))
    for order in ORDERS:
        if min(R.shape) < order + 1:
            continue
        a = oracle.second_derivative(R, 0.7, order, "z")
        b = oracle.second_derivative(np.ascontiguousarray(R.T), 0.7, order, "x").T
        assert np.array_equal(a, b)


def test_spec_fd_time_example_and_free_evolution():
    """P=Pold=0, Pxx[2,2]=1, Pzz=0, V=2, dt=0.5 -> Pnew[2,2]=1.0, rest 0.
    S:272 / S:278: Pxx=Pzz=0 (or V=0) -> Pnew = 2P - Pold exactly."""
    z = np.zeros((5, 5))
    pxx = z.copy(); pxx[2, 2] = 1.0
    out = oracle.time_update(z, z, np.full((5, 5), 2.0), pxx, z, 0.5)
    want = z.copy(); want[2, 2] = 1.0
    assert np.array_equal(out, want)
    rng = np.random.default_rng(2)
    P, Po = rng.standard_normal((2, 6, 4))
    out = oracle.time_update(P, Po, np.zeros((6, 4)), rng.standard_normal((6, 4)),
                             rng.standard_normal((6, 4)), 0.3)
    assert np.array_equal(out, 2.0 * P - Po)


# ---------------------------------------------------------------------------
# Source time function (R#5)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("f", [10.0, 15.0, 25.0])
def test_ricker_peak_zeros_shape(f):
    t0 = 1.0 / f
    assert oracle.ricker(t0, f, t0) == 1.0
    tz = 1.0 / (math.pi * f * math.sqrt(2.0))
    assert abs(oracle.ricker(t0 + tz, f, t0)) < 1e-15
    assert abs(oracle.ricker(t0 - tz, f, t0)) < 1e-15
    # symmetric about t0; zero mean; equals -(1/(2 pi^2 f^2)) G'' for the
    # Gaussian G = exp(-pi^2 f^2 (t-t0)^2) (second derivative by central diff.)
    ts = np.linspace(t0 - 4 / f, t0 + 4 / f, 20001)
    R = np.array([oracle.ricker(t, f, t0) for t in ts])
    assert np.allclose(R, R[::-1], atol=1e-14)
    assert abs(np.trapezoid(R, ts)) < 1e-9
    a = math.pi ** 2 * f * f
    eps = 1e-4 / f
    for t in (t0 - 0.7 / f, t0 - 0.2 / f, t0 + 0.33 / f):
        G = lambda s: math.exp(-a * (s - t0) ** 2)
        g2 = (G(t + eps) - 2 * G(t) + G(t - eps)) / eps ** 2
        assert abs(oracle.ricker(t, f, t0) - (-g2 / (2 * a))) < 1e-6


# ---------------------------------------------------------------------------
# Stability limit (R#8)
# ---------------------------------------------------------------------------
def test_cfl_limits_spec_and_von_neumann():
    with open(os.path.join(GOLDEN, "cfl_limits.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                nd, order, expr = line.split(None, 2)
                assert abs(oracle.cfl_max(int(nd), int(order)) - eval(expr)) < 1e-15
    theta = np.linspace(0.0, math.pi, 100001)
    for order in ORDERS:
        g = GOLD[order]
        symbol = float(g[0]) + sum(2 * float(g[m]) * np.cos(m * theta) for m in range(1, len(g)))
        smax = np.max(np.abs(symbol))      # independent: from the golden table
        for nd in (2, 3):
            assert abs(oracle.cfl_max(nd, order) - 2 / math.sqrt(nd * smax)) < 1e-12


@pytest.mark.parametrize("ndim,order", [(2, 2), (2, 8), (3, 2), (3, 8)])
def test_stability_dichotomy(ndim, order):
    """at the limit the sourced run stays bounded; at 2x it
    exceeds 1e6 within 500 steps."""
    n = 64 if ndim == 2 else 24
    dims = (n,) * ndim
    h, v, f = 10.0, 2000.0, 25.0
    cmax = oracle.cfl_max(ndim, order)
    V = np.full(dims, v)
    src = [(tuple([n // 2] * ndim), f, 1 / f, 1.0)]
    steps = 2000 if ndim == 2 else 600
    for frac, bounded in ((0.99, True), (1.0, True)):
        dt = frac * cmax * h / v
        P, _, _ = oracle.run(V, h, dt, order, steps if ndim == 3 else 800, src, nthreads=4)
        # the field stays bounded (below 1e3 * max|w| = 1e3)
        assert np.max(np.abs(P)) < 1e3
    dt = 2.0 * cmax * h / v
    P, _, _ = oracle.run(V, h, dt, order, 500, src, nthreads=4)
    assert not np.all(np.isfinite(P)) or np.max(np.abs(P)) > 1e6


# ---------------------------------------------------------------------------
# One-step closed form: from zero state with w0 injected at s
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("order", ORDERS)
def test_one_step_closed_form(ndim, order):
    r = order // 2
    n = 4 * r + 1
    dims = (n,) * ndim
    h, dt, v = 10.0, 1e-3, 2500.0
    f, t0, amp = 20.0, 0.03, 1.7
    s = (2 * r,) * ndim
    P, Pold, _ = oracle.run(np.full(dims, v), h, dt, order, 1, [(s, f, t0, amp)])
    w0 = amp * (1 - 2 * math.pi ** 2 * f * f * t0 * t0) * math.exp(-math.pi ** 2 * f * f * t0 * t0)
    C2 = (v * dt / h) ** 2
    g = [float(x) for x in GOLD[order]]
    want = np.zeros(dims)
    want[s] = 2 * w0 + C2 * ndim * g[0] * w0
    for ax in range(ndim):
        for m in range(1, r + 1):
            for sign in (-1, 1):
                q = list(s); q[ax] += sign * m
                want[tuple(q)] = C2 * g[m] * w0
    assert np.count_nonzero(P) == 1 + 2 * ndim * r
    assert np.max(np.abs(P - want)) <= 1e-15 * abs(w0) * 10
    # Pold = P_mod^0 = the injected initial field (rotation)
    assert abs(Pold[s] - w0) <= 4e-16 * abs(w0) and np.count_nonzero(Pold) == 1


# ---------------------------------------------------------------------------
# Exact discrete solutions
# ---------------------------------------------------------------------------
def _coords(dims):
    return np.meshgrid(*[np.arange(n, dtype=np.float64) for n in dims], indexing="ij")


@pytest.mark.parametrize("ndim", [2, 3])
def test_standing_wave_exact_r1(ndim):
    """r=1, rigid box: sin(kx x) sin(kz z) [sin(ky y)] cos(w_d t) is an exact
    solution of the discrete scheme with sin(w_d dt/2) = C sqrt(sum sin^2(k_a h/2))
    (band rows at i=0, n-1 coincide with the nodes of the mode)."""
    n = 65 if ndim == 2 else 21
    steps = 200 if ndim == 2 else 60
    dims = (n,) * ndim
    h, v = 10.0, 1500.0
    L = (n - 1) * h
    modes = (2, 3, 1)[:ndim]
    ks = [math.pi * m / L for m in modes]
    dt = 0.5 * oracle.cfl_max(ndim, 2) * h / v
    C = v * dt / h
    wd = 2 * math.asin(C * math.sqrt(sum(math.sin(k * h / 2) ** 2 for k in ks)))
    X = _coords(dims)
    shape_f = np.ones(dims)
    for k, xi in zip(ks, X):
        shape_f = shape_f * np.sin(k * xi * h)
    P0, Pm1 = shape_f.copy(), shape_f * math.cos(-wd)
    P, Pold, _ = oracle.run(np.full(dims, v), h, dt, 2, steps, P0=P0, Pm1=Pm1)
    assert np.max(np.abs(P - shape_f * math.cos(wd * steps))) < 1e-11
    assert np.max(np.abs(Pold - shape_f * math.cos(wd * (steps - 1)))) < 1e-11


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("order", ORDERS)
def test_plane_wave_exact_in_domain_of_dependence(ndim, order):
    """cos(k.x - w_d t) with sin^2(w_d dt/2) = -(C^2/4) sum_a S(k_a h) is exact
    wherever the band's influence (r cells per step) has not arrived."""
    r = order // 2
    steps = 3
    n = 2 * r * (steps + 1) + 12 if ndim == 3 else 2 * r * (steps + 1) + 30
    dims = (n,) * ndim
    h, v = 10.0, 2000.0
    dt = 0.6 * oracle.cfl_max(ndim, order) * h / v
    C = v * dt / h
    ks = [0.21, -0.13, 0.17][:ndim]   # radians per cell along z, (y), x
    g = [float(x) for x in GOLD[order]]
    S = lambda th: g[0] + 2 * sum(g[m] * math.cos(m * th) for m in range(1, r + 1))
    wd = 2 * math.asin(math.sqrt(-(C * C / 4) * sum(S(k) for k in ks)))
    X = _coords(dims)
    phase = sum(k * xi for k, xi in zip(ks, X))
    P, _, _ = oracle.run(np.full(dims, v), h, dt, order, steps,
                         P0=np.cos(phase), Pm1=np.cos(phase + wd))
    m = r * (steps + 1)
    sl = tuple(slice(m, n - m) for _ in dims)
    err = np.max(np.abs(P[sl] - np.cos(phase - wd * steps)[sl]))
    assert err < 1e-13
    # and the band has polluted the outside (the pin is not vacuous)
    assert np.max(np.abs(P - np.cos(phase - wd * steps))) > 1e-6


# ---------------------------------------------------------------------------
# Convergence under refinement
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("order", ORDERS)
def test_operator_refinement_order(order):
    """Relative error of the discrete Laplacian on sin(ax+p)sin(bz+q) falls by
    ~2^(2r) per halving of h (sized by points per wavelength)."""
    r = order // 2
    errs = []
    ppws = (4, 8, 16) if r < 4 else (6, 12, 24)
    for ppw in ppws:
        h = 1.0 / ppw
        n = 4 * ppw + 2 * r + 1
        x = np.arange(n) * h
        a, b = 2 * math.pi, 2 * math.pi * 0.75
        Z, Xg = np.meshgrid(x, x, indexing="ij")
        P = np.sin(a * Xg + 0.3) * np.sin(b * Z + 0.7)
        lap = oracle.second_derivative(P, h, order, "x") + oracle.second_derivative(P, h, order, "z")
        ex = -(a * a + b * b) * P
        sl = (slice(r, n - r), slice(r, n - r))
        errs.append(np.max(np.abs(lap[sl] - ex[sl])) / np.max(np.abs(ex[sl])))
    ratio = errs[1] / errs[2]
    assert abs(ratio / 2 ** (2 * r) - 1) < 0.15, (errs, ratio)


def test_standing_wave_continuum_convergence_fixed_time():
    """S:373/S:608 with a fixed final time (the literal 'same steps' protocol
    halves T and is not a convergence test): r=1, CFL 0.5, T fixed, error vs
    the continuum standing wave falls ~4x per halving, ratio in [3.4, 4.6]."""
    v, Lbox, T = 1.0, 1.0, 0.25
    errs = []
    for n in (65, 129, 257):
        h = Lbox / (n - 1)
        dt = 0.5 * h / v
        steps = int(round(T / dt))
        Z, X = _coords((n, n))
        mode = np.sin(math.pi * X * h) * np.sin(math.pi * Z * h)
        w = v * math.pi * math.sqrt(2.0)
        P, _, _ = oracle.run(np.full((n, n), v), h, dt, 2, steps,
                             P0=mode, Pm1=mode * math.cos(-w * dt))
        errs.append(np.max(np.abs(P - mode * math.cos(w * steps * dt))))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.4 <= r1 <= 4.6 and 3.4 <= r2 <= 4.6, (errs, r1, r2)


@pytest.mark.parametrize("order", [2, 8])
def test_plane_wave_continuum_convergence(order):
    """Any r: continuum plane wave inside the domain of dependence at fixed
    CFL and final time converges at 2nd order overall (the leapfrog time error
    dominates): error ratio per h-halving in [3.4, 4.6]."""
    r = order // 2
    v, lam, T = 1.0, 1.0, 0.1
    k = 2 * math.pi / lam
    kx, kz = k * math.cos(0.4), k * math.sin(0.4)
    errs = []
    for ppw in (16, 32, 64):
        h = lam / ppw
        steps = ppw // 2            # dt = 0.2 h / v exactly: fixed CFL and final time
        dt = T / steps
        margin = r * (steps + 1) + 2
        n = 2 * margin + 2 * ppw     # measure over >= 2 wavelengths
        Z, X = _coords((n, n))
        ph = kx * X * h + kz * Z * h
        w = v * k
        P, _, _ = oracle.run(np.full((n, n), v), h, dt, order, steps,
                             P0=np.cos(ph), Pm1=np.cos(ph + w * dt))
        sl = (slice(margin, n - margin),) * 2
        errs.append(np.max(np.abs(P[sl] - np.cos(ph - w * steps * dt)[sl])))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.4 <= r1 <= 4.6 and 3.4 <= r2 <= 4.6, (errs, r1, r2)


# ---------------------------------------------------------------------------
# Invariants: energy, reciprocity, symmetry, light cone, band, zero source
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("ndim,order", [(2, 8), (3, 4)])
def test_discrete_energy_conserved(ndim, order):
    """E = sum (1/V^2)(Q^{k+1}-Q^k)^2 - dt^2 sum Q^{k+1} L Q^k is constant for
    the source-free scheme with heterogeneous V (catches V vs V^2, a wrong
    sign in 2P - Pold, a non-symmetric stencil)."""
    r = order // 2
    n = 40 if ndim == 2 else 20
    dims = (n,) * ndim
    rng = np.random.default_rng(5)
    V = rng.uniform(1500.0, 2500.0, dims)
    h = 10.0
    dt = 0.8 * oracle.cfl_max(ndim, order) * h / V.max()
    inner = tuple(slice(r, n - r) for _ in dims)
    Q0 = np.zeros(dims); Q0[inner] = rng.standard_normal(Q0[inner].shape)
    Q1 = np.zeros(dims); Q1[inner] = rng.standard_normal(Q1[inner].shape)
    axes = ("x", "z") if ndim == 2 else ("x", "y", "z")

    def L(Q):
        return sum(oracle.second_derivative(Q, h, order, a) for a in axes)

    def E(Qn, Qo):
        return np.sum((Qn - Qo) ** 2 / V ** 2) - dt * dt * np.sum(Qn * L(Qo))

    Es = [E(Q1, Q0)]
    cur, old = Q1, Q0
    for _ in range(150):
        nxt, old_, _ = oracle.run(V, h, dt, order, 1, P0=cur, Pm1=old)
        cur, old = nxt, old_
        Es.append(E(cur, old))
    Es = np.array(Es)
    assert Es.min() > 0
    assert np.max(np.abs(Es - Es[0])) / Es[0] < 1e-12


@pytest.mark.parametrize("ndim,order", [(2, 4), (3, 2), (3, 8)])
def test_weighted_reciprocity(ndim, order):
    """T_{s->q} V_s^2 == T_{q->s} V_q^2 (source injected into P, R#4): catches
    index swaps and V-vs-V^2 errors; the unweighted comparison is far off."""
    n = 48 if ndim == 2 else 22
    dims = (n,) * ndim
    rng = np.random.default_rng(7)
    V = rng.uniform(1500.0, 2500.0, dims)
    h = 10.0
    dt = 0.5 * oracle.cfl_max(ndim, order) * h / V.max()
    a = tuple([n // 3] * ndim)
    b = tuple([n // 2 + 3] + [n // 2 - 2] * (ndim - 1))
    f, t0 = 30.0, 0.03
    steps = 300 if ndim == 2 else 120
    _, _, Tab = oracle.run(V, h, dt, order, steps, [(a, f, t0, 1.0)], [b])
    _, _, Tba = oracle.run(V, h, dt, order, steps, [(b, f, t0, 1.0)], [a])
    lhs, rhs = Tab[0] * V[a] ** 2, Tba[0] * V[b] ** 2
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(lhs) < 1e-12
    assert np.linalg.norm(Tab[0] - Tba[0]) / np.linalg.norm(Tab[0]) > 1e-3


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("order", [2, 4, 8])
def test_mirror_symmetry_bitwise(ndim, order):
    """S:379 with pair-grouped taps (R#13): odd grid, centred source,
    homogeneous V -> P equal to its mirror images and to its transpose in the
    first two summed axes, to the bit."""
    n = 33 if ndim == 2 else 17
    dims = (n,) * ndim
    c = tuple([n // 2] * ndim)
    P, Pold, _ = oracle.run(np.full(dims, 2000.0), 10.0, 1e-3, order, 40,
                            [(c, 25.0, 0.04, 1.0)])
    for X in (P, Pold):
        for ax in range(ndim):
            assert np.array_equal(X, np.flip(X, axis=ax))
        # exchanging the two axes summed first (x, then z in 2D; x, then y in
        # 3D) is exact because fp addition commutes; (x+y)+z vs (z+y)+x is not
        assert np.array_equal(X, np.swapaxes(X, ndim - 2, ndim - 1))


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("order", [2, 4, 8])
def test_light_cone_and_band_zero(ndim, order):
    """After j steps from a point source in a zero field, P is exactly 0 outside
    the L1 ball of radius r*j (the stencil is axis-aligned); the band stays
    exactly 0 (R#3, Dirichlet frame), and it is non-zero inside."""
    r = order // 2
    n = 31 if ndim == 2 else 19
    dims = (n,) * ndim
    V = np.asarray(np.random.default_rng(3).uniform(1800, 2200, dims))
    s = tuple([n // 2 - 1] + [n // 2 + 1] * (ndim - 1))
    X = _coords(dims)
    dist = sum(np.abs(xi - si) for xi, si in zip(X, s))
    for j in (1, 2, 3):
        P, _, _ = oracle.run(V, 10.0, 1e-3, order, j, [(s, 25.0, 0.0, 1.0)])
        assert np.all(P[dist > r * j] == 0.0)
        if j == 1:
            assert np.count_nonzero(P) == 1 + 2 * ndim * r
    P, Pold, _ = oracle.run(V, 10.0, 1e-3, order, 60, [(s, 25.0, 0.04, 1.0)])
    band = np.zeros(dims, bool)
    for ax in range(ndim):
        idx = [slice(None)] * ndim
        idx[ax] = slice(0, r); band[tuple(idx)] = True
        idx[ax] = slice(n - r, n); band[tuple(idx)] = True
    assert np.all(P[band] == 0.0) and np.all(Pold[band] == 0.0)
    assert np.count_nonzero(P[~band]) > 0


def test_zero_source_stays_zero():
    P, Pold, T = oracle.run(np.full((20, 24), 2000.0), 10.0, 1e-3, 4, 50,
                            [((10, 12), 25.0, 0.04, 0.0)], [(5, 5), (10, 12)])
    assert not P.any() and not Pold.any() and not T.any()


def test_receivers_sample_newest_field():
    """R#6: T[j][k] = P^{k+1}[rec_j] (read after rotation), bit-identical."""
    dims = (24, 26)
    V = np.full(dims, 2000.0)
    src = [((12, 13), 25.0, 0.0, 1.0)]
    recs = [(12, 13), (12, 15), (0, 0), (20, 3)]
    _, _, T = oracle.run(V, 10.0, 1e-3, 4, 7, src, recs)
    for k in range(7):
        Pk, _, _ = oracle.run(V, 10.0, 1e-3, 4, k + 1, src)
        for j, q in enumerate(recs):
            assert T[j, k] == Pk[q]


def test_sources_add_in_registration_order_and_threads_invariant():
    dims = (30, 28)
    V = np.asarray(np.random.default_rng(9).uniform(1500, 2500, dims))
    src = [((14, 14), 25.0, 0.04, 1.0), ((14, 14), 12.0, 0.05, -0.3), ((8, 20), 20.0, 0.03, 2.0)]
    a = oracle.run(V, 10.0, 1e-3, 8, 80, src, [(3, 3)], nthreads=1)
    b = oracle.run(V, 10.0, 1e-3, 8, 80, src, [(3, 3)], nthreads=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    # superposition (linearity) across sources, to rounding
    parts = [oracle.run(V, 10.0, 1e-3, 8, 80, [s])[0] for s in src]
    assert np.max(np.abs(a[0] - sum(parts))) <= 1e-12 * np.max(np.abs(a[0]))


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("ndim,order", [(2, 8), (3, 4)])
def test_slab_mode_bitwise_equal(nranks, ndim, order):
    """CPU z-slab decomposition with memcpy halos is
    bitwise equal to the global run; the source sits on a slab face."""
    nz = 24 if ndim == 2 else 18
    dims = (nz, 26) if ndim == 2 else (nz, 14, 16)
    V = np.asarray(np.random.default_rng(11).uniform(1500, 2500, dims))
    z0, z1 = oracle.partition(nz, nranks, 1)
    s = (z0,) + tuple(d // 2 for d in dims[1:])
    recs = [(z0 - 1,) + s[1:], (z1 - 1,) + s[1:], (2,) + s[1:]]
    src = [(s, 25.0, 0.03, 1.0)]
    a = oracle.run(V, 10.0, 1e-3, order, 40, src, recs)
    b = oracle.run(V, 10.0, 1e-3, order, 40, src, recs, nranks=nranks)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_partition_even_split():
    for nz, P in ((1024, 8), (10, 3), (7, 7)):
        spans = [oracle.partition(nz, P, q) for q in range(P)]
        assert spans[0][0] == 0 and spans[-1][1] == nz
        assert all(spans[q][1] == spans[q + 1][0] for q in range(P - 1))
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)


# ---------------------------------------------------------------------------
# Green's function: pins the injection amplitude and time convention (R#4)
# ---------------------------------------------------------------------------
@pytest.mark.slow
def test_green_function_3d():
    """Unscaled injection of w into P before the stencil is the continuum
    source s(t) = w(t+dt) h^3/dt^2 at x_s, so the trace is
    T(t) = (h^3/dt^2) w(t + dt - R/v) / (4 pi v^2 R) in the direct-arrival
    window (dispersion-limited; the no-shift variant is ~20x worse)."""
    n, h, v, dt, f, t0, order = 96, 10.0, 2000.0, 0.5e-3, 10.0, 0.15, 8
    c = n // 2
    R = 12
    steps = 560
    _, _, T = oracle.run(np.full((n, n, n), v), h, dt, order, steps,
                         [((c, c, c), f, t0, 1.0)], [(c, c, c + R)], nthreads=oracle.max_threads())
    t = (np.arange(steps) + 1) * dt      # T[k] = P^{k+1}: time (k+1) dt
    Rm = R * h

    def w(tt):
        a = (math.pi * f * (tt - t0)) ** 2
        return (1 - 2 * a) * np.exp(-a)

    ana = (h ** 3 / dt ** 2) * w(t + dt - Rm / v) / (4 * math.pi * v * v * Rm)
    ana_noshift = (h ** 3 / dt ** 2) * w(t - Rm / v) / (4 * math.pi * v * v * Rm)
    win = t < 0.27
    err = np.linalg.norm(T[0][win] - ana[win]) / np.linalg.norm(ana[win])
    err0 = np.linalg.norm(T[0][win] - ana_noshift[win]) / np.linalg.norm(ana[win])
    assert err < 2e-3, err
    assert err0 > 10 * err


def test_green_function_2d():
    """2D counterpart: with the continuum source
    s(t) = w(t+dt) h^2/dt^2 the trace is
    T(t) = (h^2 / (dt^2 v^2)) int w(tau + dt) / (2 pi sqrt((t-tau)^2 - R^2/v^2)) dtau
    over tau < t - R/v.  With t - tau = (R/v) cosh(u) the integrand is smooth:
    T(t) = (h^2 / (2 pi dt^2 v^2)) int_0^inf w(t + dt - (R/v) cosh u) du.
    Checked in the window before the boundary reflections return; the
    no-shift convention (w(tau) instead of w(tau + dt)) is >10x worse."""
    n, h, v, dt, f, t0, order = 301, 10.0, 2000.0, 0.5e-3, 10.0, 0.15, 8
    c = n // 2
    R = 12
    steps = 640
    _, _, T = oracle.run(np.full((n, n), v), h, dt, order, steps, [((c, c), f, t0, 1.0)], [(c, c + R)],
                         nthreads=oracle.max_threads())
    t = (np.arange(steps) + 1) * dt
    a = R * h / v

    def w(tt):
        q = (math.pi * f * (tt - t0)) ** 2
        return (1 - 2 * q) * np.exp(-q)

    def trace(shift):
        out = np.empty(steps)
        for k, tk in enumerate(t):
            umax = math.acosh(max(1.0, (tk + shift - t0 + 0.5) / a)) + 0.5
            u = np.linspace(0.0, umax, 20001)
            g = w(tk + shift - a * np.cosh(u))
            out[k] = np.sum((g[1:] + g[:-1]) * 0.5) * (u[1] - u[0])
        return h * h / (2 * math.pi * dt * dt * v * v) * out

    ana, ana0 = trace(dt), trace(0.0)
    win = t < 0.32                     # the boundary reflection returns after ~1.4 s
    err = np.linalg.norm(T[0][win] - ana[win]) / np.linalg.norm(ana[win])
    err0 = np.linalg.norm(T[0][win] - ana0[win]) / np.linalg.norm(ana[win])
    assert err < 2e-3, err
    assert err0 > 10 * err, (err0, err)


# ---------------------------------------------------------------------------
# Absorbing sponge frame (Cerjan et al. 1985)
# ---------------------------------------------------------------------------
def test_sponge_profile_cerjan_values_and_shape():
    """Cerjan's frame: 20 cells, alpha = 0.015 -> G = exp(-0.09) = 0.9139 at the
    outermost cell (the value quoted with the method), 1 from the 20th cell
    in; symmetric; increasing inwards; Gaussian in the depth (nb - d)."""
    n, nb, a = 101, 20, 0.015
    g = oracle.sponge_profile(n, nb, a)
    assert abs(g[0] - 0.91393) < 1e-5 and abs(g[-1] - g[0]) == 0.0
    assert np.array_equal(g, g[::-1])
    assert np.all(g[nb:n - nb] == 1.0) and np.all(g[:nb] < 1.0)
    assert np.all(np.diff(g[:nb + 1]) > 0)
    depth = nb - np.arange(nb)
    # ln g is -(a * depth)^2: ratios of logs are ratios of squared depths
    assert np.allclose(np.log(g[:nb]) / np.log(g[0]), (depth / nb) ** 2, rtol=1e-12)
    assert np.all(oracle.sponge_profile(n, 0, a) == 1.0)


@pytest.mark.parametrize("ndim,order", [(2, 2), (3, 4)])
def test_sponge_zero_width_is_the_band_rule(ndim, order):
    dims = (30, 34) if ndim == 2 else (20, 22, 24)
    vel = np.random.default_rng(3).uniform(1500, 2500, dims)
    src = [(tuple(d // 2 for d in dims), 25.0, 0.02, 1.0)]
    recs = [tuple(d // 3 for d in dims)]
    a = oracle.run(vel, 10.0, 1e-3, order, 25, src, recs)
    b = oracle.run(vel, 10.0, 1e-3, order, 25, src, recs, sponge=(0, 0.015))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_sponge_v0_closed_form():
    """V = 0: each point obeys P^{k+1} = G (2 P^k - G P^{k-1}); from P^0 = P^-1 = c
    the solution is P^k = c (1 + (1 - G) k) G^k (double root G).  Catches a
    missing inner or outer G and a wrong per-axis product."""
    dims, nb, a, c = (17, 19, 23), 6, 0.08, 0.37
    P0 = np.full(dims, c)
    G = (oracle.sponge_profile(dims[0], nb, a)[:, None, None] * oracle.sponge_profile(dims[1], nb, a)[None, :, None]
         * oracle.sponge_profile(dims[2], nb, a)[None, None, :])
    for k in (1, 2, 7):
        P, Pold, _ = oracle.run(np.zeros(dims), 10.0, 1e-3, 2, k, P0=P0, Pm1=P0, sponge=(nb, a))
        assert np.allclose(P, c * (1 + (1 - G) * k) * G ** k, rtol=1e-13, atol=0)
        assert np.allclose(Pold, c * (1 + (1 - G) * (k - 1)) * G ** (k - 1), rtol=1e-13, atol=0)
    assert G.min() < 0.7                       # the test exercises real damping


def test_sponge_equals_cerjan_damp_after_step():
    """The stored-field step of the oracle is Cerjan's algorithm: run the
    original form -- update, then multiply the new AND the current field by G
    -- with the oracle's pinned derivative operator and compare."""
    dims, h, dt, order, nb, a, nt = (44, 52), 10.0, 1e-3, 4, 9, 0.05, 40
    vel = np.random.default_rng(5).uniform(1800, 2600, dims)
    src = [((20, 30), 25.0, 0.02, 1.0), ((9, 11), 18.0, 0.03, -0.6)]     # one source inside the frame
    recs = [(22, 26), (4, 5), (40, 48)]
    P, Pold, T = oracle.run(vel, h, dt, order, nt, src, recs, sponge=(nb, a))
    G = oracle.sponge_profile(dims[0], nb, a)[:, None] * oracle.sponge_profile(dims[1], nb, a)[None, :]
    cur, old = np.zeros(dims), np.zeros(dims)
    Tc = np.zeros((len(recs), nt))
    for k in range(nt):
        for idx, f, t0, amp in src:
            cur[idx] += amp * oracle.ricker(k * dt, f, t0)
        lap = oracle.second_derivative(cur, h, order, "x") + oracle.second_derivative(cur, h, order, "z")
        new = 2 * cur - old + dt * dt * vel * vel * lap
        new, cur = G * new, G * cur                       # Cerjan: damp both time levels
        old, cur = cur, new
        for j, q in enumerate(recs):
            Tc[j, k] = cur[q]
    assert np.allclose(P, cur, rtol=0, atol=1e-12 * np.abs(cur).max())
    assert np.allclose(G * Pold, old, rtol=0, atol=1e-12 * np.abs(old).max())
    assert np.allclose(T, Tc, rtol=0, atol=1e-12 * np.abs(Tc).max())


def test_sponge_mirror_symmetry_bitexact():
    n, order = 41, 4
    vel = np.full((n, n), 2000.0)
    P, Pold, _ = oracle.run(vel, 10.0, 1e-3, order, 80, [((n // 2, n // 2), 25.0, 0.03, 1.0)], sponge=(8, 0.06))
    for X in (P, Pold):
        assert np.array_equal(X, X[::-1, :]) and np.array_equal(X, X[:, ::-1]) and np.array_equal(X, X.T)


def test_sponge_absorbs_the_boundary_reflection():
    """Homogeneous 2D model, receiver near the source: after the direct wave
    has passed, the band rule alone returns the boundary reflection at full
    strength (rigid frame); Cerjan's 20-cell frame cuts it by more than 10x."""
    n, h, v, dt, f = 201, 10.0, 2000.0, 1e-3, 25.0
    c = n // 2
    vel = np.full((n, n), v)
    src = [((c, c), f, 0.04, 1.0)]
    rec = [(c, c + 10)]
    nt = 1300
    _, _, T0 = oracle.run(vel, h, dt, 2, nt, src, rec, nthreads=oracle.max_threads())
    _, _, T1 = oracle.run(vel, h, dt, 2, nt, src, rec, nthreads=oracle.max_threads(), sponge=(20, 0.015))
    t = (np.arange(nt) + 1) * dt
    direct = t < 0.25
    refl = (t > 0.7) & (t < 1.3)        # first reflections: ~0.9-1.0 s round trip to the nearest faces
    assert np.allclose(T0[0][direct], T1[0][direct], rtol=0, atol=1e-9 * np.abs(T0).max())
    r0, r1 = np.abs(T0[0][refl]).max(), np.abs(T1[0][refl]).max()
    assert r0 > 0.05 * np.abs(T0[0][direct]).max()      # the rigid frame reflects
    assert r1 < 0.1 * r0, (r0, r1)
