"""Pins of the oracle's WENO5 on non-uniform (tanh-stretched) grids, SURVEY §8(f) F4
("local mesh refinement ... hyperbolic tangent function [16]"; DESIGN.md AMB-27).

What the mathematics fixes, independently of how orc_nu_cell_coeffs computes it:
* every candidate, and hence the reconstruction for ANY nonlinear weights, is exact on
  cell averages of quadratics, on an arbitrary stretched grid (both faces);
* with the linear (ideal) weights the reconstruction is exact on cell averages of
  quartics (that is what defines d_k), and the weights sum to 1;
* the Jiang-Shu smoothness indicator of a candidate reproducing f is
  Σ_{l=1,2} Δ^{2l-1} ∫_cell (f^(l))² dx: 0 for constants, s² Δ² for f = s x, and
  4 x_m² Δ² + (13/3) Δ⁴ for f = x² (closed forms integrated by hand);
* on a uniform grid it is the uniform WENO5-JS (coefficients (2,-7,11)/6 ..., linear
  weights (0.1, 0.6, 0.3)) up to rounding;
* the RHS of an advected two-fluid wave on a smooth tanh-refined grid converges at
  fifth order to the exact flux difference divided by the local width;
* the reflective / extrapolation identities of tests/test_oracle_bc.py hold on a
  stretched grid with the ghost-width rule of AMB-27 (ghost cells take the widths of
  the cells their data come from)."""
import numpy as np
import pytest

import oracle as O
from paper_2409_10729_b200 import workloads as W

RNG = np.random.default_rng(27)


def _random_boundaries(n, lo=0.0, ratio=1.6):
    """n cells of random widths in [1, ratio] x h (a rough, non-smooth stretched grid)."""
    w = RNG.uniform(1.0, ratio, n) * 0.1
    return lo + np.concatenate([[0.0], np.cumsum(w)])


def _cell_avg_poly(coef, xl, xr):
    """Exact cell average of sum_i coef[i] x^i over [xl, xr]."""
    s = 0.0
    for i, c in enumerate(coef):
        s += c * (xr ** (i + 1) - xl ** (i + 1)) / (i + 1)
    return s / (xr - xl)


def _poly(coef, x):
    return sum(c * x ** i for i, c in enumerate(coef))


@pytest.mark.parametrize("trial", range(20))
def test_exact_on_quadratics_for_any_weights(trial):
    xb = _random_boundaries(5, lo=RNG.uniform(-1, 1))
    C, st = O.nu_cell_coeffs(xb)
    assert st == 0
    coef = RNG.normal(size=3)
    v = [_cell_avg_poly(coef, xb[j], xb[j + 1]) for j in range(5)]
    scale = max(abs(x) for x in v)
    for eps in (1e-40, 1e-16, 1e-6, 1.0):            # any nonlinear weights
        vm, _ = O.weno5nu_minus(C, *v, eps=eps)
        vp, _ = O.weno5nu_plus(C, *v, eps=eps)
        assert vm == pytest.approx(_poly(coef, xb[3]), abs=1e-13 * scale)
        assert vp == pytest.approx(_poly(coef, xb[2]), abs=1e-13 * scale)


@pytest.mark.parametrize("trial", range(20))
def test_linear_weights_exact_on_quartics(trial):
    xb = _random_boundaries(5, lo=RNG.uniform(-1, 1), ratio=1.4)
    C, st = O.nu_cell_coeffs(xb)
    assert st == 0
    dm, dp = np.array(C.dm), np.array(C.dp)
    assert np.all(dm > 0) and np.all(dp > 0)
    assert dm.sum() == pytest.approx(1.0, abs=1e-14) and dp.sum() == pytest.approx(1.0, abs=1e-14)
    coef = RNG.normal(size=5)
    v = [_cell_avg_poly(coef, xb[j], xb[j + 1]) for j in range(5)]
    scale = max(abs(x) for x in v)
    # eps >> beta: every alpha_k = d_k/eps^2 (1 + O(beta/eps)), so omega = d
    vm, wm = O.weno5nu_minus(C, *v, eps=1e30)
    vp, wp = O.weno5nu_plus(C, *v, eps=1e30)
    assert np.allclose(wm, dm, rtol=1e-14) and np.allclose(wp, dp, rtol=1e-14)
    assert vm == pytest.approx(_poly(coef, xb[3]), abs=1e-12 * scale)
    assert vp == pytest.approx(_poly(coef, xb[2]), abs=1e-12 * scale)


@pytest.mark.parametrize("trial", range(10))
def test_smoothness_indicator_closed_forms(trial):
    """beta_k from the weights: alpha_k = d_k/(beta_k + eps)^2, so
    beta_k = sqrt(d_k / alpha_k) - eps; read alpha_k ratios through omega."""
    xb = _random_boundaries(5, lo=RNG.uniform(-1, 1), ratio=1.4)
    C, _ = O.nu_cell_coeffs(xb)
    dx = xb[3] - xb[2]
    xm = 0.5 * (xb[2] + xb[3])
    for coef, want in (((0.0, 2.5), 2.5 ** 2 * dx ** 2),
                       ((0.0, 0.0, 1.0), 4 * xm ** 2 * dx ** 2 + 13.0 / 3.0 * dx ** 4)):
        v = [_cell_avg_poly(coef, xb[j], xb[j + 1]) for j in range(5)]
        # every candidate reproduces f, so all three beta_k equal `want` and the
        # weights stay at their linear values for any eps
        for eps in (1e-40, 1e-3):
            _, wm = O.weno5nu_minus(C, *v, eps=eps)
            assert np.allclose(wm, C.dm, rtol=1e-10)
        # magnitude: with eps = want, alpha_k = d_k/(2 want)^2 -> compare against a
        # perturbation that changes one beta (one candidate stencil broken)
        vb = list(v)
        vb[0] += 10 * abs(want) ** 0.5 + 1.0      # only candidate 0 sees cell m-2
        _, wb = O.weno5nu_minus(C, *vb, eps=1e-40)
        assert wb[0] < C.dm[0] * 1e-2
    # beta of candidate 1 directly: equal-weight split of two candidates
    M = np.array(C.M).reshape(3, 3, 3)
    for coef in ((1.0, 0.3, -0.7), (0.2, -1.1, 0.4)):
        v = np.array([_cell_avg_poly(coef, xb[j], xb[j + 1]) for j in range(5)])
        for k in range(3):
            a, b, c = M[k] @ v[k:k + 3]
            # q_k(t) = a + b t + c t^2 is f(x_m + dx t): b = f'(x_m) dx, c = f''/2 dx^2
            assert a == pytest.approx(_poly(coef, xm), rel=1e-12, abs=1e-12)
            assert b == pytest.approx((coef[1] + 2 * coef[2] * xm) * dx, rel=1e-11, abs=1e-12)
            assert c == pytest.approx(coef[2] * dx ** 2, rel=1e-11, abs=1e-12)


def test_uniform_grid_reduces_to_uniform_weno5():
    xb = 0.37 + 0.125 * np.arange(6)
    C, _ = O.nu_cell_coeffs(xb)
    assert np.allclose(C.dm, (0.1, 0.6, 0.3), rtol=0, atol=1e-15)
    assert np.allclose(C.dp, (0.3, 0.6, 0.1), rtol=0, atol=1e-15)
    for _ in range(200):
        v = RNG.normal(size=5) * RNG.choice([1e-3, 1.0, 1e3])
        for eps in (1e-16, 1e-6):
            a, wa = O.weno5nu_minus(C, *v, eps=eps)
            b, wb = O.weno5_minus(*v, eps=eps)
            s = np.abs(v).max()
            assert a == pytest.approx(b, abs=1e-13 * s) and np.allclose(wa, wb, atol=1e-12)
            a, _ = O.weno5nu_plus(C, *v, eps=eps)
            b, _ = O.weno5_plus(*v, eps=eps)
            assert a == pytest.approx(b, abs=1e-13 * s)


def _wave_rhs_error(n, r):
    """RHS of the advected two-fluid wave (u = p = 1, alpha_1 = 0.5 + 0.25 sin 2 pi x,
    rho_1 = 1, rho_2 = 0.5) on a tanh-refined periodic grid, against the exact
    -u (alpha_1(x_{m+1/2}) - alpha_1(x_{m-1/2}))/dx_m of the volume fraction."""
    xb = W.tanh_boundaries(n, 0.0, 1.0, r=r, xi_a=0.3, xi_b=0.7, w=0.08)
    dx = np.diff(xb)
    s = (np.cos(2 * np.pi * xb[:-1]) - np.cos(2 * np.pi * xb[1:])) / (2 * np.pi * dx)
    a1 = 0.5 + 0.25 * s                               # exact cell averages
    one = np.ones_like(a1)
    v = np.stack([a1 * 1.0, (1 - a1) * 0.5, one, one, a1, 1 - a1])[:, None, None, :]
    P = O.Problem(N=2, d=1, n=(n, 1, 1), dx=(1.0 / n, 1, 1), bc=(-1,) * 6, gamma=(1.4, 1.6),
                  pi_inf=(0.0, 0.0), x_cb=(xb, None, None))
    q = O.prim_to_cons(P, np.ascontiguousarray(v))
    r_ = O.rhs(P, q)[4, 0, 0]                         # alpha_1 row
    f = 0.5 + 0.25 * np.sin(2 * np.pi * xb)
    exact = -(f[1:] - f[:-1]) / dx
    return np.mean(np.abs(r_ - exact))


def test_rhs_fifth_order_on_a_tanh_grid():
    errs = [_wave_rhs_error(n, 0.5) for n in (16, 32, 64, 128)]
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates.min() >= 4.8, (errs, rates)
    # and the grid is really stretched: the uniform grid gives another error
    assert _wave_rhs_error(32, 0.0) != pytest.approx(errs[1], rel=1e-2)


def test_stretched_rhs_equals_uniform_when_unstretched():
    """x_cb of a uniform grid through the non-uniform path = the uniform path up to
    rounding (not bitwise: the coefficients come from linear solves)."""
    pb = W.random_problem(3, (12, 10, 9), 2, "water")
    P, v = O.Problem.from_spec(pb), W.random_prims(pb)
    q = O.prim_to_cons(P, v)
    r_u = O.rhs(P, q)
    xcb = tuple(pb.lo[k] + np.arange(pb.n[k] + 1) * pb.dx[k] for k in range(3))
    Pn = O.Problem(P.N, P.d, P.n, P.dx, P.bc, P.gamma, P.pi_inf, x_cb=xcb)
    r_n = O.rhs(Pn, q)
    scale = np.abs(r_u).reshape(pb.E, -1).max(axis=1)
    assert np.all(np.abs(r_n - r_u).reshape(pb.E, -1).max(axis=1) <= 1e-11 * scale)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_stretched_reflective_wall_is_the_mirrored_periodic_domain(axis):
    N, n = 2, [9, 8, 7]
    pb = W.random_problem(3, n, N, "water")
    q = O.prim_to_cons(O.Problem.from_spec(pb), W.random_prims(pb, seed=3 + axis))
    xcb = [W.tanh_boundaries(n[k], 0.0, 0.1 * n[k], r=0.4, w=0.1) for k in range(3)]
    ax = 3 - axis
    mirror = np.flip(q, axis=ax).copy()
    mirror[N + axis] = -mirror[N + axis]
    full = np.concatenate([mirror, q], axis=ax)
    xf = list(xcb)
    xf[axis] = np.concatenate([-xcb[axis][:0:-1], xcb[axis]])   # mirrored grid on [-L, L]
    nf = list(n)
    nf[axis] *= 2
    bc = [W.BC_PERIODIC] * 6
    bc[2 * axis] = bc[2 * axis + 1] = W.BC_REFLECTIVE
    P_half = O.Problem(N, 3, tuple(n), (0.1,) * 3, tuple(bc), pb.gamma, pb.pi_inf, x_cb=tuple(xcb))
    P_full = O.Problem(N, 3, tuple(nf), (0.1,) * 3, (W.BC_PERIODIC,) * 6, pb.gamma, pb.pi_inf,
                       x_cb=tuple(xf))
    r_half, r_full = O.rhs(P_half, q), O.rhs(P_full, full)
    sl = [slice(None)] * 4
    sl[ax] = slice(n[axis], 2 * n[axis])
    # equal up to the rounding of the two grids' boundary positions (built differently)
    np.testing.assert_allclose(r_full[tuple(sl)], r_half, rtol=0,
                               atol=1e-12 * np.abs(r_half).max())


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("side", [0, 1])
def test_stretched_extrapolation_is_the_constant_extension(axis, side):
    N, n = 2, [8, 7, 9]
    pb = W.random_problem(3, n, N, "gas")
    q = O.prim_to_cons(O.Problem.from_spec(pb), W.random_prims(pb, seed=9 + axis))
    xcb = [W.tanh_boundaries(n[k], 0.0, 0.1 * n[k], r=0.4, w=0.1) for k in range(3)]
    ax = 3 - axis
    edge = [slice(None)] * 4
    edge[ax] = slice(0, 1) if side == 0 else slice(n[axis] - 1, n[axis])
    ext = np.repeat(q[tuple(edge)], 3, axis=ax)
    full = np.concatenate([ext, q] if side == 0 else [q, ext], axis=ax)
    xe = list(xcb)
    x = xcb[axis]
    if side == 0:          # 3 more cells of the boundary cell's width (constant extension)
        xe[axis] = np.concatenate([x[0] - (x[1] - x[0]) * np.arange(3, 0, -1), x])
    else:
        xe[axis] = np.concatenate([x, x[-1] + (x[-1] - x[-2]) * np.arange(1, 4)])
    ne = list(n)
    ne[axis] += 3
    bc = [W.BC_PERIODIC] * 6
    bc[2 * axis] = bc[2 * axis + 1] = W.BC_REFLECTIVE
    bc[2 * axis + side] = W.BC_EXTRAPOLATION
    P = O.Problem(N, 3, tuple(n), (0.1,) * 3, tuple(bc), pb.gamma, pb.pi_inf, x_cb=tuple(xcb))
    Pe = O.Problem(N, 3, tuple(ne), (0.1,) * 3, tuple(bc), pb.gamma, pb.pi_inf, x_cb=tuple(xe))
    r, r_ext = O.rhs(P, q), O.rhs(Pe, full)
    sl = [slice(None)] * 4
    sl[ax] = slice(3, 3 + n[axis]) if side == 0 else slice(0, n[axis])
    np.testing.assert_allclose(r_ext[tuple(sl)], r, rtol=0,
                               atol=1e-12 * np.abs(r).max())
