"""The oracle's full solver (RHS + SSP-RK3) against exact Riemann solutions
(Toro [14] ch. 4 via oracle/exact_riemann.py): Sod (N=1), Sod with two identical
fluids (== N=1 to round-off), a two-γ Sod, and C1's water-air tube
(BASELINE.json configs[0])."""
import numpy as np
import pytest

import oracle as O
from oracle.exact_riemann import Side, sample, star_state
from paper_2409_10729_b200 import workloads as W


def _run_tube(n, N, gam, pinf, left, right, x0, T, cfl=0.4, am=1e-6, split=None):
    """left/right = (ρ, u, p) per side, fluid 1 on the left (α1 = 1-am), fluid 2 right;
    split = a fixed α1 everywhere instead (identical-fluid test)."""
    pb = W.Problem("tube", N, 1, (n, 1, 1), gamma=gam, pi_inf=pinf,
                   bc=(W.BC_EXTRAPOLATION,) * 2 + (W.BC_PERIODIC,) * 4)
    X = pb.centres()[0]
    L = X < x0
    if N == 1:
        v = np.stack([np.where(L, left[0], right[0]), np.where(L, left[1], right[1]),
                      np.where(L, left[2], right[2]), np.ones_like(X)])
    else:
        a1 = np.where(L, 1 - am, am) if split is None else np.full_like(X, split)
        v = np.stack([a1 * np.where(L, left[0], right[0]), (1 - a1) * np.where(L, left[0], right[0]),
                      np.where(L, left[1], right[1]), np.where(L, left[2], right[2]), a1, 1 - a1])
    P = O.Problem.from_spec(pb)
    q = O.prim_to_cons(P, v)
    sL = Side(*left, gam[0], pinf[0])
    sR = Side(*right, gam[-1], pinf[-1])
    smax = max(abs(left[1]) + sL.c, abs(right[1]) + sR.c) * 1.6
    steps = int(np.ceil(T / (cfl * pb.dx[0] / smax)))
    dt = T / steps
    q = O.rk3_step(P, q, dt, nsteps=steps)
    assert O.count_inadmissible(P, q) == 0
    vv = O.cons_to_prim(P, q)
    rho = vv[:N].sum(axis=0)[0, 0]
    u, p = vv[N, 0, 0], vv[N + 1, 0, 0]
    xi = (X[0, 0] - x0) / T
    ex = sample(sL, sR, xi)
    return rho, u, p, ex, X[0, 0], q


def test_sod_single_fluid_converges_to_exact():
    """SURVEY §8(c) full-solver pin: L1 convergence rate >= 0.6 under 400 -> 800 -> 1600
    cells, star plateau within 1e-3 of Toro's exact p* = 0.30313, u* = 0.927453."""
    errs = []
    for n in (400, 800, 1600):
        rho, u, p, (re, ue, pe, _), X, _ = _run_tube(n, 1, (1.4,), (0.0,), (1, 0, 1),
                                                      (0.125, 0, 0.1), 0.5, 0.2)
        errs.append([np.mean(np.abs(a - b)) for a, b in ((rho, re), (u, ue), (p, pe))])
        if n == 400:
            # star plateau between contact (x≈0.686) and shock (x≈0.850)
            m = (X > 0.72) & (X < 0.82)
            assert np.allclose(p[m], 0.30313, rtol=1e-3) and np.allclose(u[m], 0.927453, rtol=1e-3)
    errs = np.array(errs)
    rates = np.log2(errs[:-1] / errs[1:])
    assert errs[0, 0] < 2e-3 and rates.min() > 0.6, (errs, rates)


def test_two_identical_fluids_equal_single_fluid():
    """Two identical materials in a fixed volume-fraction split behave as one fluid:
    α is uniform, so Γ and Π are the single fluid's and each partial density is a
    fixed fraction of ρ (WENO weights are scale invariant up to ε).  (With a stepped
    α the component-wise reconstruction of α_iρ_i is NOT the reconstruction of ρ,
    so that case is not a pin.)"""
    r1 = _run_tube(100, 1, (1.4,), (0.0,), (1, 0, 1), (0.125, 0, 0.1), 0.5, 0.2)
    r2 = _run_tube(100, 2, (1.4, 1.4), (0.0, 0.0), (1, 0, 1), (0.125, 0, 0.1), 0.5, 0.2,
                   split=0.3)
    for a, b in zip(r1[:3], r2[:3]):
        assert np.allclose(a, b, rtol=1e-10, atol=1e-12)


def test_two_gamma_sod_plateau():
    p_ex, u_ex = star_state(Side(1, 0, 1, 1.4), Side(0.125, 0, 0.1, 1.6))
    assert p_ex == pytest.approx(0.311681, rel=1e-5) and u_ex == pytest.approx(0.907589, rel=1e-5)
    rho, u, p, (re, ue, pe, _), X, _ = _run_tube(400, 2, (1.4, 1.6), (0.0, 0.0), (1, 0, 1),
                                                  (0.125, 0, 0.1), 0.5, 0.2)
    m = (X > 0.72) & (X < 0.82)
    assert np.allclose(p[m], p_ex, rtol=3e-3) and np.allclose(u[m], u_ex, rtol=3e-3)
    assert np.mean(np.abs(p - pe)) < 5e-3


def _c1_run(n):
    """C1 (configs[0]) at n cells: the config's 200 RK3 steps of dt = 0.4 Δx/2653.30 at
    400 cells (AMB C1 reading), the same end time T = 75.38 µs at n cells."""
    pb = W.c1_water_air(n)
    P = O.Problem.from_spec(pb)
    q = O.prim_to_cons(P, W.c1_prims(pb))
    steps = pb.steps * n // 400
    q = O.rk3_step(P, q, pb.dt, nsteps=steps)
    assert O.count_inadmissible(P, q) == 0
    v = O.cons_to_prim(P, q)
    X = pb.centres()[0][0, 0]
    return X, v[0, 0, 0] + v[1, 0, 0], v[2, 0, 0], v[3, 0, 0], pb.dt * steps


C1_LEFT = Side(1000.0, 0.0, 1e9, 4.4, 6e8)    # water
C1_RIGHT = Side(50.0, 0.0, 1e5, 1.4, 0.0)     # air


def test_c1_water_air_against_exact():
    """C1 water-air tube against the exact two-stiffened-gas Riemann solution (Toro [14]
    ch. 4 with p -> p + π∞; p* = 1.419048e7 Pa, u* = 482.6104 m/s,
    ρ*L = 804.4446): L1 errors of ρ, u, p converge at rate >= 0.6 under 400 -> 800 ->
    1600 cells; the water-side star plateau (x in [0.62, 0.72], between the rarefaction
    tail at x ≈ 0.598 and the contact at x ≈ 0.736) is within 1e-3 of u*, ρ*L and p*.
    Pressure is compared on the stiffened-gas scale p + π∞,water (the EOS is an ideal
    gas in p + π∞; p itself is the small difference ρe(γ-1)... - γπ∞ there, and the
    plateau carries ~0.5 % start-up pressure waves of amplitude ~1e-4 (p* + π∞))."""
    p_star, u_star = star_state(C1_LEFT, C1_RIGHT)
    assert p_star == pytest.approx(1.419048e7, rel=1e-6)
    assert u_star == pytest.approx(482.6104, rel=1e-6)
    errs = []
    for n in (400, 800, 1600):
        X, rho, u, p, T = _c1_run(n)
        re, ue, pe, _ = sample(C1_LEFT, C1_RIGHT, (X - 0.7) / T)
        errs.append([np.mean(np.abs(rho - re)), np.mean(np.abs(u - ue)), np.mean(np.abs(p - pe))])
        m = (X > 0.62) & (X < 0.72)
        rho_star = re[m].mean()
        assert rho_star == pytest.approx(804.4446, rel=1e-5)
        assert abs(u[m].mean() / u_star - 1) < 1e-3, (n, u[m].mean())
        assert abs(rho[m].mean() / rho_star - 1) < 1e-3, (n, rho[m].mean())
        assert abs(p[m].mean() - p_star) / (p_star + 6e8) < 1e-3, (n, p[m].mean())
        m2 = (X > 0.64) & (X < 0.72)          # pointwise, off the smeared rarefaction tail
        assert np.abs(u[m2] / u_star - 1).max() < 1e-3, (n, np.abs(u[m2] / u_star - 1).max())
    errs = np.array(errs)
    rates = np.log2(errs[:-1] / errs[1:])
    assert rates.min() >= 0.6, (errs, rates)
    # L1 pressure error relative to the jump at 400 cells
    assert errs[0, 2] / 1e9 < 2e-3
