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
    errs = []
    for n in (100, 200, 400):
        rho, u, p, (re, ue, pe, _), X, _ = _run_tube(n, 1, (1.4,), (0.0,), (1, 0, 1),
                                                      (0.125, 0, 0.1), 0.5, 0.2)
        errs.append(np.mean(np.abs(rho - re)))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert errs[-1] < 4e-3 and rates.min() > 0.6, (errs, rates)
    # star plateau between contact (x≈0.686) and shock (x≈0.850) at n = 400
    m = (X > 0.72) & (X < 0.82)
    assert np.allclose(p[m], 0.30313, rtol=2e-3) and np.allclose(u[m], 0.92745, rtol=2e-3)


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


def test_c1_water_air_against_exact():
    """C1 (configs[0]): 400 cells, 200 RK3 steps at dt = 0.4 Δx/2653.30 (AMB C1 reading)."""
    pb = W.c1_water_air()
    P = O.Problem.from_spec(pb)
    q = O.prim_to_cons(P, W.c1_prims(pb))
    q = O.rk3_step(P, q, pb.dt, nsteps=pb.steps)
    assert O.count_inadmissible(P, q) == 0
    v = O.cons_to_prim(P, q)
    T = pb.dt * pb.steps
    X = pb.centres()[0][0, 0]
    sL = Side(1000.0, 0.0, 1e9, 4.4, 6e8)
    sR = Side(50.0, 0.0, 1e5, 1.4, 0.0)
    pe_star, ue_star = star_state(sL, sR)
    re, ue, pe, _ = sample(sL, sR, (X - 0.7) / T)
    p, u = v[3, 0, 0], v[2, 0, 0]
    # plateau between the contact (x ≈ 0.736) and the air shock (x ≈ 0.744) is only a
    # few cells wide at 400 cells; check the star plateau on the water side instead
    m = (X > 0.66) & (X < 0.72)
    assert np.allclose(p[m], pe_star, rtol=2e-2) and np.allclose(u[m], ue_star, rtol=2e-2)
    # L1 pressure error relative to the jump
    assert np.mean(np.abs(p - pe)) / 1e9 < 1e-2
