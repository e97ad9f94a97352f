"""Pins for the oracle's EOS (S0, S2): stiffened-gas closed forms (PAPER.md:64-68,
AMB-3), reduction to the ideal gas, N identical fluids == N = 1, exact pressure
equilibrium of the linear mixture rule."""
import numpy as np

import oracle as O
from paper_2409_10729_b200 import workloads as W


def _prob(N, d, gam, pinf):
    return O.Problem(N, d, (8, 8 if d > 1 else 1, 8 if d > 2 else 1), (0.1, 0.1, 0.1),
                     (-1,) * 6, gam, pinf)


def test_constants_closed_form():
    P = _prob(3, 3, (4.4, 1.4, 1.648), (6e8, 0.0, 0.0))
    G, Pi = O.constants(P)
    assert np.allclose(G, [1 / 3.4, 1 / 0.4, 1 / 0.648], rtol=1e-15)
    assert np.allclose(Pi, [4.4 * 6e8 / 3.4, 0.0, 0.0], rtol=1e-15)


def test_single_stiffened_gas_matches_textbook_form():
    """N = 1: p = (γ-1)(ρE - ½ρ|u|²) - γπ∞ (stiffened gas, Le Métayer & Saurel [9])."""
    rng = np.random.default_rng(1)
    for gam, pinf in ((1.4, 0.0), (4.4, 6e8), (1.648, 0.0)):
        P = _prob(1, 3, (gam,), (pinf,))
        n = 1000
        rho = rng.uniform(0.5, 1000, n)
        u = rng.uniform(-300, 300, (3, n))
        rhoE = rng.uniform(2.0, 3.0, n) * (1e5 + gam * pinf) / (gam - 1)
        q = np.stack([rho, rho * u[0], rho * u[1], rho * u[2], rhoE, np.ones(n)])
        v = O.cons_to_prim(P, q)
        ke = 0.5 * (q[1] ** 2 + q[2] ** 2 + q[3] ** 2) / rho
        p_ref = (gam - 1) * (rhoE - ke) - gam * pinf
        assert np.allclose(v[4], p_ref, rtol=1e-12, atol=1e-12 * (gam * pinf + np.abs(rhoE)).max())
        assert np.allclose(v[1:4], u, rtol=1e-15, atol=0)


def test_ideal_gas_reduction_and_roundtrip():
    rng = np.random.default_rng(2)
    P = _prob(2, 2, (1.4, 1.648), (0.0, 0.0))
    n = 2000
    a = rng.uniform(1e-6, 1 - 1e-6, n)
    v = np.stack([a * rng.uniform(0.5, 2, n), (1 - a) * rng.uniform(0.1, 0.4, n),
                  rng.uniform(-3, 3, n), rng.uniform(-3, 3, n), rng.uniform(0.1, 10, n),
                  a, 1 - a])
    q = O.prim_to_cons(P, v)
    # ideal-gas mixture: ρE = p Σ α_i/(γ_i-1) + ½ρ|u|²
    rho = v[0] + v[1]
    rhoE_ref = v[4] * (a / 0.4 + (1 - a) / 0.648) + 0.5 * rho * (v[2] ** 2 + v[3] ** 2)
    assert np.allclose(q[4], rhoE_ref, rtol=1e-14)
    v2 = O.cons_to_prim(P, q)
    # round trip within a few ulp (pressure limited by the cancellation ρE - KE)
    scale = np.abs(v) + 0.0
    scale[4] = v[4] + 0.5 * rho * (v[2] ** 2 + v[3] ** 2) / (a / 0.4 + (1 - a) / 0.648)
    assert np.all(np.abs(v2 - v) <= 8 * np.finfo(float).eps * scale + 1e-300)


def test_water_roundtrip_cancellation_bound():
    """AMB-18: p loses log10(Π/(Γp)) digits; the round-trip error is bounded by a few ulp
    of (Γp + Π + KE)/Γ, not of p."""
    rng = np.random.default_rng(3)
    P = _prob(2, 1, W.WATER[:1] + W.AIR[:1], W.WATER[1:] + W.AIR[1:])
    G, Pi = O.constants(P)
    n = 2000
    a = rng.uniform(1e-6, 1 - 1e-6, n)
    v = np.stack([a * 1000.0, (1 - a) * 1.2, rng.uniform(-100, 100, n),
                  rng.uniform(1e4, 1e9, n), a, 1 - a])
    v2 = O.cons_to_prim(P, O.prim_to_cons(P, v))
    Gm = a * G[0] + (1 - a) * G[1]
    Pm = a * Pi[0] + (1 - a) * Pi[1]
    rho = v[0] + v[1]
    scale = (Gm * v[3] + Pm + 0.5 * rho * v[2] ** 2) / Gm
    assert np.all(np.abs(v2[3] - v[3]) <= 8 * np.finfo(float).eps * scale)


def test_identical_fluids_equal_single_fluid():
    """N identical materials split by arbitrary α behave as N = 1 (Γ, Π linear in α)."""
    rng = np.random.default_rng(4)
    P1 = _prob(1, 1, (4.4,), (6e8,))
    P2 = _prob(2, 1, (4.4, 4.4), (6e8, 6e8))
    n = 500
    rho = rng.uniform(900, 1100, n)
    u = rng.uniform(-50, 50, n)
    p = rng.uniform(1e5, 1e8, n)
    a = rng.uniform(0, 1, n)
    q1 = O.prim_to_cons(P1, np.stack([rho, u, p, np.ones(n)]))
    q2 = O.prim_to_cons(P2, np.stack([a * rho, (1 - a) * rho, u, p, a, 1 - a]))
    assert np.allclose(q2[2], q1[1], rtol=1e-15)
    assert np.allclose(q2[3], q1[2], rtol=1e-14)
    v1 = O.cons_to_prim(P1, q1)
    v2 = O.cons_to_prim(P2, q2)
    assert np.allclose(v2[3], v1[2], rtol=0, atol=1e-14 * 6e8 * 4.4 / 3.4 * 3.4)


def test_pressure_equilibrium_of_mixture_rule():
    """Mixing two fluids at the same p (any α) returns exactly that p to round-off:
    ρE(α) = p Γ(α) + Π(α) + KE is linear in α (the reason for AMB-3)."""
    P = _prob(2, 1, (4.4, 1.4), (6e8, 0.0))
    G, Pi = O.constants(P)
    a = np.linspace(1e-6, 1 - 1e-6, 101)
    p0 = 1.01325e5
    v = np.stack([a * 1000.0, (1 - a) * 1.204, np.full_like(a, 10.0), np.full_like(a, p0),
                  a, 1 - a])
    v2 = O.cons_to_prim(P, O.prim_to_cons(P, v))
    bound = 8 * np.finfo(float).eps * (1 + (a * Pi[0]) / ((a * G[0] + (1 - a) * G[1]) * p0))
    assert np.all(np.abs(v2[3] / p0 - 1) <= bound)


def test_count_inadmissible_counts_the_corrupted_cells():
    """The admissibility guard (AMB-14, F3) counts exactly the cells that are not finite,
    have a non-positive mixture density, or a non-positive c^2 (negative pressure in an
    ideal gas), and nothing else."""
    import oracle as O
    from paper_2409_10729_b200 import workloads as W
    pb = W.random_problem(3, (9, 8, 7), 2, "gas")
    P = O.Problem.from_spec(pb)
    v = W.random_prims(pb, seed=3)
    q = O.prim_to_cons(P, v)
    assert O.count_inadmissible(P, q) == 0
    bad = q.copy()
    bad[0, 1, 2, 3] = np.nan                                   # not finite
    bad[0, 2, 2, 2] = -bad[0, 2, 2, 2] - bad[1, 2, 2, 2] - 1   # rho < 0
    vneg = v.copy()
    vneg[pb.n_fluids + 3, 4, 5, 6] = -0.5                      # p < 0 with pi_inf = 0
    qneg = O.prim_to_cons(P, vneg)
    bad[:, 4, 5, 6] = qneg[:, 4, 5, 6]
    assert O.count_inadmissible(P, bad) == 3
