"""Pins for the exact Riemann solver (test tool; Toro [14] ch. 4)."""
import json
import math
import os

import numpy as np
import pytest

from oracle.exact_riemann import Side, sample, star_densities, star_state

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "toro_ch4_star_values.json")


def _tol(printed: str) -> float:
    dec = len(printed.split(".")[1]) if "." in printed else 0
    return 3.0 * 10.0 ** (-dec)


def test_toro_table_star_values():
    g = json.load(open(GOLDEN))
    gam = g["gamma"]
    for t in g["tests"]:
        L = Side(*t["left"], gam)
        R = Side(*t["right"], gam)
        p, u = star_state(L, R)
        rl, rr = star_densities(L, R, p)
        for name, val in (("p_star", p), ("u_star", u), ("rho_star_L", rl), ("rho_star_R", rr)):
            printed = t[name]
            assert abs(val - float(printed)) <= _tol(printed), (t["name"], name, val, printed)


def _rh_residual(pre: Side, rho2, u2, p2, S):
    """Rankine-Hugoniot jump conditions across a shock of speed S for a stiffened gas."""
    g, pi = pre.gamma, pre.pi_inf

    def cons(r, u, p):
        E = (p + g * pi) / (g - 1.0) + 0.5 * r * u * u
        return np.array([r, r * u, E]), np.array([r * u, r * u * u + p, u * (E + p)])

    U1, F1 = cons(pre.rho, pre.u, pre.p)
    U2, F2 = cons(rho2, u2, p2)
    return (F2 - F1) - S * (U2 - U1), np.abs(F1) + np.abs(S * U1)


def test_water_air_star_state_satisfies_rankine_hugoniot():
    """C1: left water at 1e9 Pa, right air at 1e5 Pa.  The right-moving
    air shock must satisfy the RH conditions with the stiffened-gas EOS, and the left
    rarefaction must be isentropic (p+π∞)/ρ^γ = const."""
    L = Side(1000.0, 0.0, 1.0e9, 4.4, 6.0e8)
    R = Side(50.0, 0.0, 1.0e5, 1.4, 0.0)
    p, u = star_state(L, R)
    rl, rr = star_densities(L, R, p)
    # shock speed from mass conservation
    S = (rr * u - R.rho * R.u) / (rr - R.rho)
    res, scale = _rh_residual(R, rr, u, p, S)
    assert np.all(np.abs(res) <= 1e-9 * scale)
    # isentrope on the water side
    assert abs((p + L.pi_inf) / rl ** L.gamma / ((L.p + L.pi_inf) / L.rho ** L.gamma) - 1) < 1e-12
    # Riemann invariant across the left rarefaction: u + 2c/(γ-1) constant
    cl = L.c
    cs = math.sqrt(L.gamma * (p + L.pi_inf) / rl)
    assert abs((u + 2 * cs / (L.gamma - 1)) - (L.u + 2 * cl / (L.gamma - 1))) < 1e-9 * cl
    assert p == pytest.approx(1.419048e7, rel=1e-6)
    assert u == pytest.approx(482.6104, rel=1e-6)


def test_sampled_solution_is_continuous_in_fans_and_matches_states():
    L = Side(1.0, 0.0, 1.0, 1.4)
    R = Side(0.125, 0.0, 0.1, 1.4)
    xi = np.linspace(-3, 3, 6001)
    rho, u, p, side = sample(L, R, xi)
    assert rho[0] == 1.0 and p[0] == 1.0 and rho[-1] == 0.125 and p[-1] == 0.1
    # fan is continuous: largest jump inside the rarefaction is small
    head, tail = -L.c, 0.92745 - L.c * (0.30313 / 1.0) ** (0.4 / 2.8)
    m = (xi > head) & (xi < tail)
    assert np.max(np.abs(np.diff(p[m]))) < 1e-3
    assert np.all(side[xi < 0.9] == 0) and np.all(side[xi > 0.93] == 1)
