"""Exact Riemann solver for two stiffened gases -- TEST INFRASTRUCTURE ONLY.

Independent pin for the oracle's full solver (SURVEY §8(c) "Full solver vs exact
Riemann").  Toro [14] (the paper's HLLC reference) ch. 4: the pressure
function f_K(p) for shocks (Rankine-Hugoniot) and rarefactions (isentropic), solved
by Newton iteration for p*, then sampled at ξ = x/t.  A stiffened gas
p = (γ-1)ρe - γπ∞ is an ideal gas in the shifted pressure p+π∞,
so every formula of ch. 4 applies with p -> p+π∞ (each side keeps its own γ_K, π∞,K;
both pressure functions are written in the common physical p).

Pinned in tests/test_oracle_exact_riemann.py against Toro's printed star values for
the five standard tests (tests/golden/toro_ch4_star_values.json).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Side:
    rho: float
    u: float
    p: float
    gamma: float
    pi_inf: float = 0.0

    @property
    def c(self) -> float:
        return math.sqrt(self.gamma * (self.p + self.pi_inf) / self.rho)


def _f_and_df(p: float, K: Side):
    """Toro eq. (4.6)-(4.7) with p -> p + π∞ (and its derivative)."""
    g, pk, pi = K.gamma, K.p + K.pi_inf, K.pi_inf
    pp = p + pi
    if pp > pk:  # shock
        A = 2.0 / ((g + 1.0) * K.rho)
        B = (g - 1.0) / (g + 1.0) * pk
        s = math.sqrt(A / (pp + B))
        f = (pp - pk) * s
        df = s * (1.0 - 0.5 * (pp - pk) / (pp + B))
    else:  # rarefaction
        c = K.c
        e = (g - 1.0) / (2.0 * g)
        f = 2.0 * c / (g - 1.0) * ((pp / pk) ** e - 1.0)
        df = 1.0 / (K.rho * c) * (pp / pk) ** (-(g + 1.0) / (2.0 * g))
    return f, df


def star_state(L: Side, R: Side, tol: float = 1e-14, maxit: int = 200):
    """p*, u* (Toro §4.3.1, Newton-Raphson with a bisection safeguard)."""
    du = R.u - L.u
    pimin = min(L.pi_inf, R.pi_inf)
    lo = -pimin + max(1e-300, 1e-15 * pimin)  # p + π∞ > 0 on both sides

    def F(p):
        fl, dl = _f_and_df(p, L)
        fr, dr = _f_and_df(p, R)
        return fl + fr + du, dl + dr

    hi = max(L.p, R.p)
    while F(hi)[0] < 0.0:
        hi = 2.0 * hi + 1.0
    flo = F(lo)[0]
    if flo > 0.0:  # vacuum generation: not supported by this pin
        raise ValueError("vacuum is generated; exact solver not applicable")
    # initial guess: two-rarefaction-ish average, clipped into the bracket
    p = min(max(0.5 * (L.p + R.p), lo), hi)
    for _ in range(maxit):
        f, df = F(p)
        if f > 0.0:
            hi = p
        else:
            lo = p
        pn = p - f / df if df > 0 else 0.5 * (lo + hi)
        if not (lo < pn < hi):
            pn = 0.5 * (lo + hi)
        if abs(pn - p) <= tol * max(abs(pn) + min(L.pi_inf, R.pi_inf), 1e-300):
            p = pn
            break
        p = pn
    fl, _ = _f_and_df(p, L)
    fr, _ = _f_and_df(p, R)
    u = 0.5 * (L.u + R.u) + 0.5 * (fr - fl)
    return p, u


def star_densities(L: Side, R: Side, p: float):
    """ρ*L, ρ*R (Toro eqs. (4.50), (4.53), (4.57), (4.60) with p -> p+π∞)."""
    out = []
    for K in (L, R):
        g = K.gamma
        r = (p + K.pi_inf) / (K.p + K.pi_inf)
        if r > 1.0:
            gm = (g - 1.0) / (g + 1.0)
            out.append(K.rho * (r + gm) / (gm * r + 1.0))
        else:
            out.append(K.rho * r ** (1.0 / g))
    return tuple(out)


def sample(L: Side, R: Side, xi: np.ndarray):
    """Exact (ρ, u, p, side) at ξ = x/t; side = 0 left material, 1 right material."""
    ps, us = star_state(L, R)
    rsl, rsr = star_densities(L, R, ps)
    xi = np.asarray(xi, dtype=np.float64)
    rho = np.empty_like(xi)
    u = np.empty_like(xi)
    p = np.empty_like(xi)
    side = np.empty(xi.shape, dtype=np.int8)
    for idx, s in np.ndenumerate(xi):
        if s <= us:
            K, sign, rs = L, -1.0, rsl
            side[idx] = 0
        else:
            K, sign, rs = R, 1.0, rsr
            side[idx] = 1
        g, pi, c = K.gamma, K.pi_inf, K.c
        pk = K.p + pi
        pst = ps + pi
        if pst > pk:  # shock
            S = K.u + sign * c * math.sqrt((g + 1.0) / (2.0 * g) * pst / pk + (g - 1.0) / (2.0 * g))
            outside = (s <= S) if sign < 0 else (s >= S)
            if outside:
                rho[idx], u[idx], p[idx] = K.rho, K.u, K.p
            else:
                rho[idx], u[idx], p[idx] = rs, us, ps
        else:  # rarefaction
            cst = c * (pst / pk) ** ((g - 1.0) / (2.0 * g))
            head = K.u + sign * c
            tail = us + sign * cst
            if (s <= head) if sign < 0 else (s >= head):
                rho[idx], u[idx], p[idx] = K.rho, K.u, K.p
            elif (s > tail) if sign < 0 else (s < tail):
                rho[idx], u[idx], p[idx] = rs, us, ps
            else:  # inside the fan (Toro (4.56)/(4.63))
                a = 2.0 / (g + 1.0) - sign * (g - 1.0) / ((g + 1.0) * c) * (K.u - s)
                rho[idx] = K.rho * a ** (2.0 / (g - 1.0))
                u[idx] = 2.0 / (g + 1.0) * (-sign * c + (g - 1.0) / 2.0 * K.u + s)
                p[idx] = pk * a ** (2.0 * g / (g - 1.0)) - pi
    return rho, u, p, side
