"""Pins for the oracle's HLLC flux (S3; PAPER.md:84 citing Toro [14] ch. 10).

- consistency: F(v, v) is the physical flux of the 5-equation model (written here
  from the PDE, PAPER.md:56-62 with AMB-1/2/5) and u^f = u;
- supersonic faces return the upwind physical flux;
- an isolated contact (equal p and u) is resolved exactly (exact Godunov flux);
- against an independent textbook HLLC written in Toro's star-state form
  F*_K = F_K + S_K (U*_K - U_K) (Toro eqs. 10.38-10.39), extended to the partial
  densities with (α_iρ_i)*_K = (α_iρ_i)_K χ_K (Johnsen & Colonius form);
- the volume-fraction flux uses the same face velocity as the partial densities.
"""
import numpy as np

import oracle as O


def _prob(N, d, gam, pinf):
    return O.Problem(N, d, (8,) * d + (1,) * (3 - d), (0.1,) * 3, (-1,) * 6, gam, pinf)


def _phys(P, v, direction):
    """Physical flux of the 5-eq model at primitive state v along `direction`."""
    N, d = P.N, P.d
    G, Pi = O.constants(P)
    a = v[N + d + 1:]
    rho = v[:N].sum()
    u = v[N:N + d]
    p = v[N + d]
    rhoE = p * (a @ G) + a @ Pi + 0.5 * rho * (u @ u)
    un = u[direction]
    F = np.empty(P.E)
    F[:N] = v[:N] * un
    F[N:N + d] = rho * u * un
    F[N + direction] += p
    F[N + d] = un * (rhoE + p)
    F[N + d + 1:] = a * un
    return F, rhoE


def _cons(P, v):
    return O.prim_to_cons(P, v.reshape(-1, 1))[:, 0]


def _sound(P, v):
    N, d = P.N, P.d
    G, Pi = O.constants(P)
    a = v[N + d + 1:]
    rho = v[:N].sum()
    Gm, Pm = a @ G, a @ Pi
    return np.sqrt(((Gm + 1) * v[N + d] + Pm) / (rho * Gm))


def _toro_hllc(P, vL, vR, direction):
    """Independent HLLC in Toro's star-state form (conservative components)."""
    N, d = P.N, P.d
    uL, uR = vL[N + direction], vR[N + direction]
    pL, pR = vL[N + d], vR[N + d]
    rL, rR = vL[:N].sum(), vR[:N].sum()
    cL, cR = _sound(P, vL), _sound(P, vR)
    SL = min(uL - cL, uR - cR)           # Davis estimate, Toro (10.48)
    SR = max(uL + cL, uR + cR)
    Ss = (pR - pL + rL * uL * (SL - uL) - rR * uR * (SR - uR)) / (rL * (SL - uL) - rR * (SR - uR))
    FL, EL = _phys(P, vL, direction)
    FR, ER = _phys(P, vR, direction)
    UL, UR = _cons(P, vL), _cons(P, vR)

    def star(v, U, S, u, p, r, E):
        chi = (S - u) / (S - Ss)
        Us = U.copy()
        Us[:N] = v[:N] * chi
        Us[N:N + d] = r * chi * v[N:N + d]
        Us[N + direction] = r * chi * Ss
        Us[N + d] = chi * (E + (Ss - u) * (r * Ss + p / (S - u)))
        return Us

    if SL >= 0:
        return FL, 'L'
    if SR <= 0:
        return FR, 'R'
    if Ss >= 0:
        Us = star(vL, UL, SL, uL, pL, rL, EL)
        return FL + SL * (Us - UL), '*L'
    Us = star(vR, UR, SR, uR, pR, rR, ER)
    return FR + SR * (Us - UR), '*R'


def _rand_state(rng, N, d, water=False):
    a = rng.dirichlet(np.ones(N)) * (1 - 1e-6 * N) + 1e-6
    rho0 = np.array([1000.0, 1.2, 0.2][:N]) if water else np.array([1.0, 0.2, 0.5][:N])
    partial = a * rho0 * rng.uniform(0.5, 2, N)
    c = 400.0 if water else 1.5
    u = rng.uniform(-2, 2, d) * c
    p = rng.uniform(0.5, 2) * (1e5 if water else 1.0)
    return np.concatenate([partial, u, [p], a])


MATS = {
    "gas": ((1.4, 1.648, 1.6), (0.0, 0.0, 0.0)),
    "water": ((4.4, 1.4, 1.648), (6e8, 0.0, 0.0)),
}


def test_consistency_and_face_velocity():
    rng = np.random.default_rng(8)
    for mats, water in (("gas", False), ("water", True)):
        gam, pinf = MATS[mats]
        for N in (1, 2, 3):
            for d in (1, 2, 3):
                P = _prob(N, d, gam[:N], pinf[:N])
                for _ in range(20):
                    v = _rand_state(rng, N, d, water)
                    for k in range(d):
                        F, uf = O.hllc(P, k, v, v)
                        Fp, _ = _phys(P, v, k)
                        scale = np.abs(Fp) + np.abs(_cons(P, v)) * (abs(v[N + k]) + _sound(P, v))
                        assert np.all(np.abs(F - Fp) <= 1e-12 * scale), (N, d, k)
                        assert abs(uf - v[N + k]) <= 1e-12 * (abs(v[N + k]) + _sound(P, v))


def test_supersonic_upwinding():
    rng = np.random.default_rng(9)
    P = _prob(2, 2, (1.4, 1.648), (0.0, 0.0))
    hits = {"L": 0, "R": 0}
    for _ in range(400):
        vL, vR = _rand_state(rng, 2, 2), _rand_state(rng, 2, 2)
        sgn = rng.choice([-1.0, 1.0])
        vL[2] = vR[2] = sgn * rng.uniform(6, 10)  # |u| well above c
        F, uf = O.hllc(P, 0, vL, vR)
        ref, case = _toro_hllc(P, vL, vR, 0)
        if case in hits:
            hits[case] += 1
            Fu = _phys(P, vL if case == "L" else vR, 0)[0]
            assert np.array_equal(F, F) and np.allclose(F, Fu, rtol=1e-13, atol=1e-13)
            assert uf == (vL if case == "L" else vR)[2]
    assert hits["L"] > 50 and hits["R"] > 50


def test_isolated_contact_is_exact():
    """Equal p and u, different densities and volume fractions: the exact Riemann
    solution is a single contact moving at u, so the Godunov flux is the upwind flux."""
    rng = np.random.default_rng(10)
    for mats, water in (("gas", False), ("water", True)):
        gam, pinf = MATS[mats]
        P = _prob(2, 3, gam[:2], pinf[:2])
        for _ in range(100):
            vL, vR = _rand_state(rng, 2, 3, water), _rand_state(rng, 2, 3, water)
            vR[2:6] = vL[2:6]       # same velocity vector and pressure
            F, uf = O.hllc(P, 0, vL, vR)
            up = vL if vL[2] >= 0 else vR
            Fu = _phys(P, up, 0)[0]
            scale = np.abs(Fu) + np.abs(_cons(P, up)) * _sound(P, up)
            assert np.all(np.abs(F - Fu) <= 1e-12 * scale)
            assert abs(uf - vL[2]) <= 1e-12 * _sound(P, up)


def test_matches_independent_toro_form():
    rng = np.random.default_rng(11)
    cases = set()
    for mats, water in (("gas", False), ("water", True)):
        gam, pinf = MATS[mats]
        for N in (1, 2, 3):
            for d in (1, 2, 3):
                P = _prob(N, d, gam[:N], pinf[:N])
                for _ in range(60):
                    vL, vR = _rand_state(rng, N, d, water), _rand_state(rng, N, d, water)
                    k = int(rng.integers(0, d))
                    F, uf = O.hllc(P, k, vL, vR)
                    ref, case = _toro_hllc(P, vL, vR, k)
                    cases.add(case)
                    nc = 2 * N + d + 1 - N  # conservative part: everything except α rows
                    scale = (np.abs(_cons(P, vL)) + np.abs(_cons(P, vR))) * (
                        np.abs(vL[N:N + d]).max() + np.abs(vR[N:N + d]).max() + _sound(P, vL) + _sound(P, vR))
                    assert np.all(np.abs(F[:nc] - ref[:nc]) <= 1e-11 * scale[:nc]), (N, d, case)
                    # volume fractions are carried with the same face velocity as the mass
                    K = vL if case in ("L", "*L") else vR
                    assert np.allclose(F[:N] / K[:N], uf, rtol=1e-14, atol=1e-14 * abs(uf))
                    assert np.allclose(F[N + d + 1:], K[N + d + 1:] * uf, rtol=1e-15, atol=0)
    assert cases == {"L", "R", "*L", "*R"}
