"""Pins for the oracle's full RHS and RK3 (S1-S4; eq. (1)).

I1 uniform state -> rhs == 0 bitwise; I2 periodic discrete conservation; Σα = 1;
I3 pressure/velocity equilibrium across an advected interface (100 RK3 steps);
I4 axis permutation; I5 subdomain decomposition == single domain (bitwise);
fifth-order RHS convergence vs the exact flux difference of an advected wave;
RK3 amplification factor (closed form) and third-order temporal convergence.
"""
import numpy as np
import pytest

import oracle as O
from paper_2409_10729_b200 import workloads as W


def _oprob(pb, bc=None):
    return O.Problem.from_spec(pb, bc=bc)


def _cons(pb, v):
    return O.prim_to_cons(_oprob(pb), v)


@pytest.mark.parametrize("ndim,N,mats", [(1, 1, "gas"), (1, 2, "water"), (2, 2, "gas"),
                                         (2, 3, "water"), (3, 2, "water"), (3, 3, "gas")])
def test_uniform_state_rhs_is_exactly_zero(ndim, N, mats):
    n = (12, 10, 8)[:ndim]
    pb = W.random_problem(ndim, n, N, mats)
    v = W.random_prims(pb, seed=3)
    v = np.broadcast_to(v[:, :1, :1, :1], v.shape).copy()   # one random state everywhere
    q = _cons(pb, v)
    for bc in (W.BC_PERIODIC, W.BC_EXTRAPOLATION):
        r = O.rhs(_oprob(pb, bc=(bc,) * 6), q)
        assert np.all(r == 0.0)


@pytest.mark.parametrize("ndim,N,mats", [(1, 2, "water"), (2, 2, "gas"), (3, 3, "water")])
def test_periodic_conservation(ndim, N, mats):
    n = (24, 16, 12)[:ndim]
    pb = W.random_problem(ndim, n, N, mats)
    q = _cons(pb, W.random_prims(pb))
    r = O.rhs(_oprob(pb), q)
    for e in range(N + ndim + 1):  # partial densities, momenta, energy
        tot = r[e].sum()
        scale = np.abs(r[e]).max() * r[e].size
        assert abs(tot) <= 64 * np.finfo(float).eps * scale, (e, tot, scale)
    if N == 2:
        # Σ_i α_i = 1 is preserved (β of 1-α equals β of α; same face velocity)
        sa = r[N + ndim + 1] + r[N + ndim + 2]
        assert np.abs(sa).max() <= 1e-12 * np.abs(r[N + ndim + 1]).max()


def test_rhs_cells_agrees_with_full_rhs():
    pb = W.random_problem(3, (10, 9, 8), 2, "water")
    P = _oprob(pb)
    q = _cons(pb, W.random_prims(pb))
    qp = O.pad(P, q)
    rfull = O.unpad(P, O.rhs_padded(P, qp))
    rng = np.random.default_rng(0)
    cells = np.stack([rng.integers(0, m, 50) for m in pb.n], axis=1)
    rc = O.rhs_cells(P, qp, cells)
    ref = rfull[:, cells[:, 2], cells[:, 1], cells[:, 0]].T
    assert np.array_equal(rc, ref)


@pytest.mark.parametrize("mats,p0", [("gas", 1.0), ("water", 1.0e5)])
def test_pressure_velocity_equilibrium_100_steps(mats, p0):
    """I3: uniform p and u, stepped α and ρ_i: after 100 RK3 steps p and u stay uniform
    to round-off, amplified only by the stiffened-gas cancellation Π/(Γp)."""
    n = 64
    if mats == "gas":
        gam, pinf, rho = (1.4, 1.648), (0.0, 0.0), (1.0, 0.182)
    else:
        gam, pinf, rho = (4.4, 1.4), (6e8, 0.0), (1000.0, 1.2)
    pb = W.Problem("eq", 2, 1, (n, 1, 1), gamma=gam, pi_inf=pinf, bc=(W.BC_PERIODIC,) * 6)
    X = pb.centres()[0]
    a1 = np.where((X > 0.3) & (X < 0.6), 1 - 1e-6, 1e-6) * np.ones((1, 1, n))
    u0 = 0.5 * (1.0 if mats == "gas" else 400.0)
    v = np.stack([a1 * rho[0], (1 - a1) * rho[1], np.full_like(a1, u0), np.full_like(a1, p0),
                  a1, 1 - a1])
    P = _oprob(pb)
    q = _cons(pb, v)
    c = 3.0 if mats == "gas" else 1700.0
    dt = 0.4 * pb.dx[0] / (c + u0)
    q = O.rk3_step(P, q, dt, nsteps=100)
    vv = O.cons_to_prim(P, q)
    G, Pi = O.constants(P)
    amp = 1 + max(Pi[i] / (G[i] * p0) for i in range(2))
    assert np.abs(vv[3] / p0 - 1).max() <= 1e-13 * amp
    assert np.abs(vv[2] / u0 - 1).max() <= 1e-13 * amp
    # the interface did move (the test is not trivially static)
    assert np.abs(vv[4] - v[4]).max() > 0.1


def test_axis_permutation_bitwise():
    """I4: a 1D problem laid along x, y or z of a 3D grid gives identical results."""
    n = 20
    pb1 = W.random_problem(1, (n,), 2, "water")
    v1 = W.random_prims(pb1, seed=11)           # (E1, 1, 1, n): rho1 rho2 u p a1 a2
    base = [v1[0, 0, 0], v1[1, 0, 0], v1[2, 0, 0], v1[3, 0, 0], v1[4, 0, 0], v1[5, 0, 0]]
    outs = []
    for axis in range(3):
        shape = [3, 3, 3]
        shape[2 - axis] = n
        pb = W.Problem("perm", 2, 3, tuple(shape[::-1]), hi=tuple(s / n for s in shape[::-1]),
                       gamma=pb1.gamma, pi_inf=pb1.pi_inf, bc=(W.BC_PERIODIC,) * 6)
        bshape = [1, 1, 1]
        bshape[2 - axis] = n

        def f(a):
            return np.broadcast_to(a.reshape(bshape), shape)
        vel = [np.zeros(shape)] * 3
        vel = [f(base[2]) if k == axis else np.zeros(shape) for k in range(3)]
        v = np.stack([f(base[0]), f(base[1])] + vel + [f(base[3]), f(base[4]), f(base[5])])
        r = O.rhs(_oprob(pb), _cons(pb, v))
        sel = [0, 0, 0]
        sel[2 - axis] = slice(None)
        rr = r[(slice(None),) + tuple(sel)]
        outs.append(np.stack([rr[0], rr[1], rr[2 + axis], rr[5], rr[6], rr[7]]))
        others = [2 + k for k in range(3) if k != axis]
        assert np.all(r[others] == 0.0)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_decomposition_emulation_bitwise():
    """I5: P z-subdomains with ghost layers copied from neighbours == one domain."""
    pb = W.random_problem(3, (8, 6, 12), 2, "water")
    P = _oprob(pb)
    q = _cons(pb, W.random_prims(pb))
    ref = O.rhs(P, q)
    g = O.oracle.G
    parts = 3
    nzl = pb.n[2] // parts
    out = []
    for r_ in range(parts):
        sub = W.Problem("sub", 2, 3, (pb.n[0], pb.n[1], nzl), hi=(pb.hi[0], pb.hi[1], pb.hi[2] / parts),
                        gamma=pb.gamma, pi_inf=pb.pi_inf,
                        bc=(W.BC_PERIODIC,) * 4 + (O.BC_EXTERNAL, O.BC_EXTERNAL))
        Ps = _oprob(sub)
        qs = O.pad(Ps, q[:, r_ * nzl:(r_ + 1) * nzl])
        # neighbour ghost planes (periodic across ranks), interior x/y only
        for j in range(g):
            lo = ((r_ * nzl - 1 - j) % pb.n[2])
            hi = (((r_ + 1) * nzl + j) % pb.n[2])
            qs[:, g - 1 - j, g:g + pb.n[1], g:g + pb.n[0]] = q[:, lo]
            qs[:, g + nzl + j, g:g + pb.n[1], g:g + pb.n[0]] = q[:, hi]
        out.append(O.unpad(Ps, O.rhs_padded(Ps, qs)))
    assert np.array_equal(np.concatenate(out, axis=1), ref)


def _wave_rhs_error(n):
    pb = W.entropy_wave_problem(n)
    v = W.entropy_wave_prims(pb, cell_average=True)
    P = _oprob(pb)
    r = O.rhs(P, _cons(pb, v))
    # exact: u = 1, p = 1 uniform -> ∂q/∂t = -(Q(x+h/2) - Q(x-h/2))/h for every conserved
    # Q written from the point values of α1 (closed form, ρ1=1, ρ2=0.5, γ=1.4/1.6)
    h = pb.dx[0]
    X = pb.centres()[0][0, 0]

    def Q(x):
        a = 0.5 + 0.25 * np.sin(2 * np.pi * x)
        r1, r2 = a * 1.0, (1 - a) * 0.5
        rho = r1 + r2
        rhoE = a / 0.4 + (1 - a) / 0.6 + 0.5 * rho
        return np.stack([r1, r2, rho, rhoE, a, 1 - a])
    exact = -(Q(X + h / 2) - Q(X - h / 2)) / h
    return np.abs(r[:, 0, 0, :] - exact).mean(axis=1)


def test_rhs_fifth_order_convergence():
    ns = [16, 32, 64, 128]
    errs = np.array([_wave_rhs_error(n) for n in ns])     # (len(ns), E)
    orders = np.log2(errs[:-1] / errs[1:])
    assert orders[1:].min() > 4.5, orders


def test_rk3_amplification_factor():
    """S4 on y' = λy: one step multiplies by 1 + z + z²/2 + z³/6, z = λ dt."""
    rng = np.random.default_rng(12)
    y0 = rng.standard_normal(64)
    lam = rng.uniform(-3, 0.5, 64) + 0.0
    dt = 0.3
    q1 = O.rk3_combine(1, y0, y0, lam * y0, dt)
    q2 = O.rk3_combine(2, y0, q1, lam * q1, dt)
    q3 = O.rk3_combine(3, y0, q2, lam * q2, dt)
    z = lam * dt
    assert np.allclose(q3, (1 + z + z * z / 2 + z ** 3 / 6) * y0, rtol=1e-14, atol=1e-15)


def test_rk3_third_order_in_time():
    pb = W.entropy_wave_problem(32)
    P = _oprob(pb)
    q0 = _cons(pb, W.entropy_wave_prims(pb))
    T = 0.25

    def run(m):
        return O.rk3_step(P, q0, T / m, nsteps=m)
    fine = run(256)
    errs = [np.abs(run(m) - fine).max() for m in (8, 16, 32)]
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert orders.min() > 2.8, orders


def test_max_wave_rate_closed_form():
    """Uniform single stiffened gas: rate = max_k (|u_k| + sqrt(gamma (p + pi_inf)/rho))/dx_k."""
    for gam, pinf, rho, p in ((1.4, 0.0, 1.2, 1e5), (4.4, 6e8, 1000.0, 1e5)):
        pb = W.Problem("uni", 1, 3, (6, 5, 4), hi=(0.6, 1.0, 0.2), gamma=(gam,), pi_inf=(pinf,))
        u = (3.0, -250.0, 40.0)
        v = np.stack([np.full(pb.shape[1:], x) for x in (rho, *u, p, 1.0)])
        P = _oprob(pb)
        rate = O.max_wave_rate(P, _cons(pb, v))
        c = np.sqrt(gam * (p + pinf) / rho)
        ref = max((abs(u[k]) + c) / pb.dx[k] for k in range(3))
        assert rate == pytest.approx(ref, rel=1e-14)
