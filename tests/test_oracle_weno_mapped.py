"""Pins for the oracle's WENO5-M (SURVEY §8(f) F2 "mapped WENO-M"; Henrick, Aslam &
Powers, JCP 207 (2005) 542): Jiang-Shu weights mapped by
g_k(w) = w (d_k + d_k^2 - 3 d_k w + w^2) / (d_k^2 + w (1 - 2 d_k)) and renormalised.

- the mapping fixes the linear weights (g_k(d_k) = d_k), so linear data keeps omega = d;
- every candidate is exact on cell averages of quadratics, so any normalised weights are;
- mirror symmetry of v- and v+;
- ENO: across a jump the stencils that straddle it get (almost) no weight;
- the point of the mapping (Henrick et al. §3): at a critical point (f' = 0, f'' != 0)
  the reconstruction stays fifth-order, on Henrick's test function
  f(x) = sin(pi x - sin(pi x)/pi), where WENO5-JS with a small eps does not.  A mapping
  with a dropped or wrong term fails the order test or the fixed-point test.
"""
import numpy as np

import oracle as O

GL_X, GL_W = np.polynomial.legendre.leggauss(20)


def _avg(f, a, b):
    x = 0.5 * (b - a) * GL_X + 0.5 * (a + b)
    return 0.5 * np.dot(GL_W, f(x))


def test_linear_data_keeps_linear_weights():
    for slope in (1e-3, 1.0, -7.5):
        data = [2.0 + slope * k for k in range(5)]
        _, wm = O.weno5m_minus(*data)
        _, wp = O.weno5m_plus(*data)
        assert np.allclose(wm, [0.1, 0.6, 0.3], rtol=0, atol=1e-14)
        assert np.allclose(wp, [0.3, 0.6, 0.1], rtol=0, atol=1e-14)


def test_exact_on_quadratics():
    rng = np.random.default_rng(11)
    for _ in range(200):
        c = rng.uniform(-5, 5, 3)
        h = rng.uniform(0.01, 1.0)
        x0 = rng.uniform(-2, 2)
        f = lambda x: c[0] + c[1] * x + c[2] * x * x
        avg = [_avg(f, x0 + (k - 0.5) * h, x0 + (k + 0.5) * h) for k in range(-2, 3)]
        scale = max(abs(a) for a in avg) + 1
        vm, w = O.weno5m_minus(*avg)
        vp, _ = O.weno5m_plus(*avg)
        assert abs(w.sum() - 1.0) < 1e-14
        assert abs(vm - f(x0 + h / 2)) < 1e-12 * scale
        assert abs(vp - f(x0 - h / 2)) < 1e-12 * scale


def test_mirror_symmetry():
    rng = np.random.default_rng(12)
    for _ in range(300):
        v = rng.standard_normal(5) * 10 ** rng.uniform(-3, 3)
        vm, wm = O.weno5m_minus(*v)
        vp, wp = O.weno5m_plus(*v[::-1])
        assert abs(vm - vp) <= 1e-14 * np.abs(v).max()
        assert np.allclose(wm, wp[::-1], rtol=0, atol=1e-13)


def test_eno_at_a_jump():
    # jump between cells m and m+1: stencils 1 and 2 of v- straddle it
    data = [1.0, 1.0, 1.0, 10.0, 10.0]
    _, wm = O.weno5m_minus(*data)
    assert wm[0] > 1.0 - 1e-12 and wm[1] < 1e-12 and wm[2] < 1e-12


def _orders(fn, eps, off):
    f = lambda x: np.sin(np.pi * x - np.sin(np.pi * x) / np.pi)
    # critical point: pi x - sin(pi x)/pi = pi/2, by bisection on [0, 1]
    lo, hi = 0.0, 1.0
    g = lambda x: np.pi * x - np.sin(np.pi * x) / np.pi - np.pi / 2
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if g(mid) < 0 else (lo, mid)
    xc = 0.5 * (lo + hi)
    errs = []
    for k in range(4, 9):
        h = 2.0 ** -k
        face = xc + off * h                       # the face x_{m+1/2}
        cen = face - 0.5 * h + np.arange(-2, 3) * h
        avg = [_avg(f, c - h / 2, c + h / 2) for c in cen]
        v, _ = fn(*avg, eps=eps)
        errs.append(abs(v - f(face)))
    return [np.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]


def test_fifth_order_at_a_critical_point():
    for off in (0.0, 0.3):
        om = _orders(O.weno5m_minus, 1e-40, off)
        assert min(om[-3:]) > 4.7, (off, om)
    # negative control: the unmapped weights lose the order there (Henrick et al. §2)
    oj = _orders(O.weno5_minus, 1e-40, 0.0)
    assert min(oj) < 4.0, oj


def test_mapped_rhs_converges_at_fifth_order():
    """Full RHS (mapped weights) of a smooth two-fluid periodic wave: order >= 4.8."""
    import paper_2409_10729_b200.workloads as W  # noqa: F401  (inputs only)
    errs = []
    ns = (16, 32, 64)
    for n in ns:
        P = O.Problem(N=1, d=1, n=(n,), dx=(1.0 / n,), bc=(-1,) * 6, gamma=(1.4,),
                      pi_inf=(0.0,), eps=1e-16, weno_mapped=1)
        x = (np.arange(n) + 0.5) / n
        # density wave advected at u = 1, p = 1: rho = 1 + 0.5 sin(2 pi x) (cell averages)
        h = 1.0 / n
        rho = 1.0 + 0.5 * (np.cos(2 * np.pi * (x - h / 2)) - np.cos(2 * np.pi * (x + h / 2))) / (2 * np.pi * h)
        v = np.stack([rho, np.ones(n), np.ones(n), np.ones(n)])[:, None, None, :]
        q = O.prim_to_cons(P, v)
        L = O.rhs(P, q)
        # exact: d(rho)/dt = -d(rho u)/dx averaged over the cell
        ex = -(np.sin(2 * np.pi * (x + h / 2)) - np.sin(2 * np.pi * (x - h / 2))) * 0.5 / h
        errs.append(np.abs(L[0, 0, 0] - ex).mean())
    orders = [np.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert min(orders) > 4.8, orders
