"""Pins for the oracle's WENO5-JS (S3; PAPER.md:84 citing Shu [15]).

- every candidate stencil is exact on cell averages of quadratics, so the
  reconstruction is exact there whatever the nonlinear weights are;
- linear data gives equal smoothness indicators, so ω equals the linear weights;
- v⁺ is the mirror image of v⁻;
- fifth-order accuracy on smooth data (L1), and the linear-weight combination equals
  the unique quartic-exact (5-cell) reconstruction.
"""
import numpy as np

import oracle as O


def _avg_quadratic(c, xl, xr):
    # cell average of c0 + c1 x + c2 x^2 over [xl, xr]
    F = lambda x: c[0] * x + c[1] * x ** 2 / 2 + c[2] * x ** 3 / 3
    return (F(xr) - F(xl)) / (xr - xl)


def test_exact_on_quadratics_any_weights():
    rng = np.random.default_rng(5)
    for _ in range(200):
        c = rng.uniform(-5, 5, 3)
        h = rng.uniform(0.01, 1)
        x0 = rng.uniform(-2, 2)
        xs = x0 + h * np.arange(-2, 3)
        avg = [_avg_quadratic(c, x - h / 2, x + h / 2) for x in xs]
        f = lambda x: c[0] + c[1] * x + c[2] * x * x
        vm, _ = O.weno5_minus(*avg)
        vp, _ = O.weno5_plus(*avg)
        scale = max(abs(a) for a in avg) + abs(f(x0 + h / 2)) + 1
        assert abs(vm - f(x0 + h / 2)) < 1e-13 * scale
        assert abs(vp - f(x0 - h / 2)) < 1e-13 * scale


def test_linear_data_gives_linear_weights():
    for slope in (1e-3, 1.0, 7.5, -2.0):
        data = [3.0 + slope * k for k in range(5)]
        _, wm = O.weno5_minus(*data)
        _, wp = O.weno5_plus(*data)
        assert np.allclose(wm, [0.1, 0.6, 0.3], rtol=0, atol=1e-12)
        assert np.allclose(wp, [0.3, 0.6, 0.1], rtol=0, atol=1e-12)
    # constant data: β = 0 -> weights exactly the linear ones (ε only)
    _, wm = O.weno5_minus(2.0, 2.0, 2.0, 2.0, 2.0)
    assert np.allclose(wm, [0.1, 0.6, 0.3], rtol=1e-15)


def test_linear_weights_give_fifth_order_stencil():
    """With ω = d the reconstruction is the 5-cell stencil exact for quartics:
    v⁻_{m+½} = (2a − 13b + 47c + 27d − 3e)/60 (standard WENO5 optimal stencil)."""
    rng = np.random.default_rng(6)
    for _ in range(100):
        # cell averages of a quartic at unit spacing
        c = rng.uniform(-1, 1, 5)
        F = lambda x: sum(c[k] * x ** (k + 1) / (k + 1) for k in range(5))
        avg = [F(m + 0.5) - F(m - 0.5) for m in range(-2, 3)]
        f = lambda x: sum(c[k] * x ** k for k in range(5))
        # huge ε forces linear weights
        vm, w = O.weno5_minus(*avg, eps=1e15)
        assert np.allclose(w, [0.1, 0.6, 0.3], atol=1e-9)
        assert abs(vm - f(0.5)) < 1e-8
        vp, _ = O.weno5_plus(*avg, eps=1e15)
        assert abs(vp - f(-0.5)) < 1e-8


def test_mirror_symmetry():
    rng = np.random.default_rng(7)
    for _ in range(500):
        d = rng.standard_normal(5) * 10 ** rng.uniform(-3, 3)
        vp, wp = O.weno5_plus(*d)
        vm, wm = O.weno5_minus(*d[::-1])
        assert abs(vp - vm) <= 1e-13 * (np.abs(d).max())
        assert np.allclose(wp, wm[::-1], atol=1e-12)


def test_eno_property_at_a_step():
    """Near a jump the reconstruction stays within the data range (non-oscillatory)."""
    for k in range(5):
        d = [0.0] * k + [1.0] * (5 - k)
        vm, _ = O.weno5_minus(*d)
        vp, _ = O.weno5_plus(*d)
        assert -1e-10 <= vm <= 1 + 1e-10 and -1e-10 <= vp <= 1 + 1e-10


def test_fifth_order_convergence_smooth():
    errs = []
    ns = [16, 32, 64, 128]
    for n in ns:
        h = 1.0 / n
        x = (np.arange(n) + 0.5) * h
        avg = 1 + 0.5 * (np.cos(2 * np.pi * (x - h / 2)) - np.cos(2 * np.pi * (x + h / 2))) / (2 * np.pi * h)
        err = 0.0
        for m in range(n):
            st = [avg[(m + s) % n] for s in range(-2, 3)]
            vm, _ = O.weno5_minus(*st)
            err += abs(vm - (1 + 0.5 * np.sin(2 * np.pi * (x[m] + h / 2)))) * h
        errs.append(err)
    orders = [np.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert min(orders[1:]) > 4.5, orders


# ----------------------------------------------------------------- WENO3 (F2)

def test_weno3_exact_on_linear_and_linear_weights():
    rng = np.random.default_rng(15)
    for _ in range(200):
        c0, c1 = rng.uniform(-5, 5, 2)
        h = rng.uniform(0.01, 1)
        x0 = rng.uniform(-2, 2)
        avg = [c0 + c1 * (x0 + k * h) for k in (-1, 0, 1)]     # cell averages of a line
        vm, wm = O.weno3_minus(*avg)
        vp, wp = O.weno3_plus(*avg)
        scale = max(abs(a) for a in avg) + 1
        assert abs(vm - (c0 + c1 * (x0 + h / 2))) < 1e-13 * scale
        assert abs(vp - (c0 + c1 * (x0 - h / 2))) < 1e-13 * scale
        assert np.allclose(wm, [1 / 3, 2 / 3], atol=1e-12) and np.allclose(wp, [2 / 3, 1 / 3], atol=1e-12)


def test_weno3_linear_weights_give_third_order_stencil():
    """With the linear weights the reconstruction is the 3-cell stencil exact for
    quadratics: v-_{m+1/2} = (-a + 5b + 2c)/6."""
    rng = np.random.default_rng(16)
    for _ in range(100):
        c = rng.uniform(-1, 1, 3)
        F = lambda x: c[0] * x + c[1] * x ** 2 / 2 + c[2] * x ** 3 / 3
        avg = [F(m + 0.5) - F(m - 0.5) for m in (-1, 0, 1)]
        f = lambda x: c[0] + c[1] * x + c[2] * x * x
        vm, _ = O.weno3_minus(*avg, eps=1e15)
        vp, _ = O.weno3_plus(*avg, eps=1e15)
        assert abs(vm - f(0.5)) < 1e-9 and abs(vp - f(-0.5)) < 1e-9


def test_weno3_mirror_and_eno():
    rng = np.random.default_rng(17)
    for _ in range(300):
        d = rng.standard_normal(3) * 10 ** rng.uniform(-3, 3)
        assert abs(O.weno3_plus(*d)[0] - O.weno3_minus(*d[::-1])[0]) <= 1e-13 * np.abs(d).max()
    for k in range(3):
        d = [0.0] * k + [1.0] * (3 - k)
        assert -1e-10 <= O.weno3_minus(*d)[0] <= 1 + 1e-10


def test_weno3_rhs_convergence():
    """Full RHS with WENO3 on the advected two-fluid wave: order >= 1.9 in L1 (WENO3-JS
    drops to second order at smooth extrema)."""
    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0])
    from paper_2409_10729_b200 import workloads as W
    errs = []
    for n in (32, 64, 128, 256):
        pb = W.entropy_wave_problem(n)
        pb.weno_order = 3
        P = O.Problem.from_spec(pb)
        v = W.entropy_wave_prims(pb)
        r = O.rhs(P, O.prim_to_cons(P, v))
        h = pb.dx[0]
        X = pb.centres()[0][0, 0]
        a = lambda x: 0.5 + 0.25 * np.sin(2 * np.pi * x)
        exact = -(a(X + h / 2) - a(X - h / 2)) / h
        errs.append(np.abs(r[4, 0, 0] - exact).mean())
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert orders[-1] > 1.9, orders
