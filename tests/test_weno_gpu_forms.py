"""The algebra of the GPU's WENO5 forms, checked on the CPU against the oracle.

`csrc/physics.cuh` evaluates WENO5-JS in two rearranged
forms that are not written the way the specification is:
  * `weno5_d` (the lean form): integer-scaled linear weights, candidates from the
    differences D0..D3;
  * `weno5_fewop_d`: every candidate correction ONE operation on the beta differences
    s_k, r_k (X = ((2/3)s0 + D1, 3r1 + s1, D2 - r2) for v-, -(r0 + D1, 3r1 - s1,
    D2 - (2/3)s2) for v+) over the denominators 2P0 + 12P1 + 6P2 and 6P0 + 12P1 + 2P2;
  * `weno5_fewop_s`: the same with the curvature terms S_k = (13/3)s_k^2 + eps' formed
    first (shared between neighbouring cells by the x pair and carried by the marches),
    r0 either 3D1 - D0 or 2D1 + s0.
All three are transcribed here operation by operation in numpy (fp64, same order; numpy
does not contract a*b+c, so the products round separately -- the identity, not the
rounding, is what this checks) and compared with the oracle's weno5_minus/plus
(`oracle/mfc_oracle.c`, the plain alpha_k = d_k/(beta_k+eps)^2, omega = alpha/sum
definition) on random stencils spanning many scales, steps and near-uniform data.
The GPU parity tests (`-m gpu`) check the kernels themselves.
"""
import numpy as np

import oracle as O

K133, K23 = 13.0 / 3.0, 2.0 / 3.0


def _beta_terms(D0, D1, D2, D3, eps4):
    s = (D1 - D0, D2 - D1, D3 - D2)
    r = (3.0 * D1 - D0, D1 + D2, D3 - 3.0 * D2)
    t = [(K133 * sk * sk + (rk * rk + eps4)) ** 2 for sk, rk in zip(s, r)]
    P = (t[1] * t[2], t[0] * t[2], t[0] * t[1])
    return s, r, P


def weno5_lean(a, b, c, d, e, eps):
    D0, D1, D2, D3 = b - a, c - b, d - c, e - d
    s, r, (P0, P1, P2) = _beta_terms(D0, D1, D2, D3, 4.0 * eps)
    xm = (5.0 / 6.0 * D1 - 1.0 / 3.0 * D0, 2.0 * D2 + D1, 2.0 * D2 - 0.5 * D3)
    Dm = 6.0 * P1 + (3.0 * P2 + P0)
    Nm = P2 * xm[2] + (P1 * xm[1] + P0 * xm[0])
    xp = (-2.0 * D1 + 0.5 * D0, -2.0 * D1 - D2, 1.0 / 3.0 * D3 - 5.0 / 6.0 * D2)
    Dp = 3.0 * P0 + (6.0 * P1 + P2)
    Np = P2 * xp[2] + (P1 * xp[1] + P0 * xp[0])
    return c + Nm / Dm, c + Np / Dp


def weno5_fewop(a, b, c, d, e, eps):
    D0, D1, D2, D3 = b - a, c - b, d - c, e - d
    (s0, s1, s2), (r0, r1, r2), (P0, P1, P2) = _beta_terms(D0, D1, D2, D3, 4.0 * eps)
    xm0, xm1, xm2 = K23 * s0 + D1, 3.0 * r1 + s1, D2 - r2
    Dm = 12.0 * P1 + (6.0 * P2 + 2.0 * P0)
    Nm = P2 * xm2 + (P1 * xm1 + P0 * xm0)
    yp0, yp1, yp2 = r0 + D1, 3.0 * r1 - s1, -K23 * s2 + D2
    Dp = 12.0 * P1 + (2.0 * P2 + 6.0 * P0)
    Np = P2 * yp2 + (P1 * yp1 + P0 * yp0)
    return c + Nm / Dm, c - Np / Dp


def weno5_fewop_s(a, b, c, d, e, eps, r0_from_s0=False):
    """`weno5_fewop_s` (x pair, marches): curvature terms S_k = (13/3)s_k^2 + eps' formed
    first, t_k = (r_k^2 + S_k)^2; r0 = 3D1 - D0, or 2D1 + s0 in the marches that carry s0."""
    D0, D1, D2, D3 = b - a, c - b, d - c, e - d
    s0, s1, s2 = D1 - D0, D2 - D1, D3 - D2
    S = [K133 * sk * sk + 4.0 * eps for sk in (s0, s1, s2)]
    r0 = 2.0 * D1 + s0 if r0_from_s0 else 3.0 * D1 - D0
    r1, r2 = D1 + D2, D3 - 3.0 * D2
    t = [(rk * rk + Sk) ** 2 for rk, Sk in zip((r0, r1, r2), S)]
    P0, P1, P2 = t[1] * t[2], t[0] * t[2], t[0] * t[1]
    xm0, xm1, xm2 = K23 * s0 + D1, 3.0 * r1 + s1, D2 - r2
    Dm = 12.0 * P1 + (6.0 * P2 + 2.0 * P0)
    Nm = P2 * xm2 + (P1 * xm1 + P0 * xm0)
    yp0, yp1, yp2 = r0 + D1, 3.0 * r1 - s1, -K23 * s2 + D2
    Dp = 12.0 * P1 + (2.0 * P2 + 6.0 * P0)
    Np = P2 * yp2 + (P1 * yp1 + P0 * yp0)
    return c + Nm / Dm, c - Np / Dp


def weno5_fewop_s_march(a, b, c, d, e, eps):
    return weno5_fewop_s(a, b, c, d, e, eps, r0_from_s0=True)


def _stencils(n=4000, seed=10729):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        kind = i % 4
        v = rng.standard_normal(5) * 10.0 ** rng.uniform(-4, 9)
        if kind == 1:                      # a step somewhere in the stencil
            v[rng.integers(1, 5):] += rng.standard_normal() * 10.0 ** rng.uniform(0, 9)
        elif kind == 2:                    # near-uniform (beta ~ eps regime)
            v = rng.uniform(0.5, 2.0) + rng.standard_normal(5) * 10.0 ** rng.uniform(-17, -6)
        elif kind == 3:                    # smooth: samples of a sine
            h = 10.0 ** rng.uniform(-4, -1)
            v = np.sin(rng.uniform(0, 6) + h * np.arange(5)) * 10.0 ** rng.uniform(-3, 9)
        out.append(v)
    return out


def _check(form, eps):
    for v in _stencils():
        vm_ref, _ = O.weno5_minus(*v, eps=eps)
        vp_ref, _ = O.weno5_plus(*v, eps=eps)
        vm, vp = form(*v, eps)
        scale = np.abs(v).max()
        assert abs(vm - vm_ref) <= 4e-15 * scale, (form.__name__, v, vm, vm_ref)
        assert abs(vp - vp_ref) <= 4e-15 * scale, (form.__name__, v, vp, vp_ref)


def test_lean_form_equals_specification():
    for eps in (1e-16, 1e-6, 1e-40):
        _check(weno5_lean, eps)


def test_fewop_form_equals_specification():
    for eps in (1e-16, 1e-6, 1e-40):
        _check(weno5_fewop, eps)


def test_curvature_term_forms_equal_specification():
    for eps in (1e-16, 1e-6, 1e-40):
        _check(weno5_fewop_s, eps)
        _check(weno5_fewop_s_march, eps)


def test_fewop_candidate_identities():
    """The one-operation candidate corrections are the specification's 6(p_k - c),
    scaled by (1/3, 2, 1) for v- and (1, 2, 1/3) for v+ (exact on integers)."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        a, b, c, d, e = (float(x) for x in rng.integers(-1000, 1000, 5))
        D0, D1, D2, D3 = b - a, c - b, d - c, e - d
        s0, s1, s2 = D1 - D0, D2 - D1, D3 - D2
        r0, r1, r2 = 3 * D1 - D0, D1 + D2, D3 - 3 * D2
        Am = (2 * a - 7 * b + 11 * c - 6 * c, -b + 5 * c + 2 * d - 6 * c, 2 * c + 5 * d - e - 6 * c)
        Ap = (-a + 5 * b + 2 * c - 6 * c, 2 * b + 5 * c - d - 6 * c, 11 * c - 7 * d + 2 * e - 6 * c)
        assert 3 * (K23 * s0 + D1) == Am[0] or abs(3 * (K23 * s0 + D1) - Am[0]) < 1e-9
        assert 3 * r1 + s1 == 2 * Am[1]
        assert D2 - r2 == Am[2]
        assert -(r0 + D1) == Ap[0]
        assert -(3 * r1 - s1) == 2 * Ap[1]
        assert abs(-3 * (D2 - K23 * s2) - Ap[2]) < 1e-9


def _weno5m_sums(a, A, d, W):
    """`weno5m_sums_a`: mapped, un-normalised weights Q_k = num_k den_i den_j of one side
    from the Jiang-Shu weights a_k = d_k P_k."""
    num, den = [], []
    for k in range(3):
        w = a[k] * W
        num.append(w * (w * (w - 3.0 * d[k]) + (d[k] * d[k] + d[k])))
        den.append(w * (1.0 - 2.0 * d[k]) + d[k] * d[k])
    Q = (num[0] * (den[1] * den[2]), num[1] * (den[0] * den[2]), num[2] * (den[0] * den[1]))
    return Q[2] * A[2] + (Q[1] * A[1] + Q[0] * A[0]), (Q[0] + Q[1]) + Q[2]


def weno5m_one_rcp(a, b, c, d, e, eps):
    """`weno5m` with MFC_WENO5M_ONE_RCP and MFC_WENO5M_ALPHA: both sides together,
    1/Zm = Zp/(Zm Zp) and 1/Sm = Sp/(Sm Sp) (one reciprocal per pair of divisions), the
    weights a_k = d_k P_k formed once."""
    D0, D1, D2, D3 = b - a, c - b, d - c, e - d
    _, _, P = _beta_terms(D0, D1, D2, D3, 4.0 * eps)
    Am = (5.0 * D1 - 2.0 * D0, 2.0 * D2 + D1, 4.0 * D2 - D3)
    Ap = (-4.0 * D1 + D0, -2.0 * D1 - D2, 2.0 * D3 - 5.0 * D2)
    dm, dp = (0.1, 0.6, 0.3), (0.3, 0.6, 0.1)
    a1 = 0.6 * P[1]
    am, ap = (0.1 * P[0], a1, 0.3 * P[2]), (0.3 * P[0], a1, 0.1 * P[2])
    Zm, Zp = (am[0] + am[1]) + am[2], (ap[0] + ap[1]) + ap[2]
    R1 = 1.0 / (Zm * Zp)
    Nm, Sm = _weno5m_sums(am, Am, dm, Zp * R1)
    Np, Sp = _weno5m_sums(ap, Ap, dp, Zm * R1)
    R2 = 1.0 / (Sm * Sp) * (1.0 / 6.0)
    return c + Nm * Sp * R2, c + Np * Sm * R2


def test_weno5m_one_rcp_form_equals_oracle():
    """The two-sided WENO5-M form against the oracle's
    orc_weno5m_minus/plus (pinned in test_oracle_weno_mapped.py), over the same stencil
    mix (values up to ~1e9 and steps up to ~1e9: Zm Zp ~ P^2 stays finite)."""
    for eps in (1e-16, 1e-6):
        for v in _stencils(2000):
            vm_ref = O.weno5m_minus(*v, eps=eps)
            vp_ref = O.weno5m_plus(*v, eps=eps)
            vm_ref = vm_ref[0] if isinstance(vm_ref, tuple) else vm_ref
            vp_ref = vp_ref[0] if isinstance(vp_ref, tuple) else vp_ref
            vm, vp = weno5m_one_rcp(*v, eps)
            scale = np.abs(v).max()
            assert np.isfinite(vm) and np.isfinite(vp)
            assert abs(vm - vm_ref) <= 1e-14 * scale, (v, vm, vm_ref)
            assert abs(vp - vp_ref) <= 1e-14 * scale, (v, vp, vp_ref)


def weno3_one_rcp(a, b, c, eps):
    """`weno3` with MFC_WENO3_ONE_RCP: 1/Zm = Zp/(Zm Zp), 1/Zp = Zm/(Zm Zp)."""
    D0, D1 = b - a, c - b
    t0, t1 = (D0 * D0 + eps) ** 2, (D1 * D1 + eps) ** 2
    wm0, wm1 = t1 * (1.0 / 3.0), t0 * (2.0 / 3.0)
    wp0, wp1 = t1 * (2.0 / 3.0), t0 * (1.0 / 3.0)
    Zm, Zp = wm0 + wm1, wp0 + wp1
    R = 1.0 / (Zm * Zp) * 0.5
    return b + (wm1 * D1 + wm0 * D0) * Zp * R, b - (wp1 * D1 + wp0 * D0) * Zm * R


def test_weno3_one_rcp_form_equals_oracle():
    """The two-sided WENO3 form (F2, AMB-26) against the oracle's orc_weno3_minus/plus on
    the stencil mix, at both ends of mfc_set_weno_eps's range."""
    for eps in (1e-16, 1e-30, 1e-2):
        for v in _stencils(2000):
            a, b, c = v[1], v[2], v[3]
            vm_ref, _ = O.weno3_minus(a, b, c, eps=eps)
            vp_ref, _ = O.weno3_plus(a, b, c, eps=eps)
            vm, vp = weno3_one_rcp(a, b, c, eps)
            scale = max(abs(a), abs(b), abs(c))
            assert abs(vm - vm_ref) <= 4e-15 * scale, (v, vm, vm_ref)
            assert abs(vp - vp_ref) <= 4e-15 * scale, (v, vp, vp_ref)
