"""Helpers shared by the GPU parity tests: run the same seeded input through the
oracle (CPU, fp64) and through libmfc (GPU, via the C ABI) and compare with the
metric of DESIGN.md AMB-17:

    per equation e:  max_cells |gpu_e - cpu_e| / scale_e  <= tol
    RHS, flux-scaled: scale_e = max( max_cells |cpu_e| ,  Phi_e / dx_min )
    RHS, strict:      scale_e = max_cells |cpu_e|
    state:            scale_e = max_cells |cpu_e|
    (and gpu == 0 exactly wherever the oracle's whole output e is identically 0).

Phi_e is the magnitude of equation e's face flux (a_max = max(|u| + c)):
    partial densities, volume fractions: max|q_e| * a_max
    every momentum component:           max(rho) * a_max^2   (bounds rho u^2 + p)
    energy:                             (max|rhoE| + max|p|) * a_max
Rounding in any correct implementation of the flux difference is relative to
Phi_e / dx, so the flux-scaled error is asserted <= 1e-12 for every equation, and the
STRICT error (the north star's "1e-12 relative" read literally) for every equation
whose RHS is not itself a cancellation of much larger fluxes: cond_e =
(Phi_e/dx) / max|cpu_e| <= COND_STRICT.  An equation above that (the air partial
density at rest in C1, the zero tangential momenta of C2/C3/C5 where p is uniform
along the sweep, alpha of a single fluid) has an exact RHS that is ~0 and an oracle
RHS that is rounding noise of size ~eps * Phi_e/dx; its strict error is recorded in
the parity log (per equation, with cond_e) and listed in DESIGN.md, not asserted.
"""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2409_10729_b200 import workloads as W

RHS_TOL = 1e-12       # BASELINE.json north_star: per RHS evaluation
STEP100_TOL = 1e-10   # BASELINE.json north_star: after 100 RK3 steps
COND_STRICT = 1e2     # strict 1e-12 asserted where the RHS is >= 1 % of its flux scale
FLUX_ULPS = 64 * np.finfo(float).eps   # and every equation within 64 ulp of its flux scale
# stretched grids: the oracle solves the cell-average systems, the library uses the
# primitive function's Lagrange derivatives -- two derivations of the coefficient tables
# that agree to a few ulp each, which the reconstruction of a strongly stretched random
# grid amplifies (worst seen: 1.2e-14 = 53 ulp, profiles/parity_fuzz_r213.json)
FLUX_ULPS_STRETCHED = 256 * np.finfo(float).eps

# achieved errors, written to $MFC_PARITY_LOG by tests/conftest.py at session end
RECORD = {}


def record(name: str, err, tol, strict=None, cond=None):
    RECORD[name] = {"max_err": float(np.max(err)), "tol": float(np.max(tol)),
                    "per_eq": [float(x) for x in np.atleast_1d(err)]}
    if strict is not None:
        RECORD[name]["strict_per_eq"] = [float(x) for x in np.atleast_1d(strict)]
        RECORD[name]["strict_max_err"] = float(np.max(strict))
    if cond is not None:
        RECORD[name]["cond_per_eq"] = [float(x) for x in np.atleast_1d(cond)]
        wc = np.atleast_1d(cond) <= COND_STRICT
        RECORD[name]["strict_max_err_well_conditioned"] = (
            float(np.max(np.atleast_1d(strict)[wc])) if wc.any() else 0.0)


def rel_err(gpu: np.ndarray, cpu: np.ndarray, floor=None) -> np.ndarray:
    """Per-equation normalised max error (AMB-17); floor[e] = flux scale (RHS only).
    Without a floor, an oracle output that is identically 0 requires gpu == 0 exactly
    (the strict metric; I1's exactly uniform states are tested that way separately); with
    the flux-scale floor the scale is the floor even then (an RHS that is 0 only by the
    luck of the oracle's rounding, e.g. a 3-cell periodic field uniform up to ulps)."""
    E = cpu.shape[0]
    out = np.zeros(E)
    for e in range(E):
        scale = np.abs(cpu[e]).max()
        if floor is not None:
            scale = max(scale, floor[e])
        diff = np.abs(gpu[e] - cpu[e]).max()
        if scale == 0.0:
            out[e] = 0.0 if diff == 0.0 else np.inf
        else:
            out[e] = diff / scale
    return out


def check_rhs(name: str, pb, v: np.ndarray, q: np.ndarray, got: np.ndarray, ref: np.ndarray,
              tol: float = RHS_TOL):
    """The RHS parity assertion of AMB-17: flux-scaled error <= tol for every equation,
    strict error <= tol for every well-conditioned equation; both recorded per equation."""
    phi = rhs_flux_scale(pb, v, q)
    flux = rel_err(got, ref, phi)
    strict = rel_err(got, ref)
    mx = np.abs(ref).reshape(ref.shape[0], -1).max(axis=1)
    cond = np.where(mx > 0, phi / np.where(mx > 0, mx, 1.0), np.inf)
    record(name, flux, tol, strict, cond)
    assert np.all(flux <= tol), (name, "flux-scaled", flux)
    ulps = FLUX_ULPS_STRETCHED if getattr(pb, "stretched", False) else FLUX_ULPS
    assert np.all(flux <= ulps), (name, "flux-scaled above the ulp bound", flux)
    wc = cond <= COND_STRICT
    assert np.all(strict[wc] <= tol), (name, "strict (well-conditioned)", strict, cond)
    return flux, strict, cond


def state_err(pb, got: np.ndarray, ref: np.ndarray) -> tuple:
    """State metric after k steps (AMB-17): max|gpu_e - cpu_e| / max|cpu_e| per equation,
    except that the momentum components are one vector and share its scale
    max_k max|cpu_(rho u_k)| (a tangential momentum that is identically 0 in exact
    arithmetic -- C3 before the shock reaches the droplet -- is otherwise compared as
    round-off against round-off).  Returns (metric, strict per-component errors)."""
    strict = rel_err(got, ref)
    N, d = pb.n_fluids, pb.ndim
    mom = np.abs(ref[N:N + d]).max()
    err = strict.copy()
    for e in range(N, N + d):
        diff = np.abs(got[e] - ref[e]).max()
        err[e] = 0.0 if diff == 0.0 else (diff / mom if mom > 0 else np.inf)
    return err, strict


def check_against_oracle(name: str, pb, v, q, rhs_gpu=None, state_gpu=None, dt=0.0,
                         nsteps=0):
    """A gathered multi-rank result (decomposed, fused-halo, IPC) against the ORACLE on
    the whole domain, not only against the GPU's own single-domain run: the RHS under
    check_rhs, the state after nsteps RK3 steps under the 1e-10 state metric."""
    P = O.Problem.from_spec(pb)
    if rhs_gpu is not None:
        check_rhs("rhs " + name, pb, v, q, rhs_gpu, O.rhs(P, q))
    if state_gpu is not None:
        ref = O.rk3_step(P, q, dt, nsteps=nsteps)
        err, strict = state_err(pb, state_gpu, ref)
        record(f"{nsteps} RK3 steps " + name, err, STEP100_TOL, strict)
        assert np.all(err <= STEP100_TOL), (name, err)


def oracle_inputs(pb: W.Problem, seed: int = W.SEED):
    """Seeded primitive fields -> conserved via the ORACLE's EOS (test infrastructure);
    the same conserved array is handed to both sides."""
    P = O.Problem.from_spec(pb)
    v = W.prims_for(pb, seed)
    q = O.prim_to_cons(P, v)
    return P, v, q


def gpu_solver(pb: W.Problem, **kw):
    from paper_2409_10729_b200.mfc import Solver
    return Solver(pb, **kw)


def gpu_rhs(pb: W.Problem, q: np.ndarray, **kw) -> np.ndarray:
    import torch
    s = gpu_solver(pb, **kw)
    qd = s.state_from_cons(q)
    r = s.rhs(qd)
    torch.cuda.synchronize()
    return s.interior(r).cpu().numpy()


def gpu_steps(pb: W.Problem, q: np.ndarray, dt: float, nsteps: int, **kw) -> np.ndarray:
    import torch
    s = gpu_solver(pb, **kw)
    qd = s.state_from_cons(q)
    for _ in range(nsteps):
        s.rk3_step(qd, dt)
    torch.cuda.synchronize()
    return s.interior(qd).cpu().numpy()


def max_wave_speed(pb: W.Problem, v: np.ndarray) -> float:
    N, d = pb.n_fluids, pb.ndim
    a = v[N + d + 1:]
    rho = v[:N].sum(axis=0)
    G = sum(a[i] / (pb.gamma[i] - 1) for i in range(N))
    Pi = sum(a[i] * pb.gamma[i] * pb.pi_inf[i] / (pb.gamma[i] - 1) for i in range(N))
    c = np.sqrt(((G + 1) * v[N + d] + Pi) / (rho * G))
    umax = sum(np.abs(v[N + k]) for k in range(d))
    return float((umax + c).max())


def rhs_flux_scale(pb: W.Problem, v: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Per-equation face-flux magnitude Phi_e over dx_min (see module docstring)."""
    N, d = pb.n_fluids, pb.ndim
    amax = max_wave_speed(pb, v)
    dxm = min(pb.dx[:d])
    rho = v[:N].sum(axis=0)
    phi = np.empty(q.shape[0])
    for e in range(q.shape[0]):
        if N <= e < N + d:
            phi[e] = rho.max() * amax * amax
        elif e == N + d:
            phi[e] = (np.abs(q[e]).max() + np.abs(v[e]).max()) * amax
        else:
            phi[e] = np.abs(q[e]).max() * amax
    return phi / dxm


def stable_dt(pb: W.Problem, v: np.ndarray, cfl: float = 0.3) -> float:
    """CFL time step from the primitive fields (sound speed of the mixture EOS computed
    from the generator's own material constants; test setup only)."""
    N, d = pb.n_fluids, pb.ndim
    a = v[N + d + 1:]
    rho = v[:N].sum(axis=0)
    G = sum(a[i] / (pb.gamma[i] - 1) for i in range(N))
    Pi = sum(a[i] * pb.gamma[i] * pb.pi_inf[i] / (pb.gamma[i] - 1) for i in range(N))
    c = np.sqrt(((G + 1) * v[N + d] + Pi) / (rho * G))
    umax = max(np.abs(v[N + k]).max() for k in range(d))
    return cfl * min(pb.dx[:d]) / (umax + c.max())
