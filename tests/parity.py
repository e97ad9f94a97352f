"""Helpers shared by the GPU parity tests: run the same seeded input through the
oracle (CPU, fp64) and through libmfc (GPU, via the C ABI) and compare with the
metric of DESIGN.md AMB-17:

    per equation e:  max_cells |gpu_e - cpu_e| / scale_e  <= tol
    RHS:   scale_e = max( max_cells |cpu_e| ,  max_cells |q_e| * a_max / dx_min )
    state: scale_e = max_cells |cpu_e|
    (and gpu == 0 exactly wherever the oracle's whole output e is identically 0).

a_max = max(|u| + c).  The second RHS term is the size of ONE face-flux difference
of equation e (|q_e| times a wave speed over a cell width): rounding in any correct
implementation of the flux is relative to it, so a component whose RHS happens to
be tiny (e.g. the air partial density at rest in C1, exact RHS 0, oracle round-off
1.2e-10 vs flux scale 7.5e6) is not compared against its own noise.
"""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2409_10729_b200 import workloads as W

RHS_TOL = 1e-12       # BASELINE.json north_star: per RHS evaluation
STEP100_TOL = 1e-10   # BASELINE.json north_star: after 100 RK3 steps


def rel_err(gpu: np.ndarray, cpu: np.ndarray, floor=None) -> np.ndarray:
    """Per-equation normalised max error (AMB-17); floor[e] = flux scale (RHS only)."""
    E = cpu.shape[0]
    out = np.zeros(E)
    for e in range(E):
        scale = np.abs(cpu[e]).max()
        if floor is not None:
            scale = max(scale, floor[e]) if scale > 0.0 else scale
        diff = np.abs(gpu[e] - cpu[e]).max()
        if scale == 0.0:
            out[e] = 0.0 if diff == 0.0 else np.inf
        else:
            out[e] = diff / scale
    return out


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
    """Per-equation size of one face-flux difference: max|q_e| * a_max / dx_min."""
    amax = max_wave_speed(pb, v)
    dxm = min(pb.dx[:pb.ndim])
    return np.array([np.abs(q[e]).max() * amax / dxm for e in range(q.shape[0])])


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
