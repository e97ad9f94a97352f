"""Helpers shared by the GPU parity tests: run the same seeded input through the
oracle (CPU, fp64) and through libmfc (GPU, via the C ABI) and compare with the
metric of DESIGN.md AMB-17:

    per equation e:  max_cells |gpu - cpu| / max_cells |cpu_e|  <= tol
    (and gpu == 0 exactly wherever the oracle's whole rhs_e is identically 0).
"""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2409_10729_b200 import workloads as W

RHS_TOL = 1e-12       # BASELINE.json north_star: per RHS evaluation
STEP100_TOL = 1e-10   # BASELINE.json north_star: after 100 RK3 steps


def rel_err(gpu: np.ndarray, cpu: np.ndarray) -> np.ndarray:
    """Per-equation normalised max error (AMB-17)."""
    E = cpu.shape[0]
    out = np.zeros(E)
    for e in range(E):
        scale = np.abs(cpu[e]).max()
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
