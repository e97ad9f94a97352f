"""Decomposition invariance on ONE GPU (loopback transport):
P subdomains exchanging halos with device copies (the same pack / unpack kernels the
NCCL path uses) reproduce the single-domain result BITWISE (each face flux is computed
from identical inputs by identical code)."""
import numpy as np
import pytest

import oracle as O
from paper_2409_10729_b200 import workloads as W

from parity import check_against_oracle, oracle_inputs, stable_dt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2409_10729_b200 import mfc  # noqa: E402


def _split_run(pb, q, procs, dt, nsteps, rhs_only=False):
    P = int(np.prod(procs))
    solvers = [mfc.Solver(pb, procs=procs, rank=r, nranks=P, loopback=True) for r in range(P)]
    qs = []
    for s in solvers:
        L = s.layout
        lo, n = L.lo_global, L.n_local
        qs.append(s.state_from_cons(q[:, lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]]))
    if rhs_only:
        outs = [s.empty_state() for s in solvers]
        mfc.rhs_group(solvers, qs, outs)
        res = outs
    else:
        for _ in range(nsteps):
            mfc.rk3_step_group(solvers, qs, dt)
        res = qs
    torch.cuda.synchronize()
    full = np.empty_like(q)
    for s, t in zip(solvers, res):
        L = s.layout
        lo, n = L.lo_global, L.n_local
        full[:, lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]] = s.interior(t).cpu().numpy()
    return full


def _single(pb, q, dt, nsteps, rhs_only=False):
    s = mfc.Solver(pb)
    qd = s.state_from_cons(q)
    if rhs_only:
        r = s.rhs(qd)
        torch.cuda.synchronize()
        return s.interior(r).cpu().numpy()
    for _ in range(nsteps):
        s.rk3_step(qd, dt)
    torch.cuda.synchronize()
    return s.interior(qd).cpu().numpy()


@pytest.mark.parametrize("procs", [(1, 1, 2), (1, 1, 4), (1, 2, 2), (2, 2, 2), (1, 1, 3)])
def test_loopback_rhs_and_steps_bitwise(procs):
    pb = W.random_problem(3, (24, 20, 30), 2, "water")
    P_, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    r_split = _split_run(pb, q, procs, dt, 0, rhs_only=True)
    q_split = _split_run(pb, q, procs, dt, 5)
    assert np.array_equal(r_split, _single(pb, q, dt, 0, rhs_only=True))
    assert np.array_equal(q_split, _single(pb, q, dt, 5))
    check_against_oracle(f"loopback procs={procs} " + pb.name, pb, v, q, r_split, q_split, dt, 5)


def test_loopback_nonperiodic_z():
    pb = W.random_problem(3, (16, 12, 24), 3, "gas",
                          bc=(W.BC_PERIODIC, W.BC_PERIODIC, W.BC_REFLECTIVE, W.BC_REFLECTIVE,
                              W.BC_EXTRAPOLATION, W.BC_REFLECTIVE))
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    q_split = _split_run(pb, q, (1, 1, 4), dt, 3)
    assert np.array_equal(q_split, _single(pb, q, dt, 3))
    check_against_oracle("loopback procs=(1,1,4) nonperiodic " + pb.name, pb, v, q, None,
                         q_split, dt, 3)
