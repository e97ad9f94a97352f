"""libmfc's NCCL halo path on one GPU (MFC_TRANSPORT_NCCL_SELF, include/mfc.h): every
periodic face is a rank face whose neighbour is the rank itself, so its ghost layers go
pack -> ncclSend / ncclRecv (to self, one-rank communicator, on the comm stream,
overlapped with the sweeps that do not need them) -> unpack, and the reductions are
one-rank NCCL all-reduces.  NCCL refuses two ranks on one device, so this is the
hardware check of that code this build can run: the send / receive ordering when both
faces of every axis have the same peer (the 2-rank periodic case of z-slabs), the face
sizes of every axis, the event ordering against the sweeps.  Results must be bitwise
those of the plain single domain (whose periodic ghosts are index maps inside the
sweeps) and within the parity metric of the oracle."""
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

P_, R_, X_ = W.BC_PERIODIC, W.BC_REFLECTIVE, W.BC_EXTRAPOLATION

CASES = [
    (3, (24, 20, 18), 2, (P_,) * 6),                     # every face through NCCL
    (3, (33, 17, 12), 3, (P_, P_, R_, X_, P_, P_)),      # x and z through NCCL, y physical
    (2, (40, 24, 1), 2, (X_, R_, P_, P_, P_, P_)),       # 2D: y only
    (1, (50, 1, 1), 2, (P_, P_, P_, P_, P_, P_)),        # 1D
]


def _run(pb, q, dt, nsteps, **kw):
    s = mfc.Solver(pb, **kw)
    qd = s.state_from_cons(q)
    r = s.rhs(qd)
    rate = s.max_wave_rate(qd).item()
    bad = s.count_inadmissible(qd).item()
    for _ in range(nsteps):
        s.rk3_step(qd, dt)
    torch.cuda.synchronize()
    launches = s.last_launch_count()
    s.comm_status()
    out = (s.interior(r).cpu().numpy(), s.interior(qd).cpu().numpy(), rate, bad, launches,
           s.neighbors)
    s.close()
    return out


@pytest.mark.parametrize("case", range(len(CASES)), ids=[f"case{i}" for i in range(len(CASES))])
def test_nccl_self_exchange_bitwise(case):
    d, n, N, bc = CASES[case]
    pb = W.random_problem(d, n[:d], N, "water", bc=bc)
    P, v, q = oracle_inputs(pb, seed=100 + case)
    dt = stable_dt(pb, v, 0.3)
    r0, q0, rate0, bad0, l0, nb0 = _run(pb, q, dt, 3)
    r1, q1, rate1, bad1, l1, nb1 = _run(pb, q, dt, 3, nccl_self=True)
    assert np.array_equal(r0, r1)
    assert np.array_equal(q0, q1)
    assert rate0 == rate1 and bad0 == bad1 == 0
    # the periodic faces really went through the exchange: neighbour = self, and the
    # step launched the pack / unpack kernels besides the sweeps
    nper = sum(1 for f in range(2 * d) if bc[f] == P_)
    assert sum(1 for f in range(2 * d) if nb1[f] == 0) == nper
    assert l1 > l0
    check_against_oracle(f"nccl-self {pb.name} {n[:d]} bc={bc[:2 * d]}", pb, v, q, r1, q1, dt, 3)


def test_nccl_self_rk3_steps_and_advance_host():
    """mfc_rk3_steps (plain launches with a communicator) and mfc_advance_host (the
    non-streamed copy path: streaming needs a domain without rank faces) agree bitwise
    with the per-step single-domain result."""
    pb = W.random_problem(3, (20, 18, 16), 2, "gas")
    P, v, q = oracle_inputs(pb, seed=7)
    dt = stable_dt(pb, v, 0.3)
    _, q0, *_ = _run(pb, q, dt, 4)
    s = mfc.Solver(pb, nccl_self=True)
    qd = s.state_from_cons(q)
    s.rk3_steps(qd, dt, 4)
    torch.cuda.synchronize()
    assert np.array_equal(s.interior(qd).cpu().numpy(), q0)
    qh = torch.from_numpy(np.ascontiguousarray(q)).pin_memory()
    out = torch.empty_like(qh).pin_memory()
    qd2 = s.empty_state()
    for i in range(4):
        s.advance_host(qh if i == 0 else out, out, qd2, 1, dt)
    assert np.array_equal(out.numpy(), q0)
    s.close()


def test_nccl_self_fullsize_c3():
    """C3 256^3 (BASELINE configs[2]) with all six faces through the NCCL path: one RHS
    and two RK3 steps bitwise equal to the plain single domain (multi-segment marches,
    the full-size face messages of 12.6 MB)."""
    pb = W.c3_droplet(256)
    outs = []
    for kw in ({}, {"nccl_self": True}):
        s = mfc.Solver(pb, **kw)
        q = s.state_from_prims(W.c3_prims(pb))
        r = s.rhs(q)
        for _ in range(2):
            s.rk3_step(q, pb.dt)
        torch.cuda.synchronize()
        outs.append((s.interior(r), s.interior(q)))   # (the ghost layers differ: filled
        s.comm_status()                               #  only by the exchange)
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
