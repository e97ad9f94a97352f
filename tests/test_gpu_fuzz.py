"""Seeded random configurations (sizes including odd, tiny and multi-segment extents,
N = 1..3, d = 1..3, every boundary-condition combination, uniform or stretched axes,
WENO5-JS / WENO3 / WENO5-M, decomposed or not): RHS and 3 RK3 steps against the oracle
under the parity metric of tests/parity.py.  Catches the corners the named cases do not
(partial warps, odd periodic rows of the x pair, mixed stretched / uniform axes, ...)."""
import numpy as np
import pytest

import oracle as O
from paper_2409_10729_b200 import workloads as W

from parity import check_against_oracle, check_rhs, gpu_rhs, oracle_inputs, stable_dt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2409_10729_b200 import mfc  # noqa: E402

BCS = (W.BC_PERIODIC, W.BC_REFLECTIVE, W.BC_EXTRAPOLATION)


def _config(seed):
    rng = np.random.default_rng(seed)
    d = int(rng.integers(1, 4))
    N = int(rng.integers(1, 4))
    sizes = [int(rng.choice([3, 4, 7, 31, 33, 64, 65, 130, 257, 300])) for _ in range(d)]
    while np.prod(sizes) > 120_000:
        k = int(np.argmax(sizes))
        sizes[k] = max(3, sizes[k] // 2)
    bc = []
    for _ in range(d):
        lo = int(rng.choice(BCS))
        hi = lo if lo == W.BC_PERIODIC else int(rng.choice(BCS[1:]))
        bc += [lo, hi]
    bc += [W.BC_PERIODIC] * (6 - len(bc))
    pb = W.random_problem(d, tuple(sizes), N, str(rng.choice(["gas", "water"])), bc=tuple(bc))
    variant = str(rng.choice(["5", "5", "3", "5m", "st"]))
    if variant == "3":
        pb.weno_order = 3
    elif variant == "5m":
        pb.weno_mapped = True
    elif variant == "st":
        axes = tuple(k for k in range(d) if rng.random() < 0.7) or (0,)
        pb = W.stretched(pb, axes, r=float(rng.uniform(0.2, 0.6)), w=float(rng.uniform(0.03, 0.1)))
    # a decomposition along an axis with enough cells (loopback group)
    procs = [1, 1, 1]
    if rng.random() < 0.4:
        k = int(rng.integers(0, d))
        if sizes[k] >= 6:
            procs[k] = 2
    return pb, tuple(procs), variant


@pytest.mark.parametrize("seed", range(150))
def test_random_configuration(seed):
    pb, procs, variant = _config(1000 + seed)
    P, v, q = oracle_inputs(pb, seed=seed)
    dt = stable_dt(pb, v, 0.2)
    if pb.stretched:
        hmin = min(np.diff(pb.boundaries(k)).min() for k in range(pb.ndim))
        dt *= hmin / min(pb.dx[:pb.ndim])
    name = f"fuzz {seed} {pb.name} {pb.n[:pb.ndim]} bc={pb.bc[:2 * pb.ndim]} {variant} procs={procs}"
    nr = int(np.prod(procs))
    # the method has no positivity limiter (AMB-14): a random input that turns
    # inadmissible within 3 steps (cavitating water) is compared on its RHS only
    steps_ok = O.count_inadmissible(P, O.rk3_step(P, q, dt, nsteps=3)) == 0
    if nr == 1:
        got = gpu_rhs(pb, q)
        check_rhs("rhs " + name, pb, v, q, got, O.rhs(P, q))
        s = mfc.Solver(pb)
        qd = s.state_from_cons(q)
        for _ in range(3):
            s.rk3_step(qd, dt)
        torch.cuda.synchronize()
        if steps_ok:
            check_against_oracle(name, pb, v, q, None, s.interior(qd).cpu().numpy(), dt, 3)
        return
    solvers = [mfc.Solver(pb, procs=procs, rank=r, nranks=nr, loopback=True) for r in range(nr)]
    qs = []
    for s in solvers:
        lo, n = s.layout.lo_global, s.layout.n_local
        qs.append(s.state_from_cons(q[:, lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]]))
    outs = [s.empty_state() for s in solvers]
    mfc.rhs_group(solvers, qs, outs)
    for _ in range(3):
        mfc.rk3_step_group(solvers, qs, dt)
    torch.cuda.synchronize()
    r_full, q_full = np.empty_like(q), np.empty_like(q)
    for s, r_, t in zip(solvers, outs, qs):
        lo, n = s.layout.lo_global, s.layout.n_local
        sl = (slice(None), slice(lo[2], lo[2] + n[2]), slice(lo[1], lo[1] + n[1]),
              slice(lo[0], lo[0] + n[0]))
        r_full[sl] = s.interior(r_).cpu().numpy()
        q_full[sl] = s.interior(t).cpu().numpy()
    check_against_oracle(name, pb, v, q, r_full, q_full if steps_ok else None, dt, 3)
