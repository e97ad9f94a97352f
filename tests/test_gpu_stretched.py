"""Stretched (tanh-refined) grids on the GPU, SURVEY §8(f) F4 (DESIGN.md AMB-27):
the library derives its own non-uniform WENO5 coefficient tables (primitive-function
Lagrange derivatives, csrc/mfc.cu upload_nu_table) and the sweeps read them per cell;
the oracle solves the cell-average systems (oracle/mfc_oracle.c orc_nu_cell_coeffs).
Parity under the same metric as the uniform path (tests/parity.py check_rhs): 1e-12
per RHS, 1e-10 after 100 RK3 steps; decompositions bitwise equal to one domain."""
import dataclasses

import numpy as np
import pytest

import oracle as O
from paper_2409_10729_b200 import workloads as W

from parity import (STEP100_TOL, check_against_oracle, check_rhs, gpu_rhs, gpu_solver, gpu_steps,
                    oracle_inputs, record, stable_dt, state_err)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2409_10729_b200 import mfc  # noqa: E402


def _st(pb, axes=(0, 1, 2), **kw):
    return W.stretched(pb, axes, **kw)


def _dt(pb, v, cfl=0.25):
    """CFL dt from the smallest cell of the stretched grid."""
    hmin = min(np.diff(pb.boundaries(k)).min() for k in range(pb.ndim))
    return stable_dt(pb, v, cfl) * hmin / min(pb.dx[:pb.ndim])


RHS_CASES = [
    ("C1-st", lambda: _st(W.c1_water_air())),
    ("C2-96x48-st", lambda: _st(W.c2_shock_bubble(96, 48))),
    ("C3-40-st", lambda: _st(W.c3_droplet(40))),
    ("C3-40-st-y-only", lambda: _st(W.c3_droplet(40), axes=(1,), r=0.6, w=0.03)),
    ("C5-36-st", lambda: _st(W.c5_three_fluid(36))),
    ("GR-3D-N3-water-refl-st", lambda: _st(W.random_problem(3, (20, 21, 22), 3, "water",
                                                            bc=(-2, -3, -3, -2, -1, -1)))),
    ("GR-2D-long-rows-st", lambda: _st(W.random_problem(2, (300, 9), 2, "water"))),
    ("GR-1D-N1-st", lambda: _st(W.random_problem(1, (77,), 1, "gas"), r=0.7, w=0.1)),
]


@pytest.mark.parametrize("name,make", RHS_CASES, ids=[c[0] for c in RHS_CASES])
def test_stretched_rhs_parity(name, make):
    pb = make()
    assert pb.stretched
    P, v, q = oracle_inputs(pb)
    ref = O.rhs(P, q)
    got = gpu_rhs(pb, q)
    check_rhs("rhs " + name + " " + "x".join(str(k) for k in pb.n[:pb.ndim]), pb, v, q, got, ref)
    # the stretching is really used: the uniform-grid RHS differs far beyond tolerance
    uni = gpu_rhs(dataclasses.replace(pb, x_cb=(None, None, None)), q)
    d = np.abs(uni - got).reshape(pb.E, -1).max(axis=1)
    assert np.any(d > 1e-6 * np.abs(got).reshape(pb.E, -1).max(axis=1)), d


STEP_CASES = [
    ("C3-24-st", lambda: _st(W.c3_droplet(24))),
    ("GR-3D-N2-water-st", lambda: _st(W.random_problem(3, (20, 17, 18), 2, "water"))),
    ("C1-st", lambda: _st(W.c1_water_air())),
]


@pytest.mark.parametrize("name,make", STEP_CASES, ids=[c[0] for c in STEP_CASES])
def test_stretched_100_steps_parity(name, make):
    pb = make()
    P, v, q = oracle_inputs(pb)
    dt = _dt(pb, v)
    ref = O.rk3_step(P, q, dt, nsteps=100)
    assert O.count_inadmissible(P, ref) == 0
    got = gpu_steps(pb, q, dt, 100)
    err, strict = state_err(pb, got, ref)
    record("100 RK3 steps " + name, err, STEP100_TOL, strict)
    assert np.all(err <= STEP100_TOL), (name, err)


@pytest.mark.parametrize("procs", [(1, 1, 2), (2, 2, 2), (1, 3, 1)])
def test_stretched_decomposition_bitwise(procs):
    """Subdomains take their slice of the global tables (ghost cells of split faces are
    the neighbour's real cells): loopback split == one domain, bitwise; and the oracle."""
    pb = _st(W.random_problem(3, (24, 21, 30), 2, "water"))
    P_, v, q = oracle_inputs(pb)
    dt = _dt(pb, v)
    nr = int(np.prod(procs))
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
    r_split, q_split = np.empty_like(q), np.empty_like(q)
    for s, r_, t in zip(solvers, outs, qs):
        lo, n = s.layout.lo_global, s.layout.n_local
        sl = (slice(None), slice(lo[2], lo[2] + n[2]), slice(lo[1], lo[1] + n[1]),
              slice(lo[0], lo[0] + n[0]))
        r_split[sl] = s.interior(r_).cpu().numpy()
        q_split[sl] = s.interior(t).cpu().numpy()
    assert np.array_equal(r_split, gpu_rhs(pb, q))
    assert np.array_equal(q_split, gpu_steps(pb, q, dt, 3))
    check_against_oracle(f"stretched loopback procs={procs} " + pb.name, pb, v, q, r_split,
                         q_split, dt, 3)


def test_stretched_graph_and_wave_rate():
    pb = _st(W.c3_droplet(24))
    P, v, q = oracle_inputs(pb)
    s = gpu_solver(pb)
    qd = s.state_from_cons(q)
    ref = O.max_wave_rate(P, q)
    got = s.max_wave_rate(qd).item()
    record("max wave rate " + pb.name, abs(got - ref) / ref, 1e-14)
    assert got == pytest.approx(ref, rel=1e-14)
    dt = 0.3 / ref
    a, b = s.state_from_cons(q), s.state_from_cons(q)
    for _ in range(4):
        s.rk3_step(a, dt)
    s.rk3_steps(b, dt, 4)
    torch.cuda.synchronize()
    assert torch.equal(s.interior(a), s.interior(b))


def test_uniform_boundaries_through_the_stretched_path():
    """Uniform x_cb through the non-uniform tables = the uniform kernels up to rounding."""
    pb = W.random_problem(3, (20, 18, 16), 2, "water")
    P, v, q = oracle_inputs(pb)
    xcb = tuple(pb.boundaries(k) for k in range(3))
    a = gpu_rhs(pb, q)
    b = gpu_rhs(dataclasses.replace(pb, x_cb=xcb), q)
    scale = np.abs(a).reshape(pb.E, -1).max(axis=1)
    assert np.all(np.abs(a - b).reshape(pb.E, -1).max(axis=1) <= 1e-11 * scale)


def test_set_grid_errors():
    pb = W.random_problem(3, (12, 10, 9), 2, "gas")
    s = gpu_solver(pb)
    with pytest.raises(mfc.MfcError, match="EINVAL"):
        s.set_grid(0, np.linspace(0, 1, 12))                    # n + 1 = 13 needed
    with pytest.raises(mfc.MfcError, match="EINVAL"):
        x = pb.boundaries(1).copy()
        x[4] = x[3]
        s.set_grid(1, x)                                         # not increasing
    with pytest.raises(mfc.MfcError, match="EINVAL"):
        x = pb.boundaries(2).copy()
        x[5] = np.nan
        s.set_grid(2, x)                                         # not finite
    s.set_grid(0, pb.boundaries(0))
    with pytest.raises(mfc.MfcError, match="EUNSUPPORTED"):
        mfc._check(mfc.lib.mfc_set_weno_order(s._h, 3), "mfc_set_weno_order")
    s.set_grid(0, None)
    mfc._check(mfc.lib.mfc_set_weno_order(s._h, 3), "mfc_set_weno_order")


def test_c3_full_size_stretched_rhs():
    """The bench's --stretch configuration at full size (256^3, all axes refined around
    the droplet): full RHS against the oracle."""
    pb = _st(W.c3_droplet(256))
    P, v, q = oracle_inputs(pb)
    got = gpu_rhs(pb, q)
    ref = O.rhs(P, q)
    check_rhs("rhs C3 full 256^3 stretched (bench --stretch launch config)", pb, v, q, got, ref)


def test_stretched_fused_halo_and_streamed_advance_host():
    """The stretched tables through the other step paths: the fused-halo loopback group
    (peer stores from the ORD-7 marches) and the streamed host-to-host step, both
    bitwise equal to the plain single-domain step."""
    pb = _st(W.random_problem(3, (20, 18, 36), 2, "water"))
    P_, v, q = oracle_inputs(pb)
    dt = _dt(pb, v)
    ref = gpu_steps(pb, q, dt, 2)
    procs = (1, 2, 2)
    solvers = [mfc.Solver(pb, procs=procs, rank=r, nranks=4, loopback=True) for r in range(4)]
    qs = []
    for s in solvers:
        lo, n = s.layout.lo_global, s.layout.n_local
        qs.append(s.state_from_cons(q[:, lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]]))
    mfc.fused_halo_group(solvers, qs)
    mfc.halo_exchange_group(solvers, qs)
    for _ in range(2):
        mfc.rk3_step_group(solvers, qs, dt)
    torch.cuda.synchronize()
    got = np.empty_like(q)
    for s, t in zip(solvers, qs):
        lo, n = s.layout.lo_global, s.layout.n_local
        got[:, lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]] = s.interior(t).cpu().numpy()
    assert np.array_equal(got, ref)
    # streamed advance_host (one step, z-chunks) == one device step
    one = gpu_steps(pb, q, dt, 1)
    s = mfc.Solver(pb)
    s.set_stream_chunks(5)
    qi = torch.as_tensor(q).pin_memory()
    qo = torch.empty_like(qi).pin_memory()
    s.advance_host(qi, qo, s.empty_state(), 1, dt)
    assert s.last_launch_count() > 9
    assert np.array_equal(qo.numpy(), one)
