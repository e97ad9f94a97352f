"""Parity at BASELINE.json's full single-GPU size, in the launch configuration bench.py
times: C3 (256^3, N = 2, E = 8).  The oracle computes the full RHS (~10 s on the host
cores) and one full SSP-RK3 step; the GPU runs the same Solver configuration as the
bench.  C5 (512^3, N = 3) is checked on sampled cells computed one by one by the
oracle (orc_rhs_cells) from a local patch of the field."""
import dataclasses

import numpy as np
import pytest

import oracle as O
from paper_2409_10729_b200 import workloads as W

from parity import (RHS_TOL, check_rhs, max_wave_speed, oracle_inputs, record, rel_err,
                    rhs_flux_scale)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2409_10729_b200 import mfc  # noqa: E402


@pytest.fixture(scope="module")
def c3():
    pb = W.c3_droplet(256)
    P, v, q = oracle_inputs(pb)
    return pb, P, v, q


def test_c3_full_rhs(c3):
    pb, P, v, q = c3
    s = mfc.Solver(pb)
    qd = s.state_from_cons(q)
    rd = s.rhs(qd)
    torch.cuda.synchronize()
    got = s.interior(rd).cpu().numpy()
    del rd
    ref = O.rhs(P, q)
    check_rhs("rhs C3 full 256^3 (bench launch config)", pb, v, q, got, ref)


@pytest.mark.parametrize("order,mapped", [(3, False), (5, True)], ids=["weno3", "weno5m"])
def test_c3_full_rhs_weno_options(c3, order, mapped):
    """The reconstruction options bench.py --weno {3,5m} times (F2), at the full C3 size."""
    pb, _, v, q = c3
    pb = dataclasses.replace(pb, weno_order=order, weno_mapped=mapped)
    s = mfc.Solver(pb)
    qd = s.state_from_cons(q)
    rd = s.rhs(qd)
    torch.cuda.synchronize()
    got = s.interior(rd).cpu().numpy()
    del rd, qd
    ref = O.rhs(O.Problem.from_spec(pb), q)
    check_rhs(f"rhs C3 full 256^3 weno{order}{'m' if mapped else ''}", pb, v, q, got, ref)


def test_c3_full_rk3_step(c3):
    pb, P, v, q = c3
    s = mfc.Solver(pb)
    qd = s.state_from_cons(q)
    s.rk3_step(qd, pb.dt)
    torch.cuda.synchronize()
    got = s.interior(qd).cpu().numpy()
    ref = O.rk3_step(P, q, pb.dt, 1)
    err = rel_err(got - q, ref - q, pb.dt * rhs_flux_scale(pb, v, q))
    record("1 RK3 step increment C3 full 256^3", err, 10 * RHS_TOL)
    assert np.all(err <= 10 * RHS_TOL), err


def test_c2_full_rhs_and_step():
    """C2 at its BASELINE size (1024 x 512, 2D, E = 7; x extrapolation, y reflective),
    the configuration `bench.py --config C2` times: full RHS and one RK3 step."""
    pb = W.c2_shock_bubble()
    P, v, q = oracle_inputs(pb)
    s = mfc.Solver(pb)
    qd = s.state_from_cons(q)
    rd = s.rhs(qd)
    torch.cuda.synchronize()
    got = s.interior(rd).cpu().numpy()
    ref = O.rhs(P, q)
    check_rhs("rhs C2 full 1024x512 (bench launch config)", pb, v, q, got, ref)
    s.rk3_step(qd, pb.dt)
    torch.cuda.synchronize()
    got = s.interior(qd).cpu().numpy()
    ref = O.rk3_step(P, q, pb.dt, 1)
    err = rel_err(got - q, ref - q, pb.dt * rhs_flux_scale(pb, v, q))
    record("1 RK3 step increment C2 full 1024x512", err, 10 * RHS_TOL)
    assert np.all(err <= 10 * RHS_TOL), err


def test_c3_full_advance_host_streamed(c3):
    """The e2e call of bench.py at full size: mfc_advance_host streams the step in
    z-chunks; it must equal the device step (test above) bit for bit."""
    pb, P, v, q = c3
    s = mfc.Solver(pb)
    qd = s.state_from_cons(q)
    s.rk3_step(qd, pb.dt)
    torch.cuda.synchronize()
    ref = s.interior(qd).cpu().numpy()
    del s, qd
    s = mfc.Solver(pb)                       # fresh context, NaN workspace
    s.workspace.fill_(float("nan"))
    q_in = torch.as_tensor(q).pin_memory()
    q_out = torch.empty_like(q_in).pin_memory()
    s.advance_host(q_in, q_out, s.empty_state(), 1, pb.dt)
    assert s.last_launch_count() > 9        # streamed
    assert np.array_equal(q_out.numpy(), ref)


def test_c5_full_size_sampled():
    """512^3, 3 fluids (E = 10, 10.7 GB state): the GPU computes the whole RHS; the
    oracle computes it at 400 sampled cells (incl. the domain corners, the droplet and
    bubble interfaces and the shock slab) from a 13^3 patch around each cell."""
    n = 512
    pb = W.c5_three_fluid(n)
    rng = np.random.default_rng(7)
    cells = [rng.integers(0, n, 3) for _ in range(380)]
    cells += [np.array(c) for c in ((0, 0, 0), (n - 1, n - 1, n - 1), (0, n - 1, 0), (n - 1, 0, n // 2))]
    cells += [np.array((int(0.2 * n) + k, n // 2, n // 2)) for k in range(-2, 3)]          # shock
    cells += [np.array((int(0.35 * n) + k, n // 2, n // 2)) for k in range(-2, 3)]         # droplet edge
    cells += [np.array((int(0.67 * n) + k, n // 2, n // 2)) for k in range(-3, 3)]         # bubble edge
    cells = np.array(cells, dtype=np.int64)
    # GPU: full field, generated and uploaded in z-slabs, converted by mfc_prim_to_cons
    s = mfc.Solver(pb)
    vd = s.empty_state()
    vint = s.interior(vd)
    amax = 0.0
    for z0 in range(0, n, 64):
        vs = W.c5_prims(pb, z0, z0 + 64)
        vint[:, z0:z0 + 64].copy_(torch.as_tensor(vs))
        amax = max(amax, max_wave_speed(pb, vs))
        del vs
    qd = s.empty_state()
    s.prim_to_cons(vd, qd)
    del vd, vint
    rd = s.rhs(qd)
    torch.cuda.synchronize()
    rint = s.interior(rd)
    ci = torch.as_tensor(cells, device=rd.device)
    got = rint[:, ci[:, 2], ci[:, 1], ci[:, 0]].T.cpu().numpy()
    qint = s.interior(qd)
    qmax = qint.abs().amax(dim=(1, 2, 3)).cpu().numpy()
    rhomax = qint[:pb.n_fluids].sum(dim=0).amax().item()
    pmax = 1.01325e5 * 2.3202
    # oracle: one cell at a time on a periodic 13^3 patch centred on it
    E = pb.E
    ref = np.empty((len(cells), E))
    h = 6
    sub = W.Problem("patch", 3, 3, (2 * h + 1,) * 3, hi=tuple((2 * h + 1) / n for _ in range(3)),
                    gamma=pb.gamma, pi_inf=pb.pi_inf, bc=(O.BC_EXTERNAL,) * 6)
    Ps = O.Problem.from_spec(sub)
    off = torch.arange(-h, h + 1, device=rd.device)
    for i, (x, y, z) in enumerate(cells):
        ix, iy, iz = (x + off) % n, (y + off) % n, (z + off) % n
        patch = qint[:, iz][:, :, iy][:, :, :, ix].cpu().numpy()
        ref[i] = O.rhs_cells(Ps, O.pad(Ps, np.ascontiguousarray(patch)), np.array([[h, h, h]]))[0]
    # flux-magnitude scale (tests/parity.py) from the full-field maxima
    N, d = pb.n_fluids, pb.ndim
    phi = np.array([rhomax * amax * amax if N <= e < N + d else
                    ((qmax[e] + pmax) * amax if e == N + d else qmax[e] * amax) for e in range(E)])
    err = rel_err(got.T, ref.T, phi * n)
    record("rhs C5 512^3 sampled (400 cells)", err, RHS_TOL)
    assert np.all(err <= RHS_TOL), err
