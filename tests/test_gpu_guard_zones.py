"""Out-of-bounds and uninitialised-read detection without compute-sanitizer.

compute-sanitizer is closed on the GPU pool since r304 ("runs under it have left GPUs
needing a reset"; profiles/r3/sanitize_memcheck_r304.log); its last clean pass (r212)
predates the one-launch halo pack / unpack kernels (r222) and the cell-major
stretched-grid marches (b70381b).  This test does the two checks that matter for them
with the library's own entry points:

* every device buffer the library touches -- the state tensors (interior, ghost
  layers, pitch padding), the RHS output and the workspace (stage buffers, accumulator,
  halo pack buffers, streaming rings, stretched-grid coefficient tables) -- is a view
  into a larger tensor whose GUARD BANDS hold a NaN sentinel bit pattern: after rhs /
  steps / graph replays / halo exchanges / streamed host steps the guard bands must be
  bit-for-bit unchanged (no write outside any buffer);
* everything except the input interior is filled with the same sentinel before the run
  (ghosts, padding, the whole workspace), and the results must be BITWISE equal to the
  same run on plain allocations: a read of a guard band, of a ghost cell before it is
  filled or of workspace before it is written would pull the NaN into the result.
"""
import numpy as np
import pytest

from paper_2409_10729_b200 import workloads as W

from parity import oracle_inputs, stable_dt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2409_10729_b200 import mfc  # noqa: E402

G = 8192                                # guard doubles per side (64 KB, keeps 256-B alignment)
SENT = 0x7FF4DEAD0000BEEF               # a NaN bit pattern (signalling payload)


class Guarded:
    """n float64 elements at offset G of a (n + 2G) tensor; everything starts as SENT."""

    def __init__(self, n, device):
        self.n = n
        self.big = torch.empty(n + 2 * G, dtype=torch.float64, device=device)
        self.big.view(torch.int64).fill_(SENT)
        self.t = self.big[G:G + n]

    def intact(self):
        b = self.big.view(torch.int64)
        return bool((b[:G] == SENT).all()) and bool((b[G + self.n:] == SENT).all())


def guard_solver(s, pb):
    """Rebind the solver's workspace to a guarded, sentinel-filled allocation (and
    rebuild the stretched-grid tables, which live in it)."""
    nb = s.layout.workspace_bytes
    ws = Guarded((nb + 7) // 8, s.device)
    mfc._check(mfc.lib.mfc_bind_workspace(s._h, mfc._ptr(ws.t), nb), "mfc_bind_workspace")
    s.workspace = ws.t
    for k, xb in enumerate(getattr(pb, "x_cb", None) or ()):
        if xb is not None and k < pb.ndim:
            s.set_grid(k, xb)
    return ws


def guarded_state(s, plain):
    """A guarded copy of `plain` (a state tensor of s's layout) whose ghost layers and
    padding hold the sentinel: only the interior is copied."""
    g = Guarded(s.layout.n_elems, s.device)
    s.interior(g.t).copy_(s.interior(plain))
    return g


def _interior(s, t):
    return s.interior(t).cpu().numpy()


def _bitwise(a, b):
    return np.array_equal(a.view(np.int64), b.view(np.int64))


def _single_run(pb, q, dt, nsteps, guard, graph_steps=0):
    s = mfc.Solver(pb)
    qd = s.state_from_cons(q)
    bufs = []
    if guard:
        bufs.append(guard_solver(s, pb))
        gq = guarded_state(s, qd)
        go = Guarded(s.layout.n_elems, s.device)
        bufs += [gq, go]
        qd, out = gq.t, go.t
    else:
        out = s.empty_state()
    s.rhs(qd, out=out)
    rate = s.max_wave_rate(qd).item()
    for _ in range(nsteps):
        s.rk3_step(qd, dt)
    if graph_steps:
        s.rk3_steps(qd, dt, graph_steps)
    torch.cuda.synchronize()
    return (_interior(s, out), _interior(s, qd), rate), bufs


CASES = [
    ("3D-periodic-water-N2", lambda: W.random_problem(3, (40, 20, 18), 2, "water")),
    ("3D-refl-extrap-gas-N3", lambda: W.random_problem(3, (33, 17, 21), 3, "gas",
                                                       bc=(W.BC_REFLECTIVE, W.BC_EXTRAPOLATION) * 3)),
    ("3D-long-rows-N2", lambda: W.random_problem(3, (520, 6, 5), 2, "water")),
    ("2D-N2", lambda: W.random_problem(2, (70, 37), 2, "water",
                                       bc=(W.BC_EXTRAPOLATION, W.BC_EXTRAPOLATION,
                                           W.BC_REFLECTIVE, W.BC_REFLECTIVE, W.BC_PERIODIC,
                                           W.BC_PERIODIC))),
    ("1D-N2", lambda: W.random_problem(1, (300,), 2, "water", bc=W.BC_EXTRAPOLATION)),
    ("3D-stretched-N2", lambda: W.stretched(W.random_problem(3, (36, 20, 22), 2, "water"))),
    ("2D-stretched-N3", lambda: W.stretched(W.random_problem(2, (50, 30), 3, "gas"))),
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_guard_bands_single_domain(name, make):
    pb = make()
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    ref, _ = _single_run(pb, q, dt, 2, guard=False, graph_steps=2)
    got, bufs = _single_run(pb, q, dt, 2, guard=True, graph_steps=2)
    assert all(b.intact() for b in bufs), "write outside a buffer"
    for a, b in zip(ref[:2], got[:2]):
        assert _bitwise(a, b), "guarded run differs (read of a guard band / unwritten data)"
    assert ref[2] == got[2]


@pytest.mark.parametrize("weno", ["3", "5m"])
def test_guard_bands_weno_options(weno):
    pb = W.random_problem(3, (34, 18, 20), 2, "water")
    pb.weno_order = 3 if weno == "3" else 5
    pb.weno_mapped = weno == "5m"
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    ref, _ = _single_run(pb, q, dt, 2, guard=False)
    got, bufs = _single_run(pb, q, dt, 2, guard=True)
    assert all(b.intact() for b in bufs)
    assert _bitwise(ref[0], got[0]) and _bitwise(ref[1], got[1])


def _group_run(pb, q, procs, dt, nsteps, fused, guard):
    P = int(np.prod(procs))
    solvers = [mfc.Solver(pb, procs=procs, rank=r, nranks=P, loopback=True) for r in range(P)]
    bufs, qs = [], []
    for s in solvers:
        L = s.layout
        lo, n = L.lo_global, L.n_local
        qd = s.state_from_cons(q[:, lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]])
        if guard:
            bufs.append(guard_solver(s, pb))
            g = guarded_state(s, qd)
            bufs.append(g)
            qd = g.t
        qs.append(qd)
    if fused:   # (the registered states' ghosts are filled once, then by the stage sweeps)
        mfc.fused_halo_group(solvers, qs)
        mfc.halo_exchange_group(solvers, qs)
    for _ in range(nsteps):
        mfc.rk3_step_group(solvers, qs, dt)
    torch.cuda.synchronize()
    full = np.empty_like(q)
    for s, t in zip(solvers, qs):
        L = s.layout
        lo, n = L.lo_global, L.n_local
        full[:, lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]] = _interior(s, t)
    return full, bufs


@pytest.mark.parametrize("procs,fused,stretch", [
    ((1, 1, 2), False, False), ((1, 2, 2), False, False), ((2, 2, 2), False, False),
    ((2, 2, 2), False, True), ((1, 2, 2), True, False), ((2, 2, 2), True, True)],
    ids=["slabs-exchanged", "pencils-exchanged", "blocks-exchanged", "blocks-exchanged-stretched",
         "pencils-fused", "blocks-fused-stretched"])
def test_guard_bands_decompositions(procs, fused, stretch):
    pb = W.random_problem(3, (26, 22, 24), 2, "water",
                          bc=(W.BC_PERIODIC, W.BC_PERIODIC, W.BC_REFLECTIVE, W.BC_EXTRAPOLATION,
                              W.BC_PERIODIC, W.BC_PERIODIC))
    if stretch:
        pb = W.stretched(pb)
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    ref, _ = _group_run(pb, q, procs, dt, 3, fused, guard=False)
    got, bufs = _group_run(pb, q, procs, dt, 3, fused, guard=True)
    assert all(b.intact() for b in bufs), "write outside a buffer"
    assert np.isfinite(ref).all()
    assert _bitwise(ref, got)


def test_guard_bands_nccl_self():
    pb = W.random_problem(3, (30, 18, 16), 2, "water",
                          bc=(W.BC_PERIODIC, W.BC_PERIODIC, W.BC_REFLECTIVE, W.BC_EXTRAPOLATION,
                              W.BC_PERIODIC, W.BC_PERIODIC))
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    res = []
    for guard in (False, True):
        s = mfc.Solver(pb, nccl_self=True)
        qd = s.state_from_cons(q)
        bufs = []
        if guard:
            bufs.append(guard_solver(s, pb))
            g = guarded_state(s, qd)
            bufs.append(g)
            qd = g.t
        for _ in range(3):
            s.rk3_step(qd, dt)
        torch.cuda.synchronize()
        s.comm_status()
        res.append(_interior(s, qd))
        assert all(b.intact() for b in bufs), "write outside a buffer"
        s.close()
    assert _bitwise(res[0], res[1])


def test_guard_bands_streamed_advance_host():
    pb = W.random_problem(3, (24, 20, 128), 2, "water")
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    res = []
    for guard in (False, True):
        s = mfc.Solver(pb)
        s.set_stream_chunks(7)
        bufs = []
        qdev = s.empty_state()
        if guard:
            bufs.append(guard_solver(s, pb))
            g = Guarded(s.layout.n_elems, s.device)
            bufs.append(g)
            qdev = g.t
        q_in = torch.as_tensor(np.ascontiguousarray(q)).pin_memory()
        q_out = torch.empty_like(q_in).pin_memory()
        s.advance_host(q_in, q_out, qdev, 1, dt)
        torch.cuda.synchronize()
        res.append(q_out.numpy().copy())
        assert all(b.intact() for b in bufs), "write outside a buffer"
    assert _bitwise(res[0], res[1])
