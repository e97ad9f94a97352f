"""mfc_advance_host (host buffers in and out, the e2e call of bench.py): one step is
streamed as a wavefront over z-chunks with the PCIe copies overlapped (csrc/mfc.cu
advance_streamed); it must reproduce the one-domain device step bit for bit, for
periodic and physical z boundaries, in place (q_out == q_in), for several chunk counts
and for several steps (the unstreamed path).
The oracle pins the device step itself (test_gpu_parity.py); here one step is also
checked against the oracle to the RHS tolerance."""
import numpy as np
import pytest

import oracle as O
from paper_2409_10729_b200 import workloads as W

from parity import oracle_inputs, rel_err, stable_dt

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _device_steps(s, q, dt, n):
    qd = s.state_from_cons(q)
    for _ in range(n):
        s.rk3_step(qd, dt)
    torch.cuda.synchronize()
    return s.interior(qd).cpu().numpy()


def _host(q):
    return torch.as_tensor(np.ascontiguousarray(q)).pin_memory()


CASES = [
    ("periodic-water", lambda: W.random_problem(3, (24, 20, 128), 2, "water")),
    ("refl-extrap-gas-N3", lambda: W.random_problem(3, (33, 17, 130), 3, "gas",
                                                    bc=(W.BC_REFLECTIVE, W.BC_EXTRAPOLATION) * 3)),
    ("extrap-N1", lambda: W.random_problem(3, (40, 9, 100), 1, "gas",
                                           bc=(W.BC_EXTRAPOLATION, W.BC_REFLECTIVE) * 3)),
]


def _fresh_solver(pb, chunks=None):
    """A solver whose workspace holds NaN: a streamed step that read a stage buffer
    before the wavefront wrote it would propagate NaN into the result (ADVICE r1:
    reference steps on the SAME solver left a correct S2 behind and hid exactly that)."""
    from paper_2409_10729_b200.mfc import Solver
    s = Solver(pb)
    s.workspace.fill_(float("nan"))
    if chunks is not None:
        s.set_stream_chunks(chunks)
    return s


def _reference(pb, q, dt, n=1):
    from paper_2409_10729_b200.mfc import Solver
    return _device_steps(Solver(pb), q, dt, n)


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_advance_host_streamed_bitwise(name, make):
    pb = make()
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    ref = _reference(pb, q, dt)                  # another context: nothing shared
    s = _fresh_solver(pb)
    q_in, q_out = _host(q), _host(np.zeros_like(q))
    qdev = s.empty_state()
    s.advance_host(q_in, q_out, qdev, 1, dt)
    launches = s.last_launch_count()
    assert launches > 9, "one step was not streamed in z-chunks"
    assert np.array_equal(s.interior(qdev).cpu().numpy(), ref)   # result left in q_dev
    got = q_out.numpy()
    assert np.array_equal(got, ref), np.abs(got - ref).max()
    # in place, and a second call on the same context (stage buffers now hold the first
    # call's values, which must not leak either): the second step from q^1
    ref2 = _reference(pb, ref, dt)
    s.workspace.fill_(float("nan"))
    s.advance_host(q_in, q_in, qdev, 1, dt)
    assert np.array_equal(q_in.numpy(), ref)
    s.advance_host(q_in, q_in, qdev, 1, dt)
    assert np.array_equal(q_in.numpy(), ref2)
    # the step itself against the oracle
    P = O.Problem.from_spec(pb)
    want = O.rk3_step(P, q, dt)
    assert np.all(rel_err(got, want) <= 1e-12)


def test_advance_host_multistep_unstreamed():
    from paper_2409_10729_b200.mfc import Solver
    pb = W.random_problem(3, (24, 20, 128), 2, "water")
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    s = Solver(pb)
    ref = _device_steps(s, q, dt, 3)
    q_in, q_out = _host(q), _host(np.zeros_like(q))
    s.advance_host(q_in, q_out, s.empty_state(), 3, dt)
    assert np.array_equal(q_out.numpy(), ref)


def test_advance_host_small_grid_unstreamed():
    # too few planes for three z-chunks: the plain upload / step / download path
    from paper_2409_10729_b200.mfc import Solver
    pb = W.random_problem(3, (16, 12, 5), 2, "gas")
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    s = Solver(pb)
    ref = _device_steps(s, q, dt, 1)
    q_in, q_out = _host(q), _host(np.zeros_like(q))
    s.advance_host(q_in, q_out, s.empty_state(), 1, dt)
    assert s.last_launch_count() <= 9
    assert np.array_equal(q_out.numpy(), ref)


@pytest.mark.parametrize("zbc", [W.BC_PERIODIC, W.BC_REFLECTIVE])
@pytest.mark.parametrize("chunks", [3, 4, 7, 40])
def test_advance_host_chunk_counts(chunks, zbc):
    """45 planes -> chunks of 15 / ~11 / 7 (+ a short last one) / 3 planes; fresh
    (NaN-poisoned) workspace every time; periodic z closes the wavefront ring."""
    pb = W.random_problem(3, (20, 12, 45), 2, "water",
                          bc=(W.BC_EXTRAPOLATION, W.BC_REFLECTIVE, W.BC_PERIODIC, W.BC_PERIODIC,
                              zbc, zbc))
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    ref = _reference(pb, q, dt)
    s = _fresh_solver(pb, chunks)
    qi, qo = _host(q), _host(np.zeros_like(q))
    s.advance_host(qi, qo, s.empty_state(), 1, dt)
    assert s.last_launch_count() > 9
    assert np.array_equal(qo.numpy(), ref), np.abs(qo.numpy() - ref).max()


def test_advance_host_rejects_bad_host_buffers():
    from paper_2409_10729_b200.mfc import Solver
    pb = W.random_problem(3, (16, 12, 9), 2, "gas")
    s = Solver(pb)
    good = torch.zeros(pb.shape, dtype=torch.float64)
    with pytest.raises(ValueError):
        s.advance_host(good.float(), good, s.empty_state(), 1, 1e-6)
    with pytest.raises(ValueError):
        s.advance_host(good[:, :-1].contiguous(), good, s.empty_state(), 1, 1e-6)
    with pytest.raises(ValueError):
        s.advance_host(good, good, s.empty_state()[:-1], 1, 1e-6)
