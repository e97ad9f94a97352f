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


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_advance_host_streamed_bitwise(name, make):
    from paper_2409_10729_b200.mfc import Solver
    pb = make()
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    s = Solver(pb)
    ref = _device_steps(s, q, dt, 1)
    q_in, q_out = _host(q), _host(np.zeros_like(q))
    qdev = s.empty_state()
    s.advance_host(q_in, q_out, qdev, 1, dt)
    launches = s.last_launch_count()
    assert launches > 9, "one step was not streamed in z-chunks"
    assert np.array_equal(s.interior(qdev).cpu().numpy(), ref)   # result left in q_dev
    got = q_out.numpy()
    assert np.array_equal(got, ref), np.abs(got - ref).max()
    # in place, and a second call on the same context
    s.advance_host(q_in, q_in, qdev, 1, dt)
    assert np.array_equal(q_in.numpy(), ref)
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


@pytest.mark.parametrize("chunks", [3, 7, 40])
def test_advance_host_chunk_counts(chunks):
    # MFC_STREAM (chunk count) is read once per process: each case in a subprocess;
    # 45 planes -> chunks of 15 / 7 (+ a short last one) / 3 planes
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, 'tests');"
        "from paper_2409_10729_b200.mfc import Solver;"
        "from paper_2409_10729_b200 import workloads as W;"
        "from parity import oracle_inputs, stable_dt;"
        "pb = W.random_problem(3, (20, 12, 45), 2, 'water', bc=(W.BC_EXTRAPOLATION,"
        " W.BC_REFLECTIVE, W.BC_PERIODIC, W.BC_PERIODIC, W.BC_PERIODIC, W.BC_PERIODIC));"
        "_, v, q = oracle_inputs(pb); dt = stable_dt(pb, v); s = Solver(pb);"
        "qd = s.state_from_cons(q); s.rk3_step(qd, dt); torch.cuda.synchronize();"
        "ref = s.interior(qd).cpu().numpy();"
        "qi = torch.as_tensor(q).pin_memory(); qo = torch.empty_like(qi).pin_memory();"
        "s.advance_host(qi, qo, s.empty_state(), 1, dt);"
        "assert s.last_launch_count() > 9; assert np.array_equal(qo.numpy(), ref); print('ok')")
    env = dict(os.environ, MFC_STREAM=str(chunks))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
