"""Which buffer's guard band does a call write into, and where (diagnostic for
tests/test_gpu_guard_zones.py).  usage (GPU box): python tools/guard_diag.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from paper_2409_10729_b200 import mfc, workloads as W  # noqa: E402
from parity import oracle_inputs, stable_dt  # noqa: E402
from test_gpu_guard_zones import G, SENT, Guarded, guard_solver, guarded_state  # noqa: E402


def report(tag, bufs):
    for name, b in bufs.items():
        v = b.big.view(torch.int64)
        lo = (v[:G] != SENT).nonzero().flatten()
        hi = (v[G + b.n:] != SENT).nonzero().flatten()
        if lo.numel() or hi.numel():
            print(f"{tag}: {name} (n={b.n}) below: {lo.numel()} elems "
                  f"[{(lo.min().item() - G) if lo.numel() else ''}..{(lo.max().item() - G) if lo.numel() else ''}]"
                  f" above: {hi.numel()} elems [{hi.min().item() if hi.numel() else ''}.."
                  f"{hi.max().item() if hi.numel() else ''}] (offsets past the end)")
            if hi.numel():
                print("   values above:", b.big[G + b.n + hi[:4]].tolist())
            if lo.numel():
                print("   values below:", b.big[lo[:4]].tolist())
            v[:G] = SENT
            v[G + b.n:] = SENT


for name, pb in [("3D", W.random_problem(3, (40, 20, 18), 2, "water")),
                 ("2D", W.random_problem(2, (70, 37), 2, "water")),
                 ("1D", W.random_problem(1, (300,), 2, "water"))]:
    _, v, q = oracle_inputs(pb)
    dt = stable_dt(pb, v)
    s = mfc.Solver(pb)
    L = s.layout
    print(name, "layout", L)
    qd = s.state_from_cons(q)
    ws = guard_solver(s, pb)
    gq = guarded_state(s, qd)
    go = Guarded(L.n_elems, s.device)
    bufs = {"workspace": ws, "q": gq, "out": go}
    torch.cuda.synchronize()
    report(name + " setup", bufs)
    s.rhs(gq.t, out=go.t)
    torch.cuda.synchronize()
    report(name + " rhs", bufs)
    s.max_wave_rate(gq.t)
    torch.cuda.synchronize()
    report(name + " wave rate", bufs)
    s.rk3_step(gq.t, dt)
    torch.cuda.synchronize()
    report(name + " rk3_step", bufs)
    s.rk3_steps(gq.t, dt, 2)
    torch.cuda.synchronize()
    report(name + " rk3_steps", bufs)
