"""Timeline pieces of the e2e call at C3 256^3: pure copies (nsteps=0: H2D then D2H),
one streamed step, torch H2D/D2H of the same pinned buffers."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_10729_b200 import mfc  # noqa: E402
from paper_2409_10729_b200 import workloads as W  # noqa: E402

pb = W.c3_droplet(256)
s = mfc.Solver(pb)
q = s.state_from_prims(W.c3_prims(pb))
L = s.layout
qh_in = torch.empty((L.E, L.n_local[2], L.n_local[1], L.n_local[0]), dtype=torch.float64).pin_memory()
qh_in.copy_(s.interior(q).cpu())
qh_out = torch.empty_like(qh_in).pin_memory()
dense = torch.empty(qh_in.shape, dtype=torch.float64, device="cuda")


def wall(fn, n=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print("advance_host nsteps=0 (H2D + D2H, sequential):", round(wall(lambda: s.advance_host(qh_in, qh_out, q, 0, pb.dt)), 2), "ms")
print("advance_host nsteps=1 (streamed):", round(wall(lambda: s.advance_host(qh_in, qh_out, q, 1, pb.dt)), 2), "ms")
print("torch H2D dense 1.07 GB:", round(wall(lambda: dense.copy_(qh_in, non_blocking=True)), 2), "ms")
print("torch D2H dense 1.07 GB:", round(wall(lambda: qh_out.copy_(dense, non_blocking=True)), 2), "ms")
st = torch.cuda.Stream()


def both():
    dense.copy_(qh_in, non_blocking=True)
    with torch.cuda.stream(st):
        qh_out.copy_(q[:dense.numel()].view(dense.shape) if False else dense2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(st)


dense2 = torch.ones_like(dense)
print("torch H2D + D2H concurrently:", round(wall(both), 2), "ms")
os.environ["MFC_STREAM_TRACE"] = "1"
