"""Bidirectional PCIe copies in 33.5 MB pieces (the streamed step's piece size at C3),
alone and with the RK3 step running on a third stream."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_10729_b200 import mfc  # noqa: E402
from paper_2409_10729_b200 import workloads as W  # noqa: E402

P, piece = 32, 2 ** 22      # 32 pieces x 4 Mi doubles = 1 GiB
h_in = torch.ones(P * piece, dtype=torch.float64).pin_memory()
h_out = torch.empty(P * piece, dtype=torch.float64).pin_memory()
d_in = torch.empty(P * piece, dtype=torch.float64, device="cuda")
d_out = torch.ones(P * piece, dtype=torch.float64, device="cuda")
s_in, s_out, s_c = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
pb = W.c3_droplet(256)
sol = mfc.Solver(pb)
q = sol.state_from_prims(W.c3_prims(pb))


def run(h2d, d2h, compute, chunks=P):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = P * piece // chunks
    if compute:
        with torch.cuda.stream(s_c):
            for _ in range(3):
                sol.rk3_step(q, pb.dt, stream=s_c)
    for i in range(chunks):
        if h2d:
            with torch.cuda.stream(s_in):
                d_in[i * n:(i + 1) * n].copy_(h_in[i * n:(i + 1) * n], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s_out):
                h_out[i * n:(i + 1) * n].copy_(d_out[i * n:(i + 1) * n], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for args in [(1, 0, 0), (0, 1, 0), (1, 1, 0), (1, 1, 1), (0, 0, 1), (1, 1, 0, 1), (1, 1, 0, 256)]:
    run(*args)
    print(args, round(min(run(*args) for _ in range(3)), 2), "ms")
