"""One C3 256^3 RK3 step with MFC_TRANSPORT_NCCL_SELF (for an ncu launch list of the
NCCL halo path: pack, NCCL send/recv to self, unpack)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_10729_b200 import mfc, workloads as W  # noqa: E402

pb = W.c3_droplet(256)
s = mfc.Solver(pb, nccl_self=True)
q = s.state_from_prims(W.c3_prims(pb))
for _ in range(2):
    s.rk3_step(q, pb.dt)
torch.cuda.synchronize()
