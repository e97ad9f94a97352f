"""NVTX check (SURVEY §5 tracing): a C3-shaped 96^3 problem advanced by plain
mfc_rk3_step calls and one mfc_rhs, for `ncu --nvtx --nvtx-include "mfc@<range>/"`
(tools/gpu_nvtx.sh).  Prints the kernels launched per call for comparison with what
the filtered ncu lists contain."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_10729_b200 import mfc, workloads as W  # noqa: E402

pb = W.c3_droplet(96)
s = mfc.Solver(pb)
q = s.state_from_prims(W.c3_prims(pb))
dt = s.cfl_dt(q, 0.3)
for _ in range(2):
    s.rk3_step(q, dt)
r = s.empty_state()
s.rhs(q, r)
torch.cuda.synchronize()
print("rk3_step launches", mfc.lib.mfc_last_launch_count(s._h))
