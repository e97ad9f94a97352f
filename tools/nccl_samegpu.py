"""libmfc's NCCL halo (pack -> ncclSend/ncclRecv -> unpack on the comm stream) with two
ranks, both on GPU 0 (correctness only; NCCL may refuse two ranks on one device, which
is then what this records).  torchrun --nproc-per-node 2; gloo for the torch plumbing,
the NCCL communicator is libmfc's own.  Rank 0 compares the gathered 2-slab result
after a few RK3 steps (and one RHS) with a single-domain run: bitwise."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2409_10729_b200 import mfc, workloads as W  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
pb = W.c3_droplet(48, nz=48)
nid = mfc.broadcast_unique_id()
try:
    s = mfc.Solver(pb, procs=(1, 1, world), rank=rank, nranks=world, nccl_id=nid, device=0)
except mfc.MfcError as e:
    print(f"rank {rank}: mfc_init with NCCL failed: {e}", flush=True)
    raise SystemExit(3)
L = s.layout
full = W.c3_prims(pb)
z0, nz = L.lo_global[2], L.n_local[2]
q = s.state_from_prims(np.ascontiguousarray(full[:, z0:z0 + nz]))
dt = pb.dt
r = s.empty_state()
s.rhs(q, r)
for _ in range(4):
    s.rk3_step(q, dt)
torch.cuda.synchronize()
s.comm_status()
mine = [s.interior(q).cpu().numpy(), s.interior(r).cpu().numpy()]
got = [None] * world
dist.all_gather_object(got, mine)
if rank == 0:
    ref = mfc.Solver(pb, device=0)
    qr = ref.state_from_prims(full)
    rr = ref.empty_state()
    ref.rhs(qr, rr)
    for _ in range(4):
        ref.rk3_step(qr, dt)
    torch.cuda.synchronize()
    qg = np.concatenate([g[0] for g in got], axis=1)
    rg = np.concatenate([g[1] for g in got], axis=1)
    same_q = np.array_equal(qg, ref.interior(qr).cpu().numpy())
    same_r = np.array_equal(rg, ref.interior(rr).cpu().numpy())
    print(f"NCCL 2 ranks on one GPU, 48^3 C3 in 2 z-slabs: rhs bitwise {same_r}, "
          f"4 RK3 steps bitwise {same_q}", flush=True)
    if not (same_q and same_r):
        raise SystemExit(1)
dist.barrier()
s.close()
