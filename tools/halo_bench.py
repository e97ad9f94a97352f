"""F1 measurement on one GPU: RK3 steps of a loopback group (P subdomains of one
problem on the same device) with the exchanged halo (pack -> device copy -> unpack per
stage, overlapped on a comm stream) versus the fused halo (the last sweep of each stage
stores boundary layers straight into the neighbours' ghost layers).

usage: python tools/halo_bench.py [--steps 10] [--nccl-self] > profiles/halo_<tag>.jsonl
(--nccl-self: the single domain against MFC_TRANSPORT_NCCL_SELF, where every periodic face
goes pack -> NCCL send/recv to self -> unpack: the NCCL path's cost on one GPU.)
Each line: config, mode, ms per step (CUDA events), halo-kernel ms per step, kernel
launches per step.  Synthetic C3 fields (workloads.c3_prims), fp64.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_10729_b200 import mfc  # noqa: E402
from paper_2409_10729_b200 import workloads as W  # noqa: E402


def run(n, procs, mode, steps, warmup):
    pb = W.c3_droplet(n)
    v = W.c3_prims(pb)
    P = int(np.prod(procs))
    if mode == "nccl-self":   # one rank, every periodic face through NCCL send/recv to self
        solvers = [mfc.Solver(pb, nccl_self=True)]
    else:
        solvers = [mfc.Solver(pb, procs=procs, rank=r, nranks=P, loopback=True) for r in range(P)]
    qs = []
    for s in solvers:
        L = s.layout
        lo, nl = L.lo_global, L.n_local
        qs.append(s.state_from_prims(v[:, lo[2]:lo[2] + nl[2], lo[1]:lo[1] + nl[1], lo[0]:lo[0] + nl[0]]))
    del v
    if mode == "fused":
        mfc.fused_halo_group(solvers, qs)
        mfc.halo_exchange_group(solvers, qs)
    for _ in range(warmup):
        mfc.rk3_step_group(solvers, qs, pb.dt)
    torch.cuda.synchronize()
    for s in solvers:
        s.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launches = 0
    for _ in range(steps):
        mfc.rk3_step_group(solvers, qs, pb.dt)
        launches += sum(s.last_launch_count() for s in solvers)
    e1.record()
    torch.cuda.synchronize()
    halo_ms = sum(s.profile_read()["halo"][0] for s in solvers)
    finite = all(bool(torch.isfinite(s.interior(q)).all()) for s, q in zip(solvers, qs))
    for s in solvers:
        s.close()
    cfg = (f"C3 {n}^3, one rank, all 6 periodic faces through libmfc's NCCL halo (self)"
           if mode == "nccl-self" else f"C3 {n}^3 as {procs} loopback subdomains on 1 GPU")
    return {"config": cfg, "mode": mode,
            "ms_per_step": e0.elapsed_time(e1) / steps, "halo_kernel_ms_per_step": halo_ms / steps,
            "launches_per_step": launches / steps, "finite": finite}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--nccl-self", action="store_true",
                    help="only the single domain and the NCCL self-exchange of C3 256^3")
    args = ap.parse_args()
    if args.nccl_self:
        for mode in ("single", "nccl-self"):
            print(json.dumps(run(256, (1, 1, 1), mode, args.steps, args.warmup)), flush=True)
        return
    for n in (256, 128, 64):              # the single domain of each size, for reference
        print(json.dumps(run(n, (1, 1, 1), "single", args.steps, args.warmup)), flush=True)
    for n, procs in ((256, (1, 1, 2)), (256, (1, 2, 2)), (128, (2, 2, 2)), (64, (2, 2, 2))):
        for mode in ("exchanged", "fused"):
            print(json.dumps(run(n, procs, mode, args.steps, args.warmup)), flush=True)


if __name__ == "__main__":
    main()
