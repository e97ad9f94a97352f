"""Compute-side scaling emulation on ONE GPU (no NVLink in the loop).

C4 weak scaling: the global domain 256 x 256 x 256P (C3's block per rank, z-slabs,
periodic z) run as a loopback group of P subdomains on one device; C5 strong scaling:
512^3 three-fluid split into P z-slabs the same way.  A loopback group executes the P
ranks' sweeps one after another on one stream with the halo as device copies
("exchanged": pack -> copy -> unpack per stage) or as the fused stores of F1 ("fused"),
so

    weak efficiency   = T(1 rank) / (T(group of P) / P)      (same per-rank block)
    strong efficiency = T(1 rank, whole domain) / T(group of P)

measure what decomposition costs in kernels (halo work, per-rank kernel efficiency at
the smaller slab, launch count) -- not the NVLink transfer, which a real P-GPU run adds
(25 MB per rank per RHS for C4, overlapped with the x/y sweeps).

usage: python tools/scaling_emulation.py [--steps 5] [--soak 3] > profiles/scaling_emulation_<tag>.jsonl
(every configuration is timed after --soak seconds of untimed steps, so all of them run in
the same power-capped state; r214/r224 had no soak and timed the single domain cold.)
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_10729_b200 import mfc  # noqa: E402
from paper_2409_10729_b200 import workloads as W  # noqa: E402


def group_step_ms(pb, prims_of, P, mode, steps, warmup, soak=0.0):
    procs = (1, 1, P)
    solvers = [mfc.Solver(pb, procs=procs, rank=r, nranks=P, loopback=True) for r in range(P)]
    qs = []
    for s in solvers:
        L = s.layout
        z0, nz = L.lo_global[2], L.n_local[2]
        qs.append(s.state_from_prims(prims_of(z0, z0 + nz)))
    if mode == "fused" and P > 1:
        mfc.fused_halo_group(solvers, qs)
        mfc.halo_exchange_group(solvers, qs)
    for _ in range(warmup):
        mfc.rk3_step_group(solvers, qs, pb.dt)
    torch.cuda.synchronize()
    # heat soak: the boards cap power near 380 W and an FP64-bound step reaches the cap
    # within about a second, so every configuration is timed in the same (hot) state
    t0 = time.time()
    while time.time() - t0 < soak:
        mfc.rk3_step_group(solvers, qs, pb.dt)
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launches = 0
    for _ in range(steps):
        mfc.rk3_step_group(solvers, qs, pb.dt)
        launches += sum(s.last_launch_count() for s in solvers)
    e1.record()
    torch.cuda.synchronize()
    finite = all(bool(torch.isfinite(s.interior(q)).all()) for s, q in zip(solvers, qs))
    for s in solvers:
        s.close()
    del qs
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / steps, launches / steps, finite


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--cases", default="C4,C5")
    ap.add_argument("--soak", type=float, default=3.0,
                    help="seconds of untimed steps before each timed run (power-cap state)")
    args = ap.parse_args()
    ranks = [int(x) for x in args.ranks.split(",")]
    for case in args.cases.split(","):
        base = None
        for P in ranks:
            if case == "C4":
                pb = W.c3_droplet(256, nz=256 * P)
                block = W.c3_droplet(256)
                v1 = W.c3_prims(block)       # every rank holds the C3 block (as bench.py)
                prims_of = lambda z0, z1: v1
            else:
                pb = W.c5_three_fluid(512)
                prims_of = lambda z0, z1, pb=pb: W.c5_prims(pb, z0, z1)
            for mode in (("exchanged", "fused") if P > 1 else ("single",)):
                ms, launches, finite = group_step_ms(pb, prims_of, P, mode, args.steps, args.warmup,
                                                     args.soak)
                if P == 1:
                    base = ms
                eff = (base / (ms / P)) if case == "C4" else (base / ms)
                print(json.dumps({
                    "case": case, "ranks": P, "mode": mode,
                    "config": (f"C4: 256^3 per rank, global 256x256x{256 * P}, z-slabs" if case == "C4"
                               else f"C5: 512^3 three-fluid in {P} z-slabs of {512 // P} planes"),
                    "group_ms_per_step": ms, "per_rank_ms_per_step": ms / P,
                    ("weak_efficiency_compute" if case == "C4" else "strong_efficiency_compute"): eff,
                    "launches_per_step": launches, "finite": finite}), flush=True)


if __name__ == "__main__":
    main()
