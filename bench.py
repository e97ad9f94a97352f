#!/usr/bin/env python
"""Benchmark: grind time of the fp64 5-equation RHS hot path (SSP-RK3 steps) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1: BASELINE.json configs[2] (C3: 3D two-fluid shock-droplet, 256^3 cells, E = 8).
N > 1 (launched by torchrun, one rank per GPU): configs[3] (C4 weak scaling): C3's 256^3
      block on every rank, z-slabs, periodic in z; the halo is fused into the stage's
      last sweep (F1: stores into the neighbours' IPC-mapped ghost layers, --halo fused),
      or the NCCL pack / send-recv / unpack baseline (--halo nccl).
One "step" = one SSP-RK3 step = 3 RHS evaluations (ghost fill + x/y/z fused sweeps each).
Metric (BASELINE.json): grind time = device time / (cells * E * RHS evaluations), in ns,
aggregate over all ranks (lower is better), plus achieved HBM GB/s of the sweeps.

Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle (oracle/, the only
other place bench.py runs it) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grind time ns/(cell*eq*RHS) at 1/2/4/8 B200; achieved HBM GB/s vs peak"
UNIT = "ns/(cell*eq*RHS)"
RHS_PER_STEP = 3


L2_BYTES = 126 * 2 ** 20


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock, power and clock-event reasons sampled DURING the timed region.

    NVML is polled every 5 ms on a thread; only the samples taken between begin() (just
    before the timed steps are enqueued) and end() (after the synchronize that closes
    them) are reported, so the median is the clock under load.  Fallback: nvidia-smi
    -lms 50 over the whole window (marked "source")."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4),
               ("hw_power_brake_slowdown", 0x80))

    def __init__(self, device: int):
        self.device = device
        self.samples = []        # (t, sm_mhz, sm_max_mhz, power_w, reason bits)
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self._h = None
        self._smi = None

    def start(self):
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByUUID(
                uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        except Exception:
            self._h = None
            self._start_smi()
        time.sleep(0.3)     # (the r1/r2 sampler's start-up pause before the timed steps, kept)

    def _poll(self):
        nv, h = self._nv, self._h
        fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                self.samples.append((time.perf_counter(),
                                     nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), smax,
                                     nv.nvmlDeviceGetPowerUsage(h) / 1000.0, int(fn(h))))
            except Exception:
                pass
            time.sleep(0.005)

    def _start_smi(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._smi = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self._t = threading.Thread(target=self._read_smi, daemon=True)
            self._t.start()
            time.sleep(0.25)
        except Exception:
            self._smi = None

    def _read_smi(self):
        for ln in self._smi.stdout:
            f = [x.strip() for x in ln.split(",")]
            try:
                bits = sum(b for (nm, b), v in zip(self.REASONS[:4], f[3:7]) if v.lower() == "active")
                self.samples.append((time.perf_counter(), float(f[0]), float(f[1]), float(f[2]), bits))
            except (ValueError, IndexError):
                continue

    def begin(self):
        self.t0 = time.perf_counter()

    def end(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if self.t1 is None:
            self.end()
        if self._h is not None:
            time.sleep(0.15)
            self._stop.set()
            self._t.join(timeout=1)
        elif self._smi is not None:
            time.sleep(0.1)
            self._smi.terminate()
            try:
                self._smi.wait(timeout=5)
            except Exception:
                self._smi.kill()
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["NVML and nvidia-smi unavailable"]}
        win = [s for s in self.samples if self.t0 is not None and self.t0 <= s[0] <= self.t1]
        src = "NVML every 5 ms inside the timed region" if self._h is not None else \
            "nvidia-smi -lms 50 inside the timed region"
        if not win:             # (a window shorter than one poll)
            win = self.samples
            src += " (no sample inside: all samples)"
        reasons = sorted({nm for nm, b in self.REASONS for s in win if s[4] & b})
        after = [s for s in self.samples if self.t1 < s[0] <= self.t1 + 0.15]
        bits = 0
        for smp in win + after:
            bits |= smp[4]
        return {"sm_mhz": statistics.median(s[1] for s in win) if win else None,
                "sm_min_mhz": min(s[1] for s in win) if win else None,
                "sm_max_mhz": max(s[2] for s in win) if win else None,
                "power_w_max": max(s[3] for s in win) if win else None,
                "samples": len(win), "source": src, "reasons": reasons,
                # the driver raises the reason flags after the clock has already dropped:
                # what it reports in the 150 ms after the timed region, and every bit seen
                "reasons_next_150ms": sorted({nm for nm, b in self.REASONS for s in after
                                              if s[4] & b}),
                "reason_bits_seen": hex(bits)}


# ------------------------------------------------------------ cpu baseline
def cpu_oracle_grind(target_s: float = 12.0, n: int = 256, max_nz: int = 256):
    """The oracle as it stands, timed on the host cores on a bounded sample of C3:
    one RK3 step on an n x n x nz block of the C3 field (nz sized for ~target_s), with
    every OpenMP thread; then the same on a 2-plane block with ONE thread.  Reported:
    wall grind (all threads), core-normalised grind (wall x cores, the paper's CPU
    normalisation P:273) and single-thread grind."""
    import oracle as O
    from paper_2409_10729_b200 import workloads as W
    O.build()

    def run(nz):
        pb = W.c3_droplet(n, nz=nz)
        P = O.Problem.from_spec(pb)
        q = O.prim_to_cons(P, W.c3_prims(pb))
        t0 = time.perf_counter()
        O.rk3_step(P, q, pb.dt, nsteps=1)
        return time.perf_counter() - t0, pb

    cores = O.num_threads()
    t, pb = run(4)
    nz = int(min(max_nz, max(4, 4 * target_s / max(t, 1e-3))))
    if nz > 4:
        t, pb = run(nz)
    grind = t / (pb.cells * pb.E * RHS_PER_STEP) * 1e9
    O.set_num_threads(1)
    try:
        t1, pb1 = run(2)
    finally:
        O.set_num_threads(cores)
    grind1 = t1 / (pb1.cells * pb1.E * RHS_PER_STEP) * 1e9
    return {"value": grind, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"1 SSP-RK3 step (3 RHS) of the C3 field on a {n}x{n}x{nz} block "
                      f"({pb.cells} cells, E={pb.E}), {t:.2f} s wall on {cores} threads; "
                      f"single thread: {n}x{n}x2 block, {t1:.2f} s",
            "core_normalised": grind * cores, "single_thread": grind1}


def run_reference(args):
    """--impl reference: the CPU oracle, each step a bounded sample of the workload."""
    import oracle as O
    from paper_2409_10729_b200 import workloads as W
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    O.build()
    # size the sample so (steps + warmup) RK3 steps take ~2 minutes in total
    pb = W.c3_droplet(256, nz=2)
    P = O.Problem.from_spec(pb)
    q = O.prim_to_cons(P, W.c3_prims(pb))
    t0 = time.perf_counter()
    O.rk3_step(P, q, pb.dt, 1)
    per_plane = (time.perf_counter() - t0) / 2
    total = args.steps + args.warmup
    nz = int(max(2, min(256, 120.0 / max(total * per_plane, 1e-6))))
    pb = W.c3_droplet(256, nz=nz)
    P = O.Problem.from_spec(pb)
    q = O.prim_to_cons(P, W.c3_prims(pb))
    for _ in range(args.warmup):
        O.rk3_step(P, q, pb.dt, 1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        q = O.rk3_step(P, q, pb.dt, 1)
    wall = time.perf_counter() - t0
    grind = wall / (pb.cells * pb.E * RHS_PER_STEP * args.steps) * 1e9
    sample = (f"{args.steps} SSP-RK3 steps of the C3 field on a 256x256x{nz} block "
              f"({pb.cells} cells, E={pb.E}) per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": grind, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3 3D two-fluid shock-droplet (oracle sample)",
                   "sample": sample},
        "cpu_baseline": {"value": grind, "unit": UNIT, "cores": O.num_threads(),
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": grind, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- ours
def algorithmic_bytes(kind: str, E: int, qn_in_x: bool = True) -> float:
    """Algorithmic HBM bytes per interior cell for one launch of each sweep kind in an
    RK3 step, averaged over the three stages (3D, row-parallel x sweep):
    x: read q^s (the stencil state; its re-read for the RK base cb*q^s is the same cell,
    counted once), write acc (16E), plus q^n in stages 2 and 3 when x adds ca*q^n
    (3D, E <= 8: qn_in_x); y: read q^s, acc, write acc (24E); z: read q^s, acc, write the
    stage result (24E), plus q^n in stages 2 and 3 otherwise."""
    qn = 8.0 * E * 2.0 / 3.0
    if kind == "sweep_x":
        return 16.0 * E + (qn if qn_in_x else 0.0)
    if kind == "sweep_y":
        return 24.0 * E
    if kind == "sweep_z":
        return 24.0 * E + (0.0 if qn_in_x else qn)
    return 0.0


def algorithmic_flops(kind: str, N: int, d: int) -> float:
    """Algorithmic fp64 flops per interior cell for one sweep launch:
    WENO5 98 per variable, HLLC 104 per face (N = 2, d = 3), differencing + source 30,
    cons->prim 20 once per RHS (a third per sweep); every +, -, *, /, sqrt, min, max
    of the specification counts as one flop."""
    E = 2 * N + d + 1
    return 98.0 * E + 104.0 + 30.0 + 20.0 / 3.0


FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2: unit counts x max clock


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2409_10729_b200 import mfc
    from paper_2409_10729_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    peer = world > 1 and args.halo == "peer"
    if args.same_device:      # protocol check only: every rank on GPU 0 (time-sliced)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if peer:   # no NCCL anywhere: gloo plumbing, halos as IPC peer stores
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if peer else dev

    def variant(p):   # --weno: reconstruction of the solver's problem (F2 options)
        p.weno_order = 3 if args.weno == "3" else 5
        p.weno_mapped = args.weno == "5m"
        return p

    n = args.n
    procs = (1, 1, world)

    def make(halo):
        """(solver, state, dt, problem, block, workload) of the configuration; `halo` picks
        the N > 1 transport (NCCL for 'nccl' and 'fused', none for the gloo 'peer' mode)."""
        nid = mfc.broadcast_unique_id() if world > 1 and halo != "peer" else None
        pm = halo == "peer"
        block = None
        if args.config == "C3":
            block = W.c3_droplet(n)                  # the per-GPU block (C3 / C4)
            if world == 1:
                pb = block
                workload = f"C3 3D two-fluid shock-droplet {n}^3 (BASELINE configs[2])"
            else:
                pb = W.c3_droplet(n, nz=n * world)   # global domain: blocks stacked along z
                workload = f"C4 weak scaling: C3 {n}^3 block per GPU, z-slabs (BASELINE configs[3])"
            if args.stretch:      # F4: tanh-refined grid on every axis of the global domain
                pb = W.stretched(pb)
                block = W.stretched(block)
                workload += ", tanh-stretched grid (F4)"
            s = mfc.Solver(variant(pb), procs=procs, rank=rank, nranks=world, nccl_id=nid,
                           device=local, peer=pm)
            # every rank holds the same C3 block (its local prims), converted on the GPU
            q = s.state_from_prims(W.c3_prims(block))
            dt = block.dt
            if args.stretch:      # CFL of the smallest cell
                dt *= min(np.diff(pb.boundaries(k)).min() for k in range(3)) / min(pb.dx)
        elif args.config == "C5" and args.stretch:
            raise SystemExit("--stretch runs C3 / C4 only")
        elif args.config == "C5":
            nn = args.n if args.n != 256 else 512
            pb = W.c5_three_fluid(nn)                # strong scaling: fixed 512^3 split in z-slabs
            workload = f"C5 3D three-fluid shock-droplet {nn}^3 total, z-slabs x{world} (BASELINE configs[4])"
            s = mfc.Solver(variant(pb), procs=procs, rank=rank, nranks=world, nccl_id=nid,
                           device=local, peer=pm)
            L0 = s.layout
            v = s.empty_state()
            vi = s.interior(v)
            z0, nzl = L0.lo_global[2], L0.n_local[2]
            for zz in range(0, nzl, 64):             # slab-wise host generation
                vi[:, zz:zz + 64].copy_(torch.as_tensor(W.c5_prims(pb, z0 + zz, z0 + min(zz + 64, nzl))))
            q = s.empty_state()
            s.prim_to_cons(v, q)
            del v, vi
            dt = pb.dt
        else:                                        # C2, single GPU
            pb = W.c2_shock_bubble()
            workload = "C2 2D air-helium shock-bubble 1024x512 (BASELINE configs[1])"
            s = mfc.Solver(variant(pb), procs=(1, 1, 1), device=local)
            q = s.state_from_prims(W.c2_prims(pb))
            dt = pb.dt
        return s, q, dt, pb, block, workload

    halo = args.halo if world > 1 else "none"
    halo_fallback = None
    s, q, dt, pb, block, workload = make(halo)
    if world > 1 and halo in ("fused", "peer"):
        # F1: stage sweeps store boundary layers into the neighbours' IPC-mapped ghosts.
        # The attach and one trial step are checked collectively: if CUDA IPC or the stream
        # memory operations are unavailable between these GPUs on ANY rank, every rank
        # drops to the NCCL pack / send-recv / unpack halo (reported in config.halo_fallback)
        err = None
        try:
            blob = s.peer_export(q)
            torch.cuda.synchronize()
            blobs = [None] * world
            dist.all_gather_object(blobs, blob)
            for face, blob_f in mfc.face_blobs(s.neighbors, blobs).items():
                s.peer_import(face, blob_f)
        except mfc.MfcError as ex:
            err = str(ex)
        ok = [err is None]
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        if all(o[0] for o in oks):
            try:
                s.halo_exchange(q)
                s.rk3_step(q, dt)
                torch.cuda.synchronize()
            except mfc.MfcError as ex:
                err = str(ex)
            dist.all_gather_object(oks, [err is None])
        if not all(o[0] for o in oks):
            if halo == "peer":
                raise SystemExit(f"--halo peer: fused halo unavailable ({err})")
            halo_fallback = f"fused halo unavailable ({err or 'on another rank'}); NCCL halo"
            s.close()
            del q
            halo = "nccl"
            s, q, dt, pb, block, workload = make(halo)
        dist.barrier()
    L = s.layout
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        s.rk3_step(q, dt)
    torch.cuda.synchronize()
    barrier()

    clk = ClockSampler(local)
    clk.start()
    barrier()
    torch.cuda.synchronize()
    # the three state buffers of a step (q, S1, S2 + acc) must not sit in the 126 MB L2
    # between timed steps: small workloads flush it (a 512 MB write) outside the timed
    # events of each step; large ones exceed it by themselves
    flush = 4 * 8 * L.n_elems < 2 * L2_BYTES
    scratch = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev) if flush else None
    # timed region: exactly K steps, library profiling OFF, one CUDA event pair per step
    # on the launching stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    launches = 0
    clk.begin()
    for i in range(args.steps):
        if flush:
            scratch.fill_(float(i))
        evs[i][0].record(stream)
        s.rk3_step(q, dt)
        launches += s.last_launch_count()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    clk.end()
    barrier()
    clocks = clk.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = sum(step_ms)
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # separate profiled pass (same configuration): every kernel launch bracketed by
    # events on its own stream -> the per-kernel split and the roofline of the dominant
    # kernel.  It repeats the timed region's thermal history -- an idle pause, the
    # warm-up steps, the sampler's pause, then as many steps as were timed -- because
    # the board lowers the SM clock ~60 ms into a full FP64 load (profiles/r3/
    # pattern_r303.txt): run straight after the timed region it would see only the
    # lowered clock, and the split would not add up to the timed step
    barrier()
    time.sleep(args.prof_cool)
    for _ in range(args.warmup):
        s.rk3_step(q, dt)
    torch.cuda.synchronize()
    barrier()
    time.sleep(0.3)
    nprof = args.steps
    s.profile(True)
    for i in range(nprof):
        if flush:
            scratch.fill_(float(i))
        s.rk3_step(q, dt)
    torch.cuda.synchronize()
    prof = s.profile_read()
    s.profile(False)

    cells_local = int(np.prod(L.n_local))
    cells_total = cells_local * world
    E = L.E
    grind = ms_max * 1e6 / (cells_total * E * RHS_PER_STEP * args.steps)

    # sustained state (reported beside the contract's value, which stays the K timed
    # steps above): after --sustained seconds of untimed steps the FP64-bound step runs
    # at the board's power limit; time 20 more steps there, clocks sampled alongside
    sustained = None
    if args.sustained > 0:
        barrier()
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < args.sustained:
            s.rk3_step(q, dt)
            torch.cuda.synchronize()
        barrier()
        clk2 = ClockSampler(local)
        clk2.start()
        evs2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(20)]
        clk2.begin()
        for i in range(20):
            if flush:
                scratch.fill_(float(i))
            evs2[i][0].record(stream)
            s.rk3_step(q, dt)
            evs2[i][1].record(stream)
        torch.cuda.synchronize()
        clk2.end()
        barrier()
        clocks2 = clk2.stop()
        st_ms = [a.elapsed_time(b) for a, b in evs2]
        t2 = torch.tensor([sum(st_ms)], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        ms2 = float(t2.item()) / 20
        sustained = {"ms_per_step": ms2, "median_ms": statistics.median(st_ms),
                     "value": ms2 * 1e6 / (cells_total * E * RHS_PER_STEP), "unit": UNIT,
                     "soak_s": args.sustained, "steps": 20, "clocks": clocks2,
                     "note": "after the soak the step runs at the board's power limit "
                             "(sw_power_cap, lower SM clock); not the contract's value"}

    # state sanity (finite) after the timed steps
    finite = bool(torch.isfinite(s.interior(q)).all().item())

    peaks = _peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    qn_in_x = pb.ndim == 3 and E <= 8
    sweeps = {k: v for k, v in prof.items() if k.startswith("sweep") and v[1]}
    dom = max(sweeps, key=lambda k: sweeps[k][0])

    def per_launch(k):
        return sweeps[k][0] / max(sweeps[k][1], 1)

    def hbm_of(k):
        b = algorithmic_bytes(k, E, qn_in_x) * cells_local
        g = b / (per_launch(k) * 1e-3) / 1e9
        return {"achieved": g, "frac": g / hbm_peak, "per_launch_ms": per_launch(k),
                "algorithmic_bytes_per_cell": algorithmic_bytes(k, E, qn_in_x)}

    flops = algorithmic_flops(dom, pb.n_fluids, pb.ndim) * cells_local
    achieved_tf = flops / (per_launch(dom) * 1e-3) / 1e12
    traffic, traffic_src = None, None
    # DRAM bytes of this kernel from the committed ncu capture -- of the workload it was
    # measured on only (C3 256^3, uniform WENO5); any other workload reports null
    wl_key = (f"{args.config}-{n}-weno{args.weno}-{'stretched' if args.stretch else 'uniform'}"
              if args.config == "C3" else args.config)
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        if tr.get("workload") == wl_key:
            traffic, traffic_src = tr.get(dom), tr.get("source")
        else:
            traffic_src = f"null: profiles/ncu_traffic.json holds {tr.get('workload')}, not {wl_key}"
    except Exception:
        pass
    # per step: 3 x (16E + 24E + 24E) + q^n reads in stages 2 and 3 (2 x 8E) = 208E B/cell
    step_alg_bytes = (16 + 24 + 24) * E * cells_local * RHS_PER_STEP + 2 * 8 * E * cells_local
    hbm_step = step_alg_bytes / (ms_max / args.steps * 1e-3) / 1e9
    step_flops = (RHS_PER_STEP * sum(algorithmic_flops(k, pb.n_fluids, pb.ndim)
                                     for k in ("sweep_x", "sweep_y", "sweep_z")) + 96.0) * cells_local
    srt = sorted(step_ms)

    line = {
        "metric": METRIC, "value": grind, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": False, "scaling": "strong" if args.config == "C5" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "cells_per_gpu": cells_local, "cells_total": cells_total,
                   "E": E, "n_fluids": pb.n_fluids, "decomposition": f"procs={list(procs)}",
                   "rhs_per_step": RHS_PER_STEP, "dt": dt,
                   "l2": (f"state {8 * L.n_elems / 1e6:.1f} MB per buffer fits L2: 512 MB L2 flush "
                          "before every timed step, outside its events" if flush else
                          f"inputs > L2: each state buffer {8 * L.n_elems / 1e9:.2f} GB >> 126 MB, no flush"),
                   "parallelism": f"z-slabs x{world}" if world > 1 else "single GPU",
                   "halo": halo,
                   **({"halo_fallback": halo_fallback} if halo_fallback else {}),
                   **({"grid": "tanh-refined on every axis (F4): cells 0.625x finer in "
                              "[0.3, 0.7], workloads.tanh_boundaries"} if args.stretch else {}),
                   **({"weno": {"3": "WENO3-JS", "5m": "WENO5-M (mapped)"}[args.weno]}
                      if args.weno != "5" else {}),
                   **({"same_device": "all ranks on GPU 0: protocol check, time-sliced, not a "
                                      "scaling number"} if args.same_device else {})},
        "step_ms": {"median": statistics.median(step_ms), "min": srt[0], "max": srt[-1],
                    "p10": srt[len(srt) // 10], "p90": srt[(9 * len(srt)) // 10],
                    "all": [round(x, 4) for x in step_ms],
                    "timing": "one CUDA event pair per step on the launching stream, "
                              "library profiling off; value = sum over the K steps (the "
                              "steps slow down in order as the board heats up: "
                              "profiles/r3/pattern_r302.txt)"},
        "hbm_gbs_step": hbm_step,
        "hbm_frac_step": hbm_step / hbm_peak,
        "fp64_tflops_step": step_flops / (ms_max / args.steps * 1e-3) / 1e12,
        "kernel_ms_per_step": {k: v[0] / nprof for k, v in prof.items() if v[1]},
        "kernel_split_source": f"separate profiled pass of {nprof} steps after the timed "
                               f"region, {args.prof_cool} s idle + {args.warmup} warm-up steps "
                               "before it as before the timed steps (events around every "
                               "launch)",
        "roofline": {"bound": "alu", "kernel": dom, "achieved": achieved_tf,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved_tf / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "per_launch_ms": per_launch(dom),
                     "algorithmic_flops_per_cell": algorithmic_flops(dom, pb.n_fluids, pb.ndim),
                     **({"flops_note": "algorithmic flops of the WENO5-JS path (DESIGN.md "
                                       "§6.3); this run uses another reconstruction"}
                        if args.weno != "5" or args.stretch else {}),
                     "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz "
                                    "(B200_PROFILING.md unit counts/clock; MEASURED_PEAKS.json "
                                    "has no FP64 entry; tools/fp64_peak.cu measured 34.1)",
                     "hbm_view": {**hbm_of(dom), "peak": hbm_peak, "unit": "GB/s",
                                  "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"},
                     "hbm_per_sweep": {k: hbm_of(k) for k in sorted(sweeps)}},
        "clocks": clocks,
        **({"sustained": sustained} if sustained else {}),
        "gpu_launches": launches,
        "state_finite": finite,
    }

    # e2e through the C ABI with host buffers (H2D + steps + D2H inside the timed region)
    if not args.no_e2e:
        import torch as T
        qh_in = T.empty((E, L.n_local[2], L.n_local[1], L.n_local[0]), dtype=T.float64).pin_memory()
        qh_in.copy_(s.interior(q).cpu())
        qh_out = T.empty_like(qh_in).pin_memory()
        ke = max(1, min(args.steps, 5))
        s.advance_host(qh_in, qh_out, q, 1, dt)   # warm-up
        barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            s.advance_host(qh_in, qh_out, q, 1, dt)
        wall = time.perf_counter() - t0
        tw = torch.tensor([wall], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        nb = int(qh_in.numel() * 8)
        line["e2e"] = {"value": float(tw.item()) * 1e9 / (cells_total * E * RHS_PER_STEP * ke),
                       "unit": UNIT, "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
                       "steps": ke, "call": "mfc_advance_host(nsteps=1) per step, pinned host buffers"}

    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_oracle_grind(args.cpu_seconds)
        except Exception as ex:  # report, never fall back
            line["cpu_baseline"] = {"error": repr(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--cells", dest="n", type=int, default=256,
                    help="cells per dimension of the per-GPU block")
    ap.add_argument("--config", default="C3", choices=["C3", "C5", "C2"],
                    help="C3/C4 (default; weak scaling for N > 1), C5 (strong scaling), C2")
    ap.add_argument("--sustained", type=float, default=2.0,
                    help="seconds of untimed steps before a 20-step sustained (power-limited) "
                         "timing reported beside the value; 0 disables")
    ap.add_argument("--prof-cool", type=float, default=1.0,
                    help="idle seconds before the profiled (per-kernel) pass, so that it "
                         "starts from the timed region's thermal state; 0 under ncu")
    ap.add_argument("--halo", default="fused", choices=["nccl", "fused", "peer"],
                    help="N>1: 'fused' (default, F1): the last sweep of each RK stage stores "
                         "its boundary layers into the neighbours' CUDA-IPC-mapped ghost "
                         "layers over NVLink, NCCL only for the plumbing; 'nccl': the "
                         "baseline pack / NCCL send-recv / unpack; 'peer': fused with gloo "
                         "plumbing and no NCCL")
    ap.add_argument("--same-device", action="store_true",
                    help="put every rank on GPU 0 (multi-process protocol check on one GPU; "
                         "its timings are time-sliced and not a scaling number)")
    ap.add_argument("--weno", default="5", choices=["5", "3", "5m"],
                    help="reconstruction: WENO5-JS (default, the named path), WENO3-JS or "
                         "WENO5-M (SURVEY §8(f) F2)")
    ap.add_argument("--stretch", action="store_true",
                    help="C3/C4 on a tanh-refined grid (SURVEY §8(f) F4; per-cell WENO tables)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    if args.warmup < 3:
        print("note: warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
