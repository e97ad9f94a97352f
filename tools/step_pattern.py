"""Per-step timing pattern of the C3 256^3 step (diagnostic, not the bench).

Prints the event time of every one of --steps consecutive RK3 steps (library profiling
off), then the per-kernel split of --prof single steps (profiling on, one read per step),
so a bimodal step-time distribution can be traced to a sweep / stage.
usage (repo root, GPU box): python tools/step_pattern.py [--steps 40] [--prof 8]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_10729_b200 import mfc, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--prof", type=int, default=8)
ap.add_argument("--graph", action="store_true", help="time mfc_rk3_steps(1) replays")
args = ap.parse_args()

blk = W.c3_droplet(args.n)
s = mfc.Solver(blk)
q = s.state_from_prims(W.c3_prims(blk))
dt = blk.dt
st = torch.cuda.current_stream()
step = (lambda: s.rk3_steps(q, dt, 1)) if args.graph else (lambda: s.rk3_step(q, dt))
for _ in range(5):
    step()
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
       for _ in range(args.steps)]
for a, b in evs:
    a.record(st)
    step()
    b.record(st)
torch.cuda.synchronize()
ms = [round(a.elapsed_time(b), 4) for a, b in evs]
print(json.dumps({"step_ms": ms}))
# the same with a synchronize after every step and the SM clock / power read by NVML
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(0).uuid))
    time.sleep(5)   # let the board cool down to the state the first pass started from
    rows = []
    for i in range(args.steps):
        a, b = evs[i]
        a.record(st)
        step()
        b.record(st)
        torch.cuda.synchronize()
        rows.append((round(a.elapsed_time(b), 4), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                     round(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0), int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))))
    print(json.dumps({"synced_steps (ms, sm_mhz, power_w, reasons)": rows}))
except Exception as ex:  # noqa: BLE001
    print(json.dumps({"nvml": repr(ex)}))
for i in range(args.prof):
    s.profile(True)
    s.rk3_step(q, dt)
    torch.cuda.synchronize()
    p = s.profile_read()
    s.profile(False)
    print(json.dumps({"prof_step": i, **{k: round(v[0], 4) for k, v in p.items() if v[1]}}))
