"""Summarise an ncu --set full report (and optionally a launch-list CSV) as markdown.

usage: python tools/ncu_summary.py prof.ncu-rep [launches.csv] > profiles/<tag>.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe instructions (of peak, active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles active"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle", "mio_throttle",
          "lg_throttle", "barrier", "branch_resolving", "no_instructions", "not_selected",
          "selected", "dispatch_stall", "membar", "sleeping", "tex_throttle", "drain"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def fp64_ops(rep):
    """DFMA / DMUL / DADD thread instructions per kernel row (SASS opcode instances)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-metric-instances",
                          "details", "--metrics", "sass__thread_inst_executed_true_per_opcode"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    for r in rows[1:]:
        cell = r[-1] if r else ""
        if "(" not in cell:
            continue
        ops = {}
        for part in cell[cell.find("(") + 1:cell.rfind(")")].split(";"):
            if ":" in part:
                k, v = part.split(":")
                ops[k.strip()] = float(v)
        res.append({k: ops.get(k, 0.0) for k in ("DFMA", "DMUL", "DADD", "MUFU")})
    return res


def main():
    rep = sys.argv[1]
    hdr, units, data = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    name_i = idx.get("Kernel Name")
    print(f"# ncu summary: `{rep.split('/')[-1]}`\n")
    try:
        ops = fp64_ops(rep)
    except Exception:  # older reports / ncu without the metric
        ops = []
    for ri, row in enumerate(data):
        kname = row[name_i]
        short = kname.split("(")[0].replace("void ", "")
        tmpl = kname[kname.find("<"):kname.rfind(">") + 1] if "<" in kname else ""
        print(f"## {short} {tmpl}\n")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in idx:
                print(f"| {label} (`{k}`) | {row[idx[k]]} {units[idx[k]]} |")
        if ri < len(ops):
            o = ops[ri]
            tot = o["DFMA"] + o["DMUL"] + o["DADD"]
            print(f"| FP64 thread instructions (SASS DFMA {o['DFMA']:.4g} + DMUL {o['DMUL']:.4g} "
                  f"+ DADD {o['DADD']:.4g}) | {tot:.4g} |")
            print(f"| MUFU thread instructions | {o['MUFU']:.4g} |")
        samples = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in idx:
                try:
                    samples[s] = float(row[idx[k]].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(samples.values())
        if tot:
            top = sorted(samples.items(), key=lambda t: -t[1])[:6]
            print("| stall samples (top) | " + ", ".join(f"{s} {100 * v / tot:.1f}%" for s, v in top) + " |")
        print()
    if len(sys.argv) > 2:
        per = defaultdict(lambda: [0.0, 0])
        with open(sys.argv[2]) as f:
            lines = [l for l in f if not l.startswith("==")]
        rows = list(csv.reader(io.StringIO("".join(lines))))
        h = rows[0]
        ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        for r in rows[1:]:
            if len(r) > vi and r[mi] == "gpu__time_duration.sum":
                k = r[ki].split("(")[0].replace("void ", "")
                t = r[ki]
                if "sweep" in k:
                    k = k + t[t.find("<"):t.find(">") + 1]
                per[k][0] += float(r[vi].replace(",", ""))
                per[k][1] += 1
        total = sum(v[0] for v in per.values())
        print("## Launch list (ncu, cold-cache, serialised): share of device time\n")
        print("| kernel | launches | total ns | share |\n|---|---|---|---|")
        for k, (t, n) in sorted(per.items(), key=lambda kv: -kv[1][0]):
            print(f"| `{k}` | {n} | {t:.0f} | {100 * t / total:.1f}% |")


if __name__ == "__main__":
    main()
