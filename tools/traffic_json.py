"""profiles/ncu_traffic.json from an ncu DRAM-bytes CSV of the 9 sweep launches of one
C3 256^3 RK3 step (tools/gpu_evidence.sh: ncu --metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum -k regex:sweep -s 45 -c 9 --csv).

usage: python tools/traffic_json.py profiles/ncu_dram9_TAG.csv "TAG (date)" > profiles/ncu_traffic.json
bench.py reads it as roofline.traffic of the default workload only (its "workload" key).
"""
import csv
import io
import json
import re
import sys
from collections import defaultdict

path, tag = sys.argv[1], sys.argv[2]
txt = "".join(ln for ln in open(path) if ln.startswith('"'))
per = defaultdict(dict)          # launch id -> {metric: value}, kernel
kern = {}
for r in csv.DictReader(io.StringIO(txt)):
    i = int(r["ID"])
    per[i][r["Metric Name"]] = float(r["Metric Value"])
    k = r["Kernel Name"]
    d = re.search(r"sweep_kernel<[^>]*>, (\d),", k)        # DIR, the first argument after Model<>
    kern[i] = "sweep_x" if "sweep_x" in k else ("sweep_y" if d and d.group(1) == "1" else "sweep_z")
stages = defaultdict(list)
for i in sorted(per):
    m = per[i]
    stages[kern[i]].append(int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]))
out = {"source": f"{tag}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                 "gpu__time_duration.sum --clock-control none, the 9 sweep launches of one C3 "
                 f"256^3 RK3 step after 3 warm-up + 2 timed steps ({path}); per launch, averaged "
                 "over the 3 stages (x reads q^n in stages 2 and 3)",
       "workload": "C3-256-weno5-uniform"}
for k in ("sweep_x", "sweep_y", "sweep_z"):
    out[k] = sum(stages[k]) / len(stages[k])
out["per_stage"] = dict(stages)
json.dump(out, sys.stdout, indent=1)
print()
