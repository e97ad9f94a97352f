#!/bin/bash
# Final round evidence in one call: tests + bench lines (gpu_evidence.sh), ncu launch list
# and full capture of the default sweeps, compute-sanitizer (4 tools).
TAG=${1:-r2final}
OUT=gpurun_out; mkdir -p $OUT
bash tools/gpu_evidence.sh $TAG
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 45 -c 3 -o $OUT/prof_$TAG python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_full_$TAG.log 2>&1
bash tools/gpu_sanitize.sh $TAG
