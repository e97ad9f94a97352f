#!/bin/bash
# ncu evidence for the current build: launch list of one bench run + full capture of
# one launch of each sweep kernel (x staged, y, z) after warm-up.
TAG=${1:-r05}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_bench_$TAG.log 2>&1
# warm-up = 3 steps x 3 stages x (3 bc + 3 sweeps); skip them, then capture 3 sweeps
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep" -s 27 -c 3 -o $OUT/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_full_$TAG.log 2>&1
