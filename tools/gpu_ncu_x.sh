#!/bin/bash
TAG=${1:-rx}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_x" -s 9 -c 1 -o $OUT/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_full_$TAG.log 2>&1
