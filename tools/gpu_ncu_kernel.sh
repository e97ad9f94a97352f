#!/bin/bash
# usage: gpu_ncu_kernel.sh TAG REGEX [skip]
TAG=$1; RE=$2; SKIP=${3:-9}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c 1 -o $OUT/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_full_$TAG.log 2>&1
