#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for T in 32 48 64 96 128; do
  MFC_SEG=$T timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $OUT/seg_$T.json 2>/dev/null
done
