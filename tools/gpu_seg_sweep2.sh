#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for cfg in "128 128 128" "256 256 64" "256 128 64" "128 128 64" "256 256 128" "128 256 128" "192 192 128"; do
  set -- $cfg
  MFC_SEG_X=$1 MFC_SEG_Y=$2 MFC_SEG_Z=$3 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $OUT/seg2_$1_$2_$3.json 2>/dev/null
done
