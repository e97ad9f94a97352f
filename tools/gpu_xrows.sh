#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for R in 1 2 4 8; do MFC_XROWS=$R timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $OUT/xrows_$R.json 2>/dev/null; done
