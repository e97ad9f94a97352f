#!/bin/bash
# x_rows block width sweep: MFC_XW = warps per row segment
OUT=gpurun_out; mkdir -p $OUT
for W in 2 4 8 16; do MFC_XW=$W timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $OUT/xw_$W.json 2>/dev/null
python -c "
import json;d=json.load(open('$OUT/xw_$W.json'));print('W=$W',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms_per_step'].items()})"; done
