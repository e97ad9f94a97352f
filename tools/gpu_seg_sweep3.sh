#!/bin/bash
# segment lengths of the y / z march sweeps (x is the row tile), C3 256^3
OUT=gpurun_out; mkdir -p $OUT
for cfg in "0 0" "64 64" "256 64" "128 128" "256 128" "128 32" "256 256"; do
  set -- $cfg
  if [ $1 = 0 ]; then E=""; else E="MFC_SEG_Y=$1 MFC_SEG_Z=$2"; fi
  env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $OUT/seg3.json 2>/dev/null
  python -c "
import json;d=json.load(open('$OUT/seg3.json'));print('y=$1 z=$2',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms_per_step'].items()})" >> $OUT/seg3.log
done
