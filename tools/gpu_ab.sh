#!/bin/bash
# A/B of env-selected variants: bash tools/gpu_ab.sh "ENV1=.." "ENV2=.." ...
OUT=gpurun_out; mkdir -p $OUT
for V in "$@"; do for rep in 1 2; do env $V timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > $OUT/ab.json 2>/dev/null
python -c "
import json;d=json.load(open('$OUT/ab.json'));print('$V',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms_per_step'].items()})"; done; done
