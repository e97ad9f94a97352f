#!/bin/bash
# A/B of env-selected variants on a bench config: bash tools/gpu_cfg_ab.sh C5 "ENV1=.." "ENV2=.." ...
CFG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for V in "$@"; do for rep in 1 2; do env $V timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/ab_$CFG.json 2>/dev/null
python -c "
import json;d=json.load(open('$OUT/ab_$CFG.json'));print('$CFG','$V',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms_per_step'].items()})"; done; done
