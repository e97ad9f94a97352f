#!/bin/bash
# usage: bash tools/gpu_cfg_sweep.sh CONFIG STEPS "ENV1" "ENV2" ...
CFG=$1; ST=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
for V in "$@"; do env $V timeout 600 python bench.py --config $CFG --steps $ST --warmup 3 --no-e2e --no-cpu > $OUT/cfg.json 2>/dev/null
python -c "
import json;d=json.load(open('$OUT/cfg.json'));print('$CFG $V',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['kernel_ms_per_step'].items()})"; done
