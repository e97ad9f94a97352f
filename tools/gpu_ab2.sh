#!/bin/bash
# same-box A/B of two libmfc builds, alternating: bash tools/gpu_ab2.sh libA.so libB.so [reps] [bench args]
OUT=gpurun_out; mkdir -p $OUT
A=$1; B=$2; REPS=${3:-3}; shift 3
for rep in $(seq $REPS); do for L in $A $B; do MFC_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --sustained 0 "$@" > $OUT/ab.json 2>/dev/null
python -c "
import json;d=json.load(open('$OUT/ab.json'));print('$L',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['kernel_ms_per_step'].items()})"; done; done
