#!/bin/bash
# same-box A/B/... of libmfc builds, round-robin: bash tools/gpu_abn.sh REPS "bench args" libA.so libB.so ...
OUT=gpurun_out; mkdir -p $OUT
REPS=$1; ARGS=$2; shift 2
for rep in $(seq $REPS); do for L in "$@"; do MFC_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --sustained 0 $ARGS > $OUT/ab.json 2>/dev/null
python -c "
import json;d=json.load(open('$OUT/ab.json'));print('$L',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['kernel_ms_per_step'].items()})"; done; done
