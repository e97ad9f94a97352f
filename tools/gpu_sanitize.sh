#!/bin/bash
# compute-sanitizer passes over small parity cases
TAG=${1:-r23}
OUT=gpurun_out; mkdir -p $OUT
SEL='degenerate or GR-2D-N2 or GR-3D-refl or C1 or eos or ghost or graph or wave_rate'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
    python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL and not 100_steps" > $OUT/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool exit $?" >> $OUT/sanitize_${tool}_$TAG.log
done
