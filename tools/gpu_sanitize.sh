#!/bin/bash
# compute-sanitizer passes over small parity cases: the sweep kernels
# (x tile incl. multi-segment rows, y/z march), EOS, ghost fills, graphs, wave rate,
# and the streamed advance_host (chunk copies, three streams)
TAG=${1:-r23}
OUT=gpurun_out; mkdir -p $OUT
SEL='degenerate or GR-2D-N2 or GR-3D-refl or long-rows or C1 or eos or ghost or graph or wave_rate'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_advance_host.py -q -x \
    -k "($SEL and not 100_steps) or periodic-water or small_grid" > $OUT/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool exit $?" >> $OUT/sanitize_${tool}_$TAG.log
done
