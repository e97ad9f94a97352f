#!/bin/bash
# compute-sanitizer passes (memcheck, racecheck, synccheck, initcheck) over small parity
# cases that run every default kernel: the x pair and x tile (incl. multi-segment rows),
# the curvature-carry y/z marches (3D accumulate), the 1D/2D marches, WENO3 / WENO5-M,
# the stretched-grid kernels (ORD 7), EOS, wave rate, CUDA graphs, fused-halo peer
# stores (loopback groups), the streamed advance_host (three streams), the one-launch
# halo pack / unpack and the NCCL self-exchange.
# usage (under gpurun): bash tools/gpu_sanitize.sh TAG
TAG=${1:-r2}
OUT=gpurun_out; mkdir -p $OUT
HEAD=$(cat .git_head 2>/dev/null || echo unknown)
SEL_P='(rhs_parity and (C1 or C3-40 or GR-3D-refl or long-rows or GR-2D-N3 or degenerate)) or eos or ghost or graph or wave_rate or weno3_rhs_parity or weno5m_rhs_parity'
for tool in memcheck racecheck synccheck initcheck; do
  LOG=$OUT/sanitize_${tool}_$TAG.log
  echo "HEAD $HEAD" > $LOG
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
    python -m pytest -q -x -p no:cacheprovider \
      "tests/test_gpu_parity.py" -k "$SEL_P" >> $LOG 2>&1
  echo "$tool parity exit $?" >> $LOG
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
    python -m pytest -q -x -p no:cacheprovider tests/test_gpu_stretched.py tests/test_gpu_fused_halo.py \
      tests/test_gpu_advance_host.py \
      -k "(rhs_parity and (C3-40-st or long-rows)) or (decomposition and procs1) or (bitwise_3d and procs3) or dims_and_bcs or periodic-water or (chunk_counts and 3-)" >> $LOG 2>&1
  echo "$tool stretched/fused/advance exit $?" >> $LOG
  # r2 pack / unpack kernels (one launch for all faces) and the NCCL self transport
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
    python -m pytest -q -x -p no:cacheprovider tests/test_gpu_decomp.py tests/test_gpu_nccl_self.py \
      -k "(bitwise and (procs0 or procs3)) or nonperiodic or (nccl_self_exchange_bitwise and (case0 or case1))" >> $LOG 2>&1
  echo "$tool halo/nccl-self exit $?" >> $LOG
done
