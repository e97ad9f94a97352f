#!/bin/bash
# Halo kernels (coalesced face order): decomposition / fused / NCCL-self tests, the
# loopback halo bench and the NCCL-self step.  usage: bash tools/gpu_halo_r2.sh TAG
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-t}
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_nccl_self.py tests/test_gpu_decomp.py tests/test_gpu_fused_halo.py tests/test_gpu_parity.py tests/test_gpu_stretched.py -q -rf > $OUT/pytest_halo_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_halo_$TAG.log
timeout 600 python tools/halo_bench.py --nccl-self --steps 10 > $OUT/halo_nccl_self_$TAG.jsonl 2> $OUT/halo_nccl_self_$TAG.err
timeout 900 python tools/halo_bench.py --steps 10 > $OUT/halo_$TAG.jsonl 2> $OUT/halo_$TAG.err
