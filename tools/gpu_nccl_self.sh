#!/bin/bash
# MFC_TRANSPORT_NCCL_SELF on the B200: tests + the step cost of the NCCL halo path.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-t}
export PYTHONUNBUFFERED=1
NCCL_DEBUG=INFO timeout 900 python -m pytest tests/test_gpu_nccl_self.py -q -rf > $OUT/pytest_nccl_self_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_nccl_self_$TAG.log
timeout 600 python tools/halo_bench.py --nccl-self --steps 10 > $OUT/halo_nccl_self_$TAG.jsonl 2> $OUT/halo_nccl_self_$TAG.err
timeout 900 python -m pytest tests/test_capi.py tests/test_gpu_parity.py -q -x > $OUT/pytest_parity_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_parity_$TAG.log
