#!/bin/bash
# NVTX ranges (domain "mfc"): ncu launch lists filtered by range, then the bench and a
# test subset to show the ranges cost nothing.  usage: bash tools/gpu_nvtx.sh TAG
TAG=${1:-nvtx}
OUT=gpurun_out; mkdir -p $OUT
python tools/nvtx_demo.py > $OUT/nvtx_demo_$TAG.log 2>&1
for R in "mfc@mfc_rk3_step/" "mfc@RK3 stage 2/" "mfc@sweep z/" "mfc@mfc_rhs/"; do
  F=$(echo "$R" | tr -c 'a-zA-Z0-9\n' '_')
  timeout 300 ncu --nvtx --nvtx-include "$R" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/nvtx_${F}_$TAG.csv python tools/nvtx_demo.py > $OUT/nvtx_${F}_$TAG.log 2>&1
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decomp.py tests/test_capi.py -m gpu -q -x > $OUT/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_$TAG.log
