#!/bin/bash
# libmfc's NCCL halo with two ranks on one GPU (tools/nccl_samegpu.py).
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1 NCCL_DEBUG=WARN
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 tools/nccl_samegpu.py > $OUT/nccl_samegpu_${1:-t}.log 2>&1; echo "exit $?" >> $OUT/nccl_samegpu_${1:-t}.log
