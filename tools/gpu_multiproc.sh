#!/bin/bash
# Multi-process launches on ONE GPU (protocol checks; timings are time-sliced, not a
# scaling number): torchrun N = 2 with the fused halo over CUDA IPC (gloo plumbing, no
# NCCL), z-slabs of C4, per-step and the graph path through the bench.
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --same-device --halo peer --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/bench_peer2_samegpu_r209.json 2> $OUT/bench_peer2_samegpu_r209.err; echo "exit $?" >> $OUT/bench_peer2_samegpu_r209.err
