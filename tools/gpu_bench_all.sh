#!/bin/bash
# bench lines for C3 (default), C5 and C2, torchrun launcher sanity, ncu evidence
TAG=${1:-r16}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python bench.py --steps 20 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/bench_C5_$TAG.json 2> $OUT/bench_C5_$TAG.err
timeout 600 python bench.py --config C2 --steps 50 --warmup 5 --no-cpu > $OUT/bench_C2_$TAG.json 2> $OUT/bench_C2_$TAG.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/bench_torchrun_$TAG.json 2> $OUT/bench_torchrun_$TAG.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
bash tools/gpu_ncu.sh $TAG
