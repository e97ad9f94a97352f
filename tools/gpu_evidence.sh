#!/bin/bash
# Round evidence (under gpurun): GPU tests with the parity log, smoke, bench lines for
# C3 (default), C5, C2, C3 stretched, WENO3 / WENO5-M, the torchrun launch, the reference
# arm, DRAM bytes of the 9 sweep launches of one step, and the F1 loopback halo timing.
# usage: bash tools/gpu_evidence.sh TAG
TAG=${1:-r2}
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
MFC_PARITY_LOG=$OUT/parity_$TAG.json timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/bench_C5_$TAG.json 2> $OUT/bench_C5_$TAG.err
timeout 600 python bench.py --config C2 --steps 50 --warmup 5 --no-cpu > $OUT/bench_C2_$TAG.json 2> $OUT/bench_C2_$TAG.err
timeout 600 python bench.py --stretch --steps 20 --warmup 3 --no-cpu > $OUT/bench_stretch_$TAG.json 2> $OUT/bench_stretch_$TAG.err
timeout 600 python bench.py --weno 3 --steps 20 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/bench_weno3_$TAG.json 2> $OUT/bench_weno3_$TAG.err
timeout 600 python bench.py --weno 5m --steps 20 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/bench_weno5m_$TAG.json 2> $OUT/bench_weno5m_$TAG.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu > $OUT/bench_torchrun_$TAG.json 2> $OUT/bench_torchrun_$TAG.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sweep -s 45 -c 9 --csv --log-file $OUT/ncu_dram9_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_dram9_$TAG.log 2>&1
timeout 900 python tools/halo_bench.py --steps 10 > $OUT/halo_$TAG.jsonl 2> $OUT/halo_$TAG.err
