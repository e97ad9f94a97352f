#!/bin/bash
# One gpurun session: GPU tests (parity log), smoke, bench, optional ncu capture.
# usage (from repo root, under gpurun): bash tools/gpu_check.sh TAG [ncu]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
MFC_PARITY_LOG=$OUT/parity_$TAG.json timeout 1500 python -m pytest tests -m gpu -q -rf --durations=12 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
if [ "$2" == "ncu" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 27 -c 3 -o $OUT/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_full_$TAG.log 2>&1
fi
