#!/bin/bash
# ncu evidence for round 2: default build (launch list + full capture of one x/y/z
# sweep), the TMA variants (full capture of their sweep), and the march-unroll A/B.
# usage (under gpurun): bash tools/gpu_prof_r2.sh TAG
TAG=${1:-r206}
OUT=gpurun_out; mkdir -p $OUT
L=$PWD/paper_2409_10729_b200
export PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_bench_$TAG.log 2>&1
# warm-up 3 steps x 9 sweeps; profiled pass runs after the timed steps: skip 3*9 + 2*9
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 45 -c 3 -o $OUT/prof_$TAG python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_full_$TAG.log 2>&1
MFC_LIB=$L/libmfc_xtma1np.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_x -s 15 -c 1 -o $OUT/prof_${TAG}_xtma python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_full_${TAG}_xtma.log 2>&1
MFC_LIB=$L/libmfc_ytma.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 30 -c 1 -o $OUT/prof_${TAG}_ytma python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_full_${TAG}_ytma.log 2>&1
bash tools/gpu_abn.sh 2 "" $L/libmfc.so $L/libmfc_u2.so $L/libmfc_u3.so > $OUT/ab_unroll_$TAG.txt 2>&1
