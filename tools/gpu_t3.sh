#!/bin/bash
OUT=gpurun_out; L=paper_2409_10729_b200
bash tools/gpu_check.sh r51
bash tools/gpu_cfg_ab.sh C5 "MFC_X_ROWS=1" "MFC_LIB=$L/libmfc_big3.so" > $OUT/t3_ab_c5.log 2>&1
timeout 600 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu > $OUT/bench_C2_r51.json 2>/dev/null
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu > $OUT/bench_C5_r51.json 2>/dev/null
