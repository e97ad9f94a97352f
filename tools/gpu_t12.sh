#!/bin/bash
# r102: WENO3 one reciprocal for both sides (MFC_WENO3_ONE_RCP) A/B, then the full GPU
# suite, smoke and bench/ncu evidence for the final build of the round
OUT=gpurun_out; mkdir -p $OUT
bash tools/gpu_abn.sh 3 "--weno 3" paper_2409_10729_b200/libmfc.so paper_2409_10729_b200/libmfc_w30.so > $OUT/ab_weno3_r102.txt 2>&1
bash tools/gpu_check.sh r102 noncu
bash tools/gpu_bench_all.sh r102b
