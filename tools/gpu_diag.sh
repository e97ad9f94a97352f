#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
python tools/diag_c1.py > $OUT/diag_c1.log 2>&1
# ncu: every launch of one short bench run (cold-cache, serialised)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_bench.log 2>&1
# full capture of sweep_y (the 2nd sweep kernel), one launch after warm-up
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 10 -c 2 -o $OUT/prof_r01 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_full.log 2>&1
ls -la $OUT
