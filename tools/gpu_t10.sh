#!/bin/bash
# r100: WENO5-M with one reciprocal per pair of divisions (MFC_WENO5M_ONE_RCP) — parity + same-box A/B
OUT=gpurun_out; mkdir -p $OUT
MFC_PARITY_LOG=$OUT/parity_weno5m_r100.json timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "5m or mapped" > $OUT/pytest_weno5m_r100.log 2>&1; echo "exit $?" >> $OUT/pytest_weno5m_r100.log
bash tools/gpu_abn.sh 3 "--weno 5m" paper_2409_10729_b200/libmfc.so paper_2409_10729_b200/libmfc_m0.so > $OUT/ab_weno5m_r100.txt 2>&1
timeout 300 python bench.py --weno 5m --steps 20 --warmup 3 --no-cpu > $OUT/bench_weno5m_r100.json 2> $OUT/bench_weno5m_r100.err
