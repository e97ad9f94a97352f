#!/bin/bash
# r101: WENO5-M weights a_k = d_k P_k formed once (MFC_WENO5M_ALPHA) A/B + eps-range GPU tests
OUT=gpurun_out; mkdir -p $OUT
MFC_PARITY_LOG=$OUT/parity_r101.json timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "5m or mapped or uniform or eps" > $OUT/pytest_r101.log 2>&1; echo "exit $?" >> $OUT/pytest_r101.log
bash tools/gpu_abn.sh 3 "--weno 5m" paper_2409_10729_b200/libmfc.so paper_2409_10729_b200/libmfc_a0.so > $OUT/ab_weno5m_r101.txt 2>&1
