#!/bin/bash
# F4 stretched grids: GPU stretched/fuzz tests on the candidate, A/B against HEAD
export PYTHONUNBUFFERED=1
L=$PWD/paper_2409_10729_b200
MFC_LIB=$L/libmfc_kv.so timeout 900 python -m pytest tests/test_gpu_stretched.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/pytest_kv.log 2>&1; tail -2 gpurun_out/pytest_kv.log
bash tools/gpu_abn.sh 3 "--stretch" $L/libmfc_HEAD.so $L/libmfc_kv.so > gpurun_out/ab_f4kv.txt 2>&1
cat gpurun_out/ab_f4kv.txt
