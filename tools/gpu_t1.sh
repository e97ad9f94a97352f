OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/t1_pytest.log 2>&1; echo "exit $?" >> $OUT/t1_pytest.log
MFC_X_ROWS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decomp.py -m gpu -q -x > $OUT/t1_pytest_rows1.log 2>&1; echo "exit $?" >> $OUT/t1_pytest_rows1.log
bash tools/gpu_ab.sh "MFC_X_ROWS=-1" > $OUT/t1_ab_c3.log 2>&1
bash tools/gpu_cfg_ab.sh C5 "MFC_X_ROWS=-1" "MFC_X_ROWS=1" > $OUT/t1_ab_c5.log 2>&1
bash tools/gpu_cfg_ab.sh C2 "MFC_X_ROWS=-1" "MFC_X_ROWS=1" > $OUT/t1_ab_c2.log 2>&1
