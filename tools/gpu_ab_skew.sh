# A/B: the software-pipelined y/z march (skew) against the default build; parity on it
export PYTHONUNBUFFERED=1
L=$PWD/paper_2409_10729_b200
cp $L/libmfc.so $L/libmfc_base.so
MFC_LIB=$L/libmfc_skew.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_decomp.py tests/test_gpu_fused_halo.py -q -k "not C3-160" > gpurun_out/pytest_skew.log 2>&1; echo "exit $?" >> gpurun_out/pytest_skew.log
bash tools/gpu_abn.sh 3 "" $L/libmfc_base.so $L/libmfc_skew.so > gpurun_out/ab_skew.txt 2>&1
bash tools/gpu_abn.sh 1 "--config C5" $L/libmfc_base.so $L/libmfc_skew.so >> gpurun_out/ab_skew.txt 2>&1
