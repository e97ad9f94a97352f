# A/B of the persistent TMA x-pair variants against the default build (same box)
export PYTHONUNBUFFERED=1
L=$PWD/paper_2409_10729_b200
MFC_LIB=$L/libmfc_xtma2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "rhs_parity or (100_steps and (C3-24 or GR-3D-520)) or graph or c3_full_rhs or c3_full_rk3 or c2_full" > gpurun_out/pytest_xtma2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_xtma2.log
bash tools/gpu_abn.sh 3 "" $L/libmfc.so $L/libmfc_xtma2.so $L/libmfc_xtma1.so > gpurun_out/ab_xtma2.txt 2>&1
