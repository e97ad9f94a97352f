# A/B: x pair with 16-byte loads (vecin: input only; vec: input and the RK-base / store
# epilogue) against the previous build; parity subset on both
export PYTHONUNBUFFERED=1
L=$PWD/paper_2409_10729_b200
for V in vec vecin; do
MFC_LIB=$L/libmfc_$V.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "rhs_parity or (100_steps and not C3-160) or graph or c3_full_rhs or c3_full_rk3 or c2_full" > gpurun_out/pytest_$V.log 2>&1; echo "exit $?" >> gpurun_out/pytest_$V.log
done
bash tools/gpu_abn.sh 3 "" $L/libmfc_base.so $L/libmfc_vec.so $L/libmfc_vecin.so > gpurun_out/ab_vec.txt 2>&1
