# A/B: previous build (base) vs micro2 (shared 12 P1 in the WENO weight sums, periodic-row
# halo from the owners in the x pair) vs cs (micro2 + the march's carried face state in
# shared memory), with the parity subset on each candidate
export PYTHONUNBUFFERED=1
L=$PWD/paper_2409_10729_b200
for V in micro2 cs; do
MFC_LIB=$L/libmfc_$V.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "rhs_parity or 100_steps or graph or c3_full_rhs or c3_full_rk3 or c2_full" > gpurun_out/pytest_$V.log 2>&1; echo "exit $?" >> gpurun_out/pytest_$V.log
done
bash tools/gpu_abn.sh 3 "" $L/libmfc_base.so $L/libmfc_micro2.so $L/libmfc_cs.so > gpurun_out/ab_micro2.txt 2>&1
