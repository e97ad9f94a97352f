# A/B of TMA variants against the default build (same box): x pair one-segment-per-block
# TMA (xtma1np), TMA rings in the y/z marches (ytma)
export PYTHONUNBUFFERED=1
L=$PWD/paper_2409_10729_b200
for V in xtma1np ytma; do
MFC_LIB=$L/libmfc_$V.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "rhs_parity or (100_steps and (C3-24 or GR-3D-520)) or graph or c3_full_rhs or c3_full_rk3 or c2_full" > gpurun_out/pytest_$V.log 2>&1; echo "exit $?" >> gpurun_out/pytest_$V.log
done
bash tools/gpu_abn.sh 3 "" $L/libmfc.so $L/libmfc_xtma1np.so $L/libmfc_ytma.so > gpurun_out/ab_tma3.txt 2>&1
