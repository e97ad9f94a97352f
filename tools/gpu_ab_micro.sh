# A/B of the current build (micro: shared 12 P1 in the WENO weight sums, one product
# fewer in HLLC's reciprocal algebra, periodic-row halo from the owners in the x pair)
# against the previous build, plus the parity subset on the new build
export PYTHONUNBUFFERED=1
L=$PWD/paper_2409_10729_b200
MFC_LIB=$L/libmfc_micro.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "rhs_parity or (100_steps and (C3-24 or C1 or GR-3D-520)) or graph or c3_full_rhs or c3_full_rk3 or c2_full" > gpurun_out/pytest_micro.log 2>&1; echo "exit $?" >> gpurun_out/pytest_micro.log
bash tools/gpu_abn.sh 4 "" $L/libmfc_base.so $L/libmfc_micro.so > gpurun_out/ab_micro.txt 2>&1
