#!/bin/bash
OUT=gpurun_out; L=paper_2409_10729_b200
{ MFC_LIB=$L/libmfc_a694a9d.so python tools/xvariant_dump.py /tmp/a.npz && python tools/xvariant_dump.py /tmp/b.npz && python tools/xvariant_dump.py --compare /tmp/a.npz /tmp/b.npz; } > $OUT/t2_bitwise.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decomp.py tests/test_gpu_fullsize.py -m gpu -q -x > $OUT/t2_pytest.log 2>&1; echo "exit $?" >> $OUT/t2_pytest.log
bash tools/gpu_ab.sh "MFC_LIB=$L/libmfc_a694a9d.so" "MFC_XT_GRID=-1" "MFC_XT_GRID=0" "MFC_LIB=$L/libmfc_a694a9d.so" "MFC_XT_GRID=-1" > $OUT/t2_ab.log 2>&1
