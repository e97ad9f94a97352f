#!/bin/bash
# x_tile vs x_rows: bitwise dumps, GPU parity with the tile kernel, same-box A/B
OUT=gpurun_out; mkdir -p $OUT
L=paper_2409_10729_b200
{
python tools/xvariant_dump.py /tmp/a.npz && MFC_X_TILE=1 python tools/xvariant_dump.py /tmp/b.npz && python tools/xvariant_dump.py --compare /tmp/a.npz /tmp/b.npz
MFC_X_TILE=1 MFC_LIB=$L/libmfc_xt3.so python tools/xvariant_dump.py /tmp/c.npz && python tools/xvariant_dump.py --compare /tmp/a.npz /tmp/c.npz
} > $OUT/xtile_bitwise.log 2>&1
MFC_X_TILE=1 timeout 900 python -m pytest tests -m gpu -q -x > $OUT/xtile_pytest.log 2>&1; echo "exit $?" >> $OUT/xtile_pytest.log
bash tools/gpu_ab.sh "MFC_X_TILE=0" "MFC_X_TILE=1" "MFC_X_TILE=1 MFC_LIB=$L/libmfc_xt3.so" "MFC_X_TILE=1 MFC_LIB=$L/libmfc_xt4.so" > $OUT/xtile_ab.log 2>&1
