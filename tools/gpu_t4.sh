#!/bin/bash
OUT=gpurun_out; L=paper_2409_10729_b200; REF=${1:-8209603}
{ MFC_LIB=$L/libmfc_$REF.so python tools/xvariant_dump.py /tmp/a.npz && python tools/xvariant_dump.py /tmp/b.npz && python tools/xvariant_dump.py --compare /tmp/a.npz /tmp/b.npz; } > $OUT/t4_bitwise.log 2>&1
bash tools/gpu_ab.sh "MFC_LIB=$L/libmfc_$REF.so" "MFC_X_ROWS=1" "MFC_LIB=$L/libmfc_$REF.so" "MFC_X_ROWS=1" > $OUT/t4_ab.log 2>&1
