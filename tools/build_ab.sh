#!/bin/bash
# Build the CUDA sources of git revision REV into paper_2409_10729_b200/libmfc_REV.so
# for same-box A/B timing (bench.py / tests honour MFC_LIB=<path>).
REV=$1
T=$(mktemp -d)
git archive $REV paper_2409_10729_b200/csrc include | tar -x -C $T
OUT=paper_2409_10729_b200/libmfc_$REV.so
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -I$T/include $T/paper_2409_10729_b200/csrc/{mfc,sweep_n1,sweep_n2,sweep_n3}.cu \
  -o $OUT -lnccl -lcuda && echo $OUT
rm -rf $T
