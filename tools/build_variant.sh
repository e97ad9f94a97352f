#!/bin/bash
# Build the WORKING TREE's CUDA sources with extra nvcc flags into
# paper_2409_10729_b200/libmfc_TAG.so (same-box A/B timing via MFC_LIB=...).
# usage: tools/build_variant.sh TAG "-DMFC_RING_PD=1 -DMFC_RKACC_MINB=3"
TAG=$1; shift
D=paper_2409_10729_b200/csrc
OUT=paper_2409_10729_b200/libmfc_$TAG.so
T=$(mktemp -d)
for f in mfc sweep_n1 sweep_n2 sweep_n3; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -Xptxas -v -Iinclude $@ -c $D/$f.cu -o $T/$f.o > $T/$f.log 2>&1 || { cat $T/$f.log | grep -i error; exit 1; } &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $T/*.o -lnccl && echo $OUT
python - $T/sweep_n2.log <<'PY'
import sys,re
t=open(sys.argv[1]).read().split("ptxas info    : Compiling entry function ")
for blk in t[1:]:
    name=blk.split("'")[1]
    m=re.search(r'Used (\d+) registers',blk)
    if not m: continue
    sp=re.search(r'(\d+) bytes spill stores',blk).group(1)
    if 'Li2ELi3EEE' in name and 'Li5E' in name: print(name[:70], m.group(1), 'spill', sp)
PY
rm -rf $T
