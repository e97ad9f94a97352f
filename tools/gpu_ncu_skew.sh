OUT=gpurun_out; L=$PWD/paper_2409_10729_b200
MFC_LIB=$L/libmfc_skew.so timeout 900 ncu --set full --clock-control none -k regex:sweep_march_skew -s 30 -c 1 -o $OUT/prof_r211_skew python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained 0 > $OUT/ncu_full_r211_skew.log 2>&1
