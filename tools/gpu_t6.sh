#!/bin/bash
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_advance_host.py tests/test_gpu_fullsize.py -m gpu -q -x > $OUT/t6_pytest.log 2>&1; echo "exit $?" >> $OUT/t6_pytest.log
for V in "MFC_STREAM=0" "MFC_STREAM=16" "MFC_STREAM=32" "MFC_STREAM=64" "MFC_STREAM=128"; do
  env $V timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $OUT/t6_b.json 2>$OUT/t6_b.err
  python -c "
import json;d=json.load(open('$OUT/t6_b.json'));print('$V',round(d['ms_per_step'],3),d['e2e'])" >> $OUT/t6_ab.log 2>&1
done
