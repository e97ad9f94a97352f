#!/bin/bash
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_advance_host.py -m gpu -q -x > $OUT/t9_pytest.log 2>&1; echo "exit $?" >> $OUT/t9_pytest.log
MFC_STREAM=48 MFC_STREAM_TRACE=1 python tools/e2e_diag.py > $OUT/e2e_diag.log 2>&1
for V in "MFC_STREAM=40" "MFC_STREAM=48" "MFC_STREAM=64" "MFC_STREAM=85"; do
  env $V timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $OUT/t9_b.json 2>$OUT/t9_b.err
  python -c "
import json;d=json.load(open('$OUT/t9_b.json'));print('$V',round(d['ms_per_step'],3),d['e2e']['value'])" >> $OUT/t9_ab.log 2>&1
done
