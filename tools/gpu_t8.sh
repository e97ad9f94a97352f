#!/bin/bash
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_advance_host.py tests/test_gpu_fullsize.py -m gpu -q -x > $OUT/t8_pytest.log 2>&1; echo "exit $?" >> $OUT/t8_pytest.log
MFC_STREAM_TRACE=1 python tools/e2e_diag.py > $OUT/e2e_diag.log 2>&1
for V in "MFC_STREAM_PITCHED=1" "MFC_STREAM=-1" "MFC_STREAM=64" "MFC_STREAM=16"; do
  env $V timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $OUT/t8_b.json 2>$OUT/t8_b.err
  python -c "
import json;d=json.load(open('$OUT/t8_b.json'));print('$V',round(d['ms_per_step'],3),d['e2e']['value'])" >> $OUT/t8_ab.log 2>&1
done
