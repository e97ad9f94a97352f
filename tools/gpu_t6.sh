#!/bin/bash
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_advance_host.py -m gpu -q -x > $OUT/t6_pytest.log 2>&1; echo "exit $?" >> $OUT/t6_pytest.log
for V in "MFC_STREAM_CE=1" "MFC_STREAM=-1" "MFC_STREAM=12" "MFC_STREAM=20"; do
  env $V timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $OUT/t6_b.json 2>$OUT/t6_b.err
  python -c "
import json;d=json.load(open('$OUT/t6_b.json'));print('$V',round(d['ms_per_step'],3),d['e2e'])" >> $OUT/t6_ab.log 2>&1
done
