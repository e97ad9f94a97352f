#!/bin/bash
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/t7_pytest.log 2>&1; echo "exit $?" >> $OUT/t7_pytest.log
bash tools/gpu_sanitize.sh r56
