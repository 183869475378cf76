#!/bin/bash
TAG=${1:-r02s14}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
grep -E "^FAILED|passed|failed|rc=" $OUT/${TAG}_pytest_gpu.log | tail -12
