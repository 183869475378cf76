#!/bin/bash
# full GPU suite (incl. the debug-check build tests) + dependent-latency probe
TAG=${1:-r02e2}
OUT=gpurun_out; mkdir -p $OUT
./scripts/lat_probe > $OUT/${TAG}_lat.txt 2>&1; cat $OUT/${TAG}_lat.txt
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=5 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
tail -3 $OUT/${TAG}_pytest_gpu.log
