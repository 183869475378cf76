#!/bin/bash
TAG=${1:-r02s18}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for rep in 1 2; do MAGUS_WARMUP_EXTRA=64 timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_cfg5_$rep.txt 2>&1; done
tail -2 $OUT/${TAG}_pytest_gpu.log; grep FAILED $OUT/${TAG}_pytest_gpu.log | head; cut -c1-200 $OUT/${TAG}_cfg5_*.txt
