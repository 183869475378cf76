#!/bin/bash
# GPU tests + bench with the one-warp solo kernel (default) and without it (MAGUS_SOLO=0), 1 GPU
TAG=${1:-ab}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for v in 1 0 1; do
  MAGUS_SOLO=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline > $OUT/${TAG}_bench_solo$v.json 2>> $OUT/${TAG}_bench.err
done
echo done
