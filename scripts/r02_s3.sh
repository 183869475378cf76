#!/bin/bash
# cfg 3 / cfg 5: step and wrong entries vs the speculative warm-up length (MAGUS_WARMUP_EXTRA ticks on top of
# roundup32(k + C - 1)).  usage: bash scripts/r02_s3.sh TAG
TAG=${1:-r02s3}
OUT=gpurun_out; mkdir -p $OUT
for x in 0 224 480 992 1984; do
  MAGUS_WARMUP_EXTRA=$x timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_cfg3_w$x.txt 2>&1
done
for x in 0 224 480 992; do
  MAGUS_WARMUP_EXTRA=$x timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_cfg5_w$x.txt 2>&1
done
for f in $OUT/${TAG}_cfg*.txt; do echo "$f: $(cut -c1-200 $f)"; done > $OUT/${TAG}_summary.txt
cat $OUT/${TAG}_summary.txt
