#!/bin/bash
# bench lines of the other BASELINE.json configs (1 GPU): 3 (64-point sweep), 4 (per-GPU shard), 5 (adversarial)
TAG=${1:-cfgs}
OUT=gpurun_out; mkdir -p $OUT
for c in 3 5 4; do
  timeout 900 python bench.py --config $c --no-e2e --steps 10 --warmup 3 > $OUT/${TAG}_cfg$c.json 2> $OUT/${TAG}_cfg$c.err
  echo "cfg$c rc=$?" >> $OUT/${TAG}_rc.txt
done
