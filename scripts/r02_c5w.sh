#!/bin/bash
# config 5 (fused kernel): speculative warm-up 32 / 64 ticks fixed vs the adaptive default (96 after the first walk)
TAG=${1:-r02c5w}
OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2; do
  timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 --preroll-ms 300 > $OUT/${TAG}_adapt_$rep.json 2>> $OUT/${TAG}.err
  MAGUS_NO_WARM_ADAPT=1 timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 --preroll-ms 300 > $OUT/${TAG}_w32_$rep.json 2>> $OUT/${TAG}.err
  MAGUS_NO_WARM_ADAPT=1 MAGUS_WARMUP_EXTRA=32 timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 --preroll-ms 300 > $OUT/${TAG}_w64_$rep.json 2>> $OUT/${TAG}.err
done
for f in $OUT/${TAG}_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), d['segmentation']['warmup_ticks'], d['segmentation']['mismatched_segments'], d['clocks']['sm_mhz'])"; done
