#!/bin/bash
# config 2 / config 5: exact warm-up vs the synthetic full warm-up state (MAGUS_SOLO_SYNTH=1) with the L-stage kernels
TAG=${1:-r02syn}
OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2 3; do
  for sy in 0 1; do
    MAGUS_SOLO_SYNTH=$sy timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c2_s${sy}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for f in $OUT/${TAG}_c2_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['segmentation']['mismatched_segments'])"; done
