#!/bin/bash
# solo kernel: two stages per loop iteration (-DMAGUS_SOLO_UNROLL=2) vs one, config 2, interleaved
TAG=${1:-r02u2}
OUT=gpurun_out; mkdir -p $OUT
LU=$PWD/paper_2502_03796_b200/lib/libmagus_u2.so
for rep in 1 2 3; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c2_u1_$rep.json 2>> $OUT/${TAG}.err
  MAGUS_LIB_PATH=$LU timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c2_u2_$rep.json 2>> $OUT/${TAG}.err
done
for f in $OUT/${TAG}_c2_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['roofline']['replay_ms_min'],4), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; done
