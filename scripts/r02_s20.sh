#!/bin/bash
# cfg 2 step overhead A/B: totals chunk 256 (default) vs 64 traces, prepass 32x32 vs 16x64; interleaved, 4 reps
TAG=${1:-r02s20}
OUT=gpurun_out; mkdir -p $OUT
L=paper_2502_03796_b200/lib
for rep in 1 2 3 4; do
  for v in base t64 t64p16; do
    if [ $v = base ]; then LP=$L/libmagus_replay.so; else LP=$L/libmagus_replay_$v.so; fi
    MAGUS_LIB_PATH=$LP timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 50 --preroll-ms 300 > $OUT/${TAG}_${v}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for v in base t64 t64p16; do
  python -c "
import json,glob
r=[json.load(open(f)) for f in sorted(glob.glob('$OUT/${TAG}_${v}_*.json'))]
print('$v', [(round(d['ms_per_step'],4), round(d['roofline']['replay_ms'],4), round(d['ms_per_step']-d['roofline']['replay_ms'],4), d['clocks']['sm_mhz']) for d in r])"
done
