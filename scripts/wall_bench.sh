#!/bin/bash
# NEXT-1 wall-clock mode (A32): entry-major vs round-major kernels on configs 2, 3 and 5 (bench lines).
mkdir -p gpurun_out
for cfg in 2 3 5; do
  for rm in 0 1; do
    echo "== cfg$cfg MAGUS_WALL_ROUNDMAJOR=$rm"
    MAGUS_WALL_ROUNDMAJOR=$rm timeout 300 python bench.py --config $cfg --wallclock --steps 5 --warmup 3 --no-e2e \
      --preroll-ms 100 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read().strip()
try:
  d=json.loads(l); r=d['roofline']
  print(d['config']['workload'], 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f ms'%r['replay_ms'], 'frac %.3f'%r['frac'], 'clk', d['clocks']['sm_mhz'])
except Exception as e: print('ERR', l[-400:])
"
  done
done
