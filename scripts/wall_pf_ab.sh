#!/bin/bash
# wall-clock kernel prefetch depth A/B (build variants under variants/; default build = 8 entries)
for rep in 1 2; do
for lib in paper_2502_03796_b200/lib/libmagus_replay.so variants/libwall_pf4.so variants/libwall_pf16.so; do
  for cfg in 2 3; do
    r=$(MAGUS_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config $cfg --wallclock --steps 3 --warmup 3 --no-e2e --preroll-ms 50 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f'%d['roofline']['replay_ms'])" 2>&1)
    echo "rep$rep $(basename $lib) cfg$cfg replay_ms=$r"
  done
done
done
