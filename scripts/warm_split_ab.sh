#!/bin/bash
# mid-block warm-up / steady switch (current build) vs whole warm-up blocks (variants/libold.so), interleaved
run() {
  MAGUS_LIB_PATH=$PWD/$2 timeout 300 python bench.py --config $3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    --preroll-ms 300 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('cfg%s %-6s replay_ms %.4f step_ms %.4f clk %s' % ('$3', '$1', d['roofline']['replay_ms'], d['ms_per_step'], d['clocks']['sm_mhz']))"
}
for rep in 1 2 3; do run old variants/libold.so 2; run new paper_2502_03796_b200/lib/libmagus_replay.so 2; done
for rep in 1 2; do run old variants/libold.so 5; run new paper_2502_03796_b200/lib/libmagus_replay.so 5; done
