#!/bin/bash
# two-length segment plan (MAGUS_SEG_BALANCE=1, default) vs uniform 32-multiple segments; cfg2 then cfg5, interleaved reps
run() {  # balance config
  MAGUS_SEG_BALANCE=$1 timeout 300 python bench.py --config $2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    --preroll-ms 300 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); g=d['segmentation']['geometry']
print('cfg%s balance=%s replay_ms %.4f step_ms %.4f S %d L %d ctas %d mism %d clk %s' % ('$2', '$1', d['roofline']['replay_ms'], d['ms_per_step'], g['n_segments'], g['segment_len'], g['ctas'], d['segmentation']['mismatched_segments'], d['clocks']['sm_mhz']))"
}
for rep in 1 2 3; do run 0 2; run 1 2; done
for rep in 1 2; do run 0 5; run 1 5; done
