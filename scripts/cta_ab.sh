#!/bin/bash
# solo kernel: one-warp CTAs per SM (register budget) x TMA stages; interleaved reps, cfg2 bench lines
run() {  # name lib target
  MAGUS_LIB_PATH=$PWD/$2 MAGUS_TARGET_WARPS_PER_SM=$3 timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e \
    --no-cpu-baseline --preroll-ms 300 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); g=d['segmentation']['geometry']
print('%-10s replay_ms %.4f step_ms %.4f S %d ctas %d mism %d clk %s' % ('$1', d['roofline']['replay_ms'], d['ms_per_step'], g['n_segments'], g['ctas'], d['segmentation']['mismatched_segments'], d['clocks']['sm_mhz']))"
}
for rep in 1 2 3; do
  run base paper_2502_03796_b200/lib/libmagus_replay.so 16
  run cta20ns2 variants/libsolo_cta20_ns2.so 20
  run cta24ns2 variants/libsolo_cta24_ns2.so 24
done
