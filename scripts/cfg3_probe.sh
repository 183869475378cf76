#!/bin/bash
# config 3 (64-point sweep): step time vs the segment plan's target warps per SM
OUT=gpurun_out; mkdir -p $OUT
for tw in 12 24 48 96; do
  MAGUS_TARGET_WARPS_PER_SM=$tw timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 \
      > $OUT/c3_tw$tw.json 2>> $OUT/c3.err
  python -c "
import json; d=json.load(open('$OUT/c3_tw$tw.json')); s=d['segmentation']
print('tw $tw', 'step %.2f replay %.2f' % (d['ms_per_step'], d['roofline']['replay_ms']), 'segs', s['n_segments'], 'mism', s['mismatched_segments'], 'rounds', s['fixup_rounds'])" >> $OUT/c3_summary.txt
done
cat $OUT/c3_summary.txt
