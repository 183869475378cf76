#!/bin/bash
# geometry sweep of the replay kernel (bench config 2); one summary line per setting
for ng in ${NGS:-8}; do
  for extra in ${EXTRAS:-32}; do for tw in ${TWS:-8 4}; do
    MAGUS_NG=$ng MAGUS_TARGET_WARPS_PER_SM=$tw MAGUS_WARMUP_EXTRA=$extra timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --preroll-ms 200 > /tmp/b.json 2>/dev/null
    python -c "
import json;d=json.load(open('/tmp/b.json'));k=d['kernel_ms'];s=d['segmentation']
print('ng=$ng tw=$tw extra=$extra', 'S=',s['n_segments'],'mism=',s['mismatched_segments'],'replay=%.3f fix=%.3f run=%.3f'%(k['replay_ms'],k['fixup_epilogue_ms'],k['run_ms']),'frac=%.3f'%d['roofline']['frac'])"
  done; done
done
