#!/bin/bash
# open-loop fast path (O stage + closed-form fix-up): open-loop GPU tests, then config-2 open-loop bench A/B
TAG=${1:-r02ol}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "open_loop or fused or small_configs" > $OUT/${TAG}_pytest.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest.log; grep -E "passed|failed|wrong entries" $OUT/${TAG}_pytest.log | tail -15
for rep in 1 2; do
  for f in 0 1; do
    MAGUS_OPEN_FAST=$f timeout 300 python bench.py --open-loop --no-e2e --steps 20 > $OUT/${TAG}_c2_f${f}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for f in $OUT/${TAG}_c2_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['segmentation']['mismatched_segments'], d['clocks']['sm_mhz'])"; done
