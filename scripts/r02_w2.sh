#!/bin/bash
# wide kernel traces per CTA: 16 vs the balanced 14 (MAGUS_WIDE_TPC): wide-plan GPU tests + config 3 A/B
TAG=${1:-r02w2}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "wide or full_size_every_trace or randomized" > $OUT/${TAG}_pytest.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest.log; tail -3 $OUT/${TAG}_pytest.log; grep -E "^E  " $OUT/${TAG}_pytest.log | head -3
for rep in 1 2; do
  for w in 16 14; do
    MAGUS_WIDE_TPC=$w timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 --preroll-ms 300 \
        > $OUT/${TAG}_c3_w${w}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for f in $OUT/${TAG}_c3_*.json; do
  python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), d['segmentation']['geometry']['threads_per_cta'], d['segmentation']['geometry']['ctas'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
