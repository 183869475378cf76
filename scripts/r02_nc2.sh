#!/bin/bash
# wide kernel: two chains per thread with the P stage (MAGUS_WIDE_NC=2) vs one (config 3), plus the wide tests with NC=2
TAG=${1:-r02nc2}
OUT=gpurun_out; mkdir -p $OUT
MAGUS_WIDE_NC=2 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "wide or full_size_every_trace or randomized" > $OUT/${TAG}_pytest.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest.log; tail -3 $OUT/${TAG}_pytest.log; grep -E "^E  " $OUT/${TAG}_pytest.log | head -3
for rep in 1 2; do
  for nc in 1 2; do
    MAGUS_WIDE_NC=$nc timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 --preroll-ms 300 \
        > $OUT/${TAG}_c3_nc${nc}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for f in $OUT/${TAG}_c3_*.json; do
  python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), d['segmentation']['geometry']['threads_per_cta'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
done
