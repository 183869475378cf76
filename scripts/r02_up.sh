#!/bin/bash
# fused kernel with the TDP f_min-always-rises specialisation (MAGUS_FUSED_UP=1, default) vs without: fused / random
# GPU tests + config 5 A/B
TAG=${1:-r02up}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fused or randomized or ragged or full_size_every_trace" > $OUT/${TAG}_pytest.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest.log; tail -2 $OUT/${TAG}_pytest.log; grep -E "^E  " $OUT/${TAG}_pytest.log | head -3
for rep in 1 2; do
  for u in 0 1; do
    MAGUS_FUSED_UP=$u timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 --preroll-ms 300 > $OUT/${TAG}_c5_u${u}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for f in $OUT/${TAG}_c5_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), d['segmentation']['mismatched_segments'], d['clocks']['sm_mhz'])"; done
