#!/bin/bash
# fused MAGUS + TDP kernel (config 5): GPU suite, then cfg5 A/B (unfused / fused at 12 and 16 CTAs per SM)
TAG=${1:-r02f1}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k fused > $OUT/${TAG}_pytest_fused.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest_fused.log; tail -3 $OUT/${TAG}_pytest_fused.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest.log; tail -3 $OUT/${TAG}_pytest.log
for rep in 1 2; do
  for v in u f12 f16; do
    case $v in u) E="MAGUS_FUSE=0";; f12) E="MAGUS_FUSE=1 MAGUS_FUSED_CTAS=12";; f16) E="MAGUS_FUSE=1 MAGUS_FUSED_CTAS=16";; esac
    env $E timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 --preroll-ms 300 \
        > $OUT/${TAG}_c5_${v}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for f in $OUT/${TAG}_c5_*.json; do
  python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), d['segmentation']['geometry']['n_segments'], d['segmentation'].get('mismatched_segments'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
done
