#!/bin/bash
# solo kernel occupancy A/B: 16 one-warp CTAs per SM (128 registers, the default) vs 18 (96 registers; the L stage
# fits without spills in its loop), config 2 and config 4 shard; interleaved
TAG=${1:-r02occ}
OUT=gpurun_out; mkdir -p $OUT
L18=$PWD/paper_2502_03796_b200/lib/libmagus_solo18.so
MAGUS_LIB_PATH=$L18 MAGUS_TARGET_WARPS_PER_SM=18 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "small_configs or full_size_every_trace" > $OUT/${TAG}_pytest18.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest18.log; tail -2 $OUT/${TAG}_pytest18.log
for rep in 1 2 3; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c2_16_$rep.json 2>> $OUT/${TAG}.err
  MAGUS_LIB_PATH=$L18 MAGUS_TARGET_WARPS_PER_SM=18 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c2_18_$rep.json 2>> $OUT/${TAG}.err
done
timeout 300 python bench.py --config 4 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 --preroll-ms 300 > $OUT/${TAG}_c4_16.json 2>> $OUT/${TAG}.err
MAGUS_LIB_PATH=$L18 MAGUS_TARGET_WARPS_PER_SM=18 timeout 300 python bench.py --config 4 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 --preroll-ms 300 > $OUT/${TAG}_c4_18.json 2>> $OUT/${TAG}.err
for f in $OUT/${TAG}_c*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['segmentation']['n_segments'], d['segmentation']['mismatched_segments'], d['clocks']['sm_mhz'])"; done
