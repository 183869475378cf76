#!/bin/bash
# batched tune-flag log in the wide P stage (LV 6): GPU suite, interleaved config-3 A/B against LV 4 (MAGUS_SOLO_BAL=20)
TAG=${1:-r02wb}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/${TAG}_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_gpu_tests.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 10 --preroll-ms 300 > $OUT/${TAG}_c3_lv6_$rep.json 2>> $OUT/${TAG}.err
  MAGUS_SOLO_BAL=20 timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 10 --preroll-ms 300 > $OUT/${TAG}_c3_lv4_$rep.json 2>> $OUT/${TAG}.err
done
for f in $OUT/${TAG}_c3_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done > $OUT/${TAG}_ab.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
cat $OUT/${TAG}_ab.txt; tail -3 $OUT/${TAG}_gpu_tests.txt; tail -1 $OUT/${TAG}_smoke.txt
