#!/bin/bash
# batched tune-flag log (solo BAL 24/25) : GPU suite, interleaved A/B against the per-tick shift (BAL 20/21), a bench line
TAG=${1:-r02lb}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_gpu_tests.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c2_b25_$rep.json 2>> $OUT/${TAG}.err
  MAGUS_SOLO_BAL=20 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c2_b21_$rep.json 2>> $OUT/${TAG}.err
done
for f in $OUT/${TAG}_c2_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['roofline']['replay_ms_min'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done > $OUT/${TAG}_ab.txt
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2>> $OUT/${TAG}.err
cat $OUT/${TAG}_ab.txt; tail -3 $OUT/${TAG}_gpu_tests.txt
