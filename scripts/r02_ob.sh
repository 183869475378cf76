#!/bin/bash
# batched tune-flag log in the open-loop O stage (BAL 34/35): GPU suite + smoke, interleaved open-loop A/B against
# the per-tick shift (MAGUS_SOLO_BAL=20 -> BAL 30/31), an open-loop bench line
TAG=${1:-r02ob}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/${TAG}_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
for rep in 1 2 3; do
  timeout 300 python bench.py --open-loop --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_ol_b35_$rep.json 2>> $OUT/${TAG}.err
  MAGUS_SOLO_BAL=20 timeout 300 python bench.py --open-loop --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_ol_b31_$rep.json 2>> $OUT/${TAG}.err
done
for f in $OUT/${TAG}_ol_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['roofline']['replay_ms_min'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done > $OUT/${TAG}_ab.txt
timeout 600 python bench.py --open-loop > $OUT/${TAG}_bench_open_loop.json 2>> $OUT/${TAG}.err
cat $OUT/${TAG}_ab.txt; tail -3 $OUT/${TAG}_gpu_tests.txt; tail -1 $OUT/${TAG}_smoke.txt
