#!/bin/bash
# batched tune-flag log in the fused MAGUS + TDP kernel (config 5): GPU suite, interleaved A/B (MAGUS_SOLO_BAL=20 turns
# the batched log off in both kernels), config-5 and config-2 bench lines
TAG=${1:-r02lb5}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_gpu_tests.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c5_lb_$rep.json 2>> $OUT/${TAG}.err
  MAGUS_SOLO_BAL=20 timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_c5_nolb_$rep.json 2>> $OUT/${TAG}.err
done
for f in $OUT/${TAG}_c5_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['roofline']['replay_ms_min'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done > $OUT/${TAG}_ab.txt
timeout 600 python bench.py --config 5 > $OUT/${TAG}_bench_cfg5.json 2>> $OUT/${TAG}.err
timeout 600 python bench.py > $OUT/${TAG}_bench_cfg2.json 2>> $OUT/${TAG}.err
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
cat $OUT/${TAG}_ab.txt; tail -3 $OUT/${TAG}_gpu_tests.txt; tail -1 $OUT/${TAG}_smoke.txt
