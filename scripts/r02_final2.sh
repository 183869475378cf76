#!/bin/bash
# round-2 closing evidence: full GPU suite, default bench lines (config 2 with e2e and the CPU baseline, configs 3-5,
# config 2 open loop), all on one box
TAG=${1:-r02fin2}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/${TAG}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=5 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log; tail -2 $OUT/${TAG}_pytest_gpu.log
timeout 900 python bench.py > $OUT/${TAG}_bench_cfg2.json 2> $OUT/${TAG}_bench.err
for c in 3 4 5; do timeout 900 python bench.py --config $c > $OUT/${TAG}_bench_cfg$c.json 2>> $OUT/${TAG}_bench.err; done
timeout 600 python bench.py --open-loop --no-e2e > $OUT/${TAG}_bench_cfg2_open_loop.json 2>> $OUT/${TAG}_bench.err
for f in $OUT/${TAG}_bench_*.json; do python -c "import json; d=json.load(open('$f')); r=d['roofline']; print('$f', d['value'], r.get('replay_ms'), d['ms_per_step'], round(r.get('frac') or 0, 3), r.get('bound'), (d.get('e2e') or {}).get('value'), d['clocks'])"; done
