#!/bin/bash
# TDP never-low closed form: full GPU suite; cfg 5 probe (closed vs replayed 270 W) and bench; cfg 2 bench
TAG=${1:-r02s13}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for rep in 1 2; do
  for nc in 0 1; do
    MAGUS_NO_TDP_CLOSED=$nc MAGUS_WARMUP_EXTRA=64 timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_cfg5_noclosed${nc}_$rep.txt 2>&1
  done
done
timeout 600 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 > $OUT/${TAG}_bench5.json 2> $OUT/${TAG}_bench5.err
timeout 600 python bench.py > $OUT/${TAG}_bench2.json 2> $OUT/${TAG}_bench2.err
tail -2 $OUT/${TAG}_pytest_gpu.log; for f in $OUT/${TAG}_cfg5_*.txt; do echo "$f: $(cut -c1-190 $f)"; done
for f in $OUT/${TAG}_bench*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['roofline']['replay_ms'], d['roofline']['frac'], d['clocks'], d['segmentation']['warmup_ticks'], d['config'].get('replayed_policies'))"; done
