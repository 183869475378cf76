#!/bin/bash
# combined MAGUS + TDP kernel (cfg 5): full GPU suite, cfg 5 probes combo vs two launches, bench lines, DRAM bytes
TAG=${1:-r02s10}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for rep in 1 2; do
  for cb in 1 0; do
    MAGUS_COMBO=$cb MAGUS_WARMUP_EXTRA=64 timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_cfg5_combo${cb}_$rep.txt 2>&1
  done
done
timeout 600 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 > $OUT/${TAG}_bench5.json 2> $OUT/${TAG}_bench5.err
MAGUS_COMBO=0 timeout 600 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 > $OUT/${TAG}_bench5_nocombo.json 2> $OUT/${TAG}_bench5b.err
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c 40 --csv \
  --log-file $OUT/${TAG}_cfg5_launches.csv python bench.py --config 5 --steps 2 --warmup 4 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
tail -3 $OUT/${TAG}_pytest_gpu.log; for f in $OUT/${TAG}_cfg5_combo*.txt; do echo "$f: $(cut -c1-180 $f)"; done
for f in $OUT/${TAG}_bench5*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['roofline']['replay_ms'], d['clocks'], d['segmentation']['warmup_ticks'], d['segmentation']['n_segments'])"; done
