#!/bin/bash
# wide plan, 2 chains per thread (default) vs 1: tests, cfg 3 probes and bench line
TAG=${1:-r02s7}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "wide or full_size_every_trace" --durations=5 > $OUT/${TAG}_pytest_wide.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_wide.log
MAGUS_WIDE_NC=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "wide" > $OUT/${TAG}_pytest_wide_nc1.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_wide_nc1.log
for rep in 1 2; do
  timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_cfg3_nc2_$rep.txt 2>&1
  MAGUS_WIDE_NC=1 timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_cfg3_nc1_$rep.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c 8 --csv \
  --log-file $OUT/${TAG}_cfg3_launches.csv python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
tail -2 $OUT/${TAG}_pytest_wide.log $OUT/${TAG}_pytest_wide_nc1.log; for f in $OUT/${TAG}_cfg3_*.txt; do echo "$f: $(cut -c1-170 $f)"; done
