#!/bin/bash
# the unsegmented wide plan: its GPU parity tests, the full-size cfg 3 test, cfg 3 probe + bench line, launch list
TAG=${1:-r02s4}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "wide or full_size_every_trace" --durations=8 > $OUT/${TAG}_pytest_wide.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_wide.log
timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_cfg3_wide.txt 2>&1
MAGUS_WIDE=0 timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_cfg3_seg.txt 2>&1
timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > $OUT/${TAG}_bench3.json 2> $OUT/${TAG}_bench3.err
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 30 --csv \
  --log-file $OUT/${TAG}_cfg3_launches.csv python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
tail -3 $OUT/${TAG}_pytest_wide.log; cut -c1-300 $OUT/${TAG}_cfg3_*.txt; cut -c1-400 $OUT/${TAG}_bench3.json
