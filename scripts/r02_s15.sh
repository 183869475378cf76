#!/bin/bash
# wide kernel with the per-warp fp64 scratch: wide / randomized / full-size tests, cfg 3 probes, launch list
TAG=${1:-r02s15}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 120 -k "wide or randomized or full_size_every_trace or sweep" > $OUT/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest.log
for rep in 1 2; do timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_cfg3_$rep.txt 2>&1; done
timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 10 > $OUT/${TAG}_bench3.json 2> $OUT/${TAG}_bench3.err
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c 8 --csv \
  --log-file $OUT/${TAG}_cfg3_launches.csv python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
tail -2 $OUT/${TAG}_pytest.log; cut -c1-200 $OUT/${TAG}_cfg3_*.txt; python -c "import json; d=json.load(open('$OUT/${TAG}_bench3.json')); print(d['ms_per_step'], d['roofline']['replay_ms'], d['clocks'])"
