#!/bin/bash
# round-2 baseline on a fresh box: bench lines of configs 2/3/5, phase split, and per-kernel instruction
# counts of one config-3 step (the ALU roofline inputs).  usage (under gpurun): bash scripts/r02_baseline.sh TAG
TAG=${1:-r02base}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/${TAG}_smi.txt
nproc > $OUT/${TAG}_nproc.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench2.json 2> $OUT/${TAG}_bench2.err
for c in 3 5; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > $OUT/${TAG}_bench$c.json 2> $OUT/${TAG}_bench$c.err
done
timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_probe3.txt 2>&1
timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_probe5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum \
  --clock-control none -c 40 --csv --log-file $OUT/${TAG}_cfg3_inst.csv \
  python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > $OUT/${TAG}_cfg3_ncu.log 2>&1
echo done
