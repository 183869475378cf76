#!/bin/bash
# GPU suite after the open-loop TDP fix; walk A/B (lookahead vs plain one-chain block) on cfg 3 / 5;
# cfg 3 launch list (per-kernel device time of one step).  usage: bash scripts/r02_s2.sh TAG
TAG=${1:-r02s2}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
WF=paper_2502_03796_b200/lib/libmagus_replay_wf.so
for rep in 1 2; do
  for c in 3 5; do
    timeout 600 python scripts/probe_cfg.py $c 0 > $OUT/${TAG}_cfg${c}_la_$rep.txt 2>&1
    MAGUS_LIB_PATH=$WF timeout 600 python scripts/probe_cfg.py $c 0 > $OUT/${TAG}_cfg${c}_wf_$rep.txt 2>&1
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none -c 60 --csv \
  --log-file $OUT/${TAG}_cfg3_launches.csv python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
for f in $OUT/${TAG}_cfg*.txt; do echo "$f: $(cut -c1-200 $f)"; done > $OUT/${TAG}_summary.txt
tail -3 $OUT/${TAG}_pytest_gpu.log >> $OUT/${TAG}_summary.txt
cat $OUT/${TAG}_summary.txt
