#!/bin/bash
# config 3: executed instructions and DRAM bytes of every wide-kernel launch of one run (kernels serialised by ncu),
# for profiles/ncu_wide_summary.json (bench.py's alu roofline numerator)
TAG=${1:-r02wi}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:magus_replay_wide -s 4 -c 4 --csv --log-file $OUT/${TAG}_cfg3_wide_launches.csv \
    python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
echo "ncu rc=$?"; python scripts/launch_summary.py $OUT/${TAG}_cfg3_wide_launches.csv
