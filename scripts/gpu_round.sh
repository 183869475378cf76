#!/bin/bash
# Round-end evidence in one gpurun session: GPU tests, the default bench line, the ncu launch list of the
# same bench command, and one ncu --set full capture of the replay kernel.  Outputs under gpurun_out/<tag>_*.
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/${TAG}_smi.txt
(nproc; lscpu | grep "Model name") > $OUT/${TAG}_host.txt
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout 600 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay -s 3 -c 1 \
    -o $OUT/${TAG}_replay python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > $OUT/${TAG}_ncu_full.log 2>&1
echo done
