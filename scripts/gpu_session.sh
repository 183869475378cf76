#!/bin/bash
# One gpurun session: GPU tests, bench, ncu launch list and one full ncu capture of the replay kernel.
# usage (under gpurun): bash scripts/gpu_session.sh <tag> [tests|notests]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/${TAG}_smi.txt
nproc > $OUT/${TAG}_nproc.txt; lscpu | grep "Model name" >> $OUT/${TAG}_nproc.txt
if [ "${2:-tests}" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/${TAG}_pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
fi
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > $OUT/${TAG}_ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay -s 3 -c 1 \
    -o $OUT/${TAG}_replay python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > $OUT/${TAG}_ncu_full.log 2>&1
echo done
