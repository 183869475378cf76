#!/bin/bash
# one full ncu capture of the replay kernel (bench config), 1 GPU
TAG=${1:-prof}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay -s 3 -c 1 \
    -o gpurun_out/${TAG} python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
