#!/bin/bash
# one full ncu capture of the kernel matching $2 (default: any replay kernel) in the default bench config
TAG=${1:-prof}
KRE=${2:-magus_replay}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
    -o gpurun_out/${TAG} python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
