#!/bin/bash
# GPU tests + fix-up A/B, then one ncu capture of the chain-walk kernel on config 5
TAG=${1:-walk}
bash scripts/fix_ab.sh $TAG
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_fix_pair_walk -s 2 -c 1 \
    -o gpurun_out/${TAG}_walk python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > gpurun_out/${TAG}_walk_ncu.log 2>&1
echo "ncu rc=$?"
