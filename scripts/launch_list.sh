#!/bin/bash
# per-launch device time of every kernel in a few bench steps (cold-cache, serialised: compare shares)
TAG=${1:-ll}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv
