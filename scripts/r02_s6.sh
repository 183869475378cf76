#!/bin/bash
# cfg 3 wide plan: run without timing events under PDL / no PDL / no graph; ncu --set full of one wide kernel
TAG=${1:-r02s6}
OUT=gpurun_out; mkdir -p $OUT
for e in "" "MAGUS_NO_PDL=1" "MAGUS_NO_GRAPH=1"; do
  env $e timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_cfg3_${e%%=*}.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay_wide -s 4 -c 1 \
    -o $OUT/${TAG}_wide python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > $OUT/${TAG}_ncu.log 2>&1
for f in $OUT/${TAG}_cfg3_*.txt; do echo "$f: $(cut -c1-160 $f)"; done
