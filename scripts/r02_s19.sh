#!/bin/bash
# cfg 5 A/B: lean TDP stage block (default) vs the round-1 block (MAGUS_TDP_LEAN=0 build), interleaved
TAG=${1:-r02s19}
OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2 3; do
  MAGUS_WARMUP_EXTRA=64 timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_lean_$rep.txt 2>&1
  MAGUS_LIB_PATH=paper_2502_03796_b200/lib/libmagus_replay_tdp0.so MAGUS_WARMUP_EXTRA=64 timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_old_$rep.txt 2>&1
done
for f in $OUT/${TAG}_*.txt; do echo "$f: $(cut -c1-140 $f)"; done
