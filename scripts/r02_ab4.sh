#!/bin/bash
# GPU suite (default build: lookahead walk, TDP solo NP=2) + walk A/B (lookahead vs the plain one-chain block,
# MAGUS_LIB_PATH variant build) on configs 3 / 5 / 4-shard + TDP solo variants on config 5 (1 GPU)
TAG=${1:-r02ab4}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=8 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
WF=paper_2502_03796_b200/lib/libmagus_replay_wf.so
for c in 3 5; do
  timeout 600 python scripts/probe_cfg.py $c 0 > $OUT/${TAG}_cfg${c}_la.txt 2>&1
  MAGUS_LIB_PATH=$WF timeout 600 python scripts/probe_cfg.py $c 0 > $OUT/${TAG}_cfg${c}_wf.txt 2>&1
done
for t in 0 1 2; do
  MAGUS_TDP_SOLO=$t timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_cfg5_tdp$t.txt 2>&1
done
MAGUS_SOLO_SYNTH=1 timeout 900 python scripts/probe_cfg.py 4 0 > $OUT/${TAG}_cfg4synth_la.txt 2>&1
MAGUS_SOLO_SYNTH=1 MAGUS_LIB_PATH=$WF timeout 900 python scripts/probe_cfg.py 4 0 > $OUT/${TAG}_cfg4synth_wf.txt 2>&1
for f in $OUT/${TAG}_cfg*.txt; do echo "$f: $(cut -c1-230 $f)"; done > $OUT/${TAG}_summary.txt
cat $OUT/${TAG}_summary.txt
