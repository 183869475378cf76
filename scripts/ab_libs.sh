#!/bin/bash
# A/B of library builds on one config: alternates the variants R times; one line per run (replay ms, step ms).
# usage: bash scripts/ab_libs.sh <config> <rounds> lib1.so lib2.so ...
CFG=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for lib in "$@"; do
    echo -n "$(basename $lib) "
    MAGUS_LIB_PATH=$PWD/$lib timeout 120 python scripts/probe_cfg.py $CFG 0 2>&1 | grep -o "ms=[0-9.]* ms_notiming=[0-9.]*.*replay_ms=[0-9.]*" | sed 's/mism.*replay_ms/replay_ms/'
  done
done
