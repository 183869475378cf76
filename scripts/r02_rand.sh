#!/bin/bash
# randomized parity sweep with the batched tune-flag log as the default stage variant
TAG=${1:-r02rand}
OUT=gpurun_out; mkdir -p $OUT
MAGUS_RANDOM_SEEDS=${SEEDS:-400} timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "random" > $OUT/${TAG}.txt 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}.txt
tail -3 $OUT/${TAG}.txt
