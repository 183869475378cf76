#!/bin/bash
# GPU tests, the bench's distributed branch at N = 1, and compute-sanitizer over every kernel family.
# usage (under gpurun): bash scripts/r02_tests.sh TAG [tests|notests] [sanitize|nosanitize]
TAG=${1:-r02t}
OUT=gpurun_out; mkdir -p $OUT
if [ "${2:-tests}" = "tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider -x --durations=15 > $OUT/${TAG}_pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
fi
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --nccl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${TAG}_torchrun_nccl.json 2> $OUT/${TAG}_torchrun_nccl.err
echo "torchrun rc=$?" >> $OUT/${TAG}_torchrun_nccl.err
if [ "${3:-sanitize}" = "sanitize" ]; then
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python scripts/sanitize_run.py > $OUT/${TAG}_sanitize_$tool.log 2>&1
    echo "$tool rc=$?" >> $OUT/${TAG}_sanitize_$tool.log
  done
fi
echo done
