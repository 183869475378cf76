#!/bin/bash
# round-2 evidence after the L stage / fused / wide-P kernels: full GPU suite, compute-sanitizer over every kernel
# family, torchrun one-rank NCCL bench smoke, bench lines of configs 2-5
TAG=${1:-r02e1}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=5 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
tail -3 $OUT/${TAG}_pytest_gpu.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_run.py > $OUT/${TAG}_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/${TAG}_sanitize_$tool.log
  tail -2 $OUT/${TAG}_sanitize_$tool.log
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --nccl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${TAG}_torchrun_nccl.json 2> $OUT/${TAG}_torchrun_nccl.err
echo "torchrun rc=$?" >> $OUT/${TAG}_torchrun_nccl.err
for c in 3 4 5; do
  timeout 900 python bench.py --config $c > $OUT/${TAG}_bench_cfg$c.json 2>> $OUT/${TAG}_bench.err
done
timeout 900 python bench.py > $OUT/${TAG}_bench_cfg2.json 2>> $OUT/${TAG}_bench.err
for f in $OUT/${TAG}_bench_cfg*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline']['bound'], d['clocks'])"; done
