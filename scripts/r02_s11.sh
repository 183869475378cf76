#!/bin/bash
# after the solo refactor: full GPU suite, cfg 2 A/B (exact warm-up vs synthetic warm-up state), torchrun NCCL smoke,
# compute-sanitizer over every kernel family (incl. the wide and combined kernels)
TAG=${1:-r02s11}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for rep in 1 2 3; do
  for sy in 0 1; do
    MAGUS_SOLO_SYNTH=$sy timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_synth${sy}_$rep.json 2>> $OUT/${TAG}.err
  done
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --nccl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${TAG}_torchrun_nccl.json 2> $OUT/${TAG}_torchrun_nccl.err
echo "torchrun rc=$?" >> $OUT/${TAG}_torchrun_nccl.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_run.py > $OUT/${TAG}_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/${TAG}_sanitize_$tool.log
done
tail -2 $OUT/${TAG}_pytest_gpu.log; tail -1 $OUT/${TAG}_torchrun_nccl.err; cut -c1-300 $OUT/${TAG}_torchrun_nccl.json; tail -2 $OUT/${TAG}_sanitize_*.log
for f in $OUT/${TAG}_synth*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['roofline']['replay_ms'],4), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['segmentation']['mismatched_segments'])"; done
