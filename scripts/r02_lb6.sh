#!/bin/bash
# GPU suite + smoke after the fused-kernel batched log; config-5 and config-2 bench lines
TAG=${1:-r02lb6}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/${TAG}_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
timeout 600 python bench.py --config 5 > $OUT/${TAG}_bench_cfg5.json 2>> $OUT/${TAG}.err
timeout 600 python bench.py > $OUT/${TAG}_bench_cfg2.json 2>> $OUT/${TAG}.err
tail -3 $OUT/${TAG}_gpu_tests.txt; tail -1 $OUT/${TAG}_smoke.txt
