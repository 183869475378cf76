#!/bin/bash
# full GPU suite (wide plan + adaptive warm-up); cfg 5 / cfg 2 / cfg 4 probes and bench lines
TAG=${1:-r02s9}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for c in 5 2; do timeout 600 python scripts/probe_cfg.py $c 0 > $OUT/${TAG}_probe$c.txt 2>&1; done
timeout 600 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 > $OUT/${TAG}_bench5.json 2> $OUT/${TAG}_bench5.err
timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 10 > $OUT/${TAG}_bench3.json 2> $OUT/${TAG}_bench3.err
timeout 900 python bench.py --config 4 --no-e2e --no-cpu-baseline --steps 5 > $OUT/${TAG}_bench4.json 2> $OUT/${TAG}_bench4.err
tail -3 $OUT/${TAG}_pytest_gpu.log; cut -c1-220 $OUT/${TAG}_probe*.txt; for c in 5 3 4; do cut -c1-900 $OUT/${TAG}_bench$c.json; done
