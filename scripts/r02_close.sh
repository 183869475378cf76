#!/bin/bash
# closing check of the committed tree: GPU suite, smoke, default bench line
TAG=${1:-r02close}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/${TAG}_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2>> $OUT/${TAG}.err
tail -2 $OUT/${TAG}_gpu_tests.txt; tail -1 $OUT/${TAG}_smoke.txt
python -c "import json; d=json.load(open('$OUT/${TAG}_bench.json')); r=d['roofline']; print(d['ms_per_step'], r['frac'], r['replay_ms'], d['clocks'])"
