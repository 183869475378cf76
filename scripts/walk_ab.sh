#!/bin/bash
# GPU tests, then configs 4 and 5 with the 1- and 2-traces-per-lane lockstep walk
TAG=${1:-wab}
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for c in 5 4; do
  for v in 1 0; do
    MAGUS_WALK_2T=$v timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 \
        > $OUT/${TAG}_cfg${c}_2t$v.json 2>> $OUT/${TAG}.err
  done
done
python - $TAG <<'PY' > $OUT/${TAG}_summary.txt
import json, sys, glob
for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}_cfg*_2t*.json")):
    d = json.load(open(f)); sg = d["segmentation"]
    print(f.split("/")[-1], "step %.3f replay %.3f" % (d["ms_per_step"], d["roofline"]["replay_ms"]), "mism", sg["mismatched_segments"])
PY
cat $OUT/${TAG}_summary.txt
