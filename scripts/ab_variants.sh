#!/bin/bash
# GPU tests, then interleaved bench repeats of replay-kernel variants selected by env vars (1 GPU).
# usage: bash scripts/ab_variants.sh <tag> "<name>=<ENV=V ...>" ...
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for rep in 1 2 3 4; do
  for v in "$@"; do
    name=${v%%=*}; envs=${v#*=}
    env $envs timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 \
        > $OUT/${TAG}_${name}_$rep.json 2>> $OUT/${TAG}.err
  done
done
python - "$TAG" "$@" <<'PY' > $OUT/${TAG}_summary.txt
import json, sys, glob
tag = sys.argv[1]
for v in sys.argv[2:]:
    name = v.split("=")[0]
    ms = []
    for f in sorted(glob.glob(f"gpurun_out/{tag}_{name}_*.json")):
        try:
            d = json.load(open(f)); ms.append((d["roofline"]["replay_ms"], d["ms_per_step"], d["clocks"]["sm_mhz"]))
        except Exception as e:
            ms.append(str(e))
    print(name, ms)
PY
cat $OUT/${TAG}_summary.txt
