#!/bin/bash
# GPU tests (default build) + the parity subset under a variant + interleaved bench A/B of variants (1 GPU).
# usage: bash scripts/r02_ab.sh TAG "VARIANT_ENV" "<name>=<ENV=V ...>" ...
TAG=$1; shift
VENV=$1; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider -x --durations=10 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
if [ -n "$VENV" ]; then
  env $VENV timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "small or full_size or tiny or window or saturating or cfg1" \
    > $OUT/${TAG}_pytest_variant.log 2>&1
  echo "variant pytest rc=$?" >> $OUT/${TAG}_pytest_variant.log
fi
for rep in 1 2 3; do
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
            d = json.load(open(f)); ms.append((round(d["roofline"]["replay_ms"], 4), round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"]))
        except Exception as e:
            ms.append(str(e))
    print(name, ms)
PY
cat $OUT/${TAG}_summary.txt
