#!/bin/bash
# Parity subset under each variant, then interleaved bench A/B (1 GPU).
# usage: bash scripts/r02_ab2.sh TAG "<name>=<ENV=V ...>" ...
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider -x --durations=10 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for v in "$@"; do
  name=${v%%=*}; envs=${v#*=}
  env $envs timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x \
    -k "small or full_size_every_trace or tiny or window or saturating or cfg1 or handwritten or open_loop or repeated" \
    > $OUT/${TAG}_pytest_$name.log 2>&1
  echo "pytest $name rc=$?" >> $OUT/${TAG}_pytest_$name.log
done
for rep in 1 2 3; do
  for v in "$@"; do
    name=${v%%=*}; envs=${v#*=}
    env $envs timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 \
        > $OUT/${TAG}_${name}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for c in 5; do
  for v in "$@"; do
    name=${v%%=*}; envs=${v#*=}
    env $envs timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 --preroll-ms 300 \
        > $OUT/${TAG}_${name}_cfg$c.json 2>> $OUT/${TAG}.err
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
            d = json.load(open(f)); ms.append((f.split("_")[-1][:-5], round(d["roofline"]["replay_ms"], 4), round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"], d["segmentation"]["mismatched_segments"]))
        except Exception as e:
            ms.append(str(e))
    print(name, ms)
    print("   ", open(f"gpurun_out/{tag}_pytest_{name}.log").read().strip().splitlines()[-2:])
PY
cat $OUT/${TAG}_summary.txt
