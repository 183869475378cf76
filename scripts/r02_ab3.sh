#!/bin/bash
# cfg2 A/B of the solo stage variants; cfg3 / cfg5 step vs the speculative warm-up length (1 GPU)
TAG=${1:-r02ab3}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "small or full_size_every_trace or tiny or window or cfg1" \
    > $OUT/${TAG}_pytest_v5.log 2>&1 <<< "" ; echo "rc=$?" >> $OUT/${TAG}_pytest_v5.log
for rep in 1 2 3; do
  for v in 2 5; do
    MAGUS_SOLO_BAL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 \
        > $OUT/${TAG}_v${v}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for x in 0 96 224 480; do
  MAGUS_WARMUP_EXTRA=$x timeout 600 python scripts/probe_cfg.py 3 0 > $OUT/${TAG}_cfg3_w$x.txt 2>&1
done
for x in 0 96 224; do
  MAGUS_WARMUP_EXTRA=$x timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_cfg5_w$x.txt 2>&1
done
python - "$TAG" <<'PY' > $OUT/${TAG}_summary.txt
import json, sys, glob
tag = sys.argv[1]
for v in (2, 5):
    ms = []
    for f in sorted(glob.glob(f"gpurun_out/{tag}_v{v}_*.json")):
        d = json.load(open(f)); ms.append((round(d["roofline"]["replay_ms"], 4), round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"]))
    print("v", v, ms)
for f in sorted(glob.glob(f"gpurun_out/{tag}_cfg*_w*.txt")):
    print(f, open(f).read().strip()[:200])
PY
cat $OUT/${TAG}_summary.txt
