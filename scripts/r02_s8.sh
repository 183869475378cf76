#!/bin/bash
# cfg 2 A/B of the solo stage variants 2 (default) / 3 / 4 / 9 (interleaved, 3 reps); cfg 5 warm-up sweep
TAG=${1:-r02s8}
OUT=gpurun_out; mkdir -p $OUT
MAGUS_SOLO_BAL=9 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "small_configs or full_size_every_trace" > $OUT/${TAG}_pytest_v9.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest_v9.log
for rep in 1 2 3; do
  for v in 2 3 4 9; do
    MAGUS_SOLO_BAL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 \
        > $OUT/${TAG}_v${v}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for x in 32 64 96 128 160 224; do
  MAGUS_WARMUP_EXTRA=$x timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_cfg5_w$x.txt 2>&1
done
python - "$TAG" <<'PY' > $OUT/${TAG}_summary.txt
import json, sys, glob
tag = sys.argv[1]
for v in (2, 3, 4, 9):
    ms = []
    for f in sorted(glob.glob(f"gpurun_out/{tag}_v{v}_*.json")):
        try:
            d = json.load(open(f)); ms.append((round(d["roofline"]["replay_ms"], 4), round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"]))
        except Exception as e:
            ms.append(str(e)[:60])
    print("v", v, ms)
for f in sorted(glob.glob(f"gpurun_out/{tag}_cfg5_w*.txt")):
    print(f, open(f).read().strip()[:190])
PY
cat $OUT/${TAG}_summary.txt; tail -2 $OUT/${TAG}_pytest_v9.log
