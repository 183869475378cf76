#!/bin/bash
# Round-2 re-entry session: GPU suite on HEAD, default cfg2 bench, cfg3/cfg5 probes, cfg2 A/B of the solo
# stage variants (MAGUS_SOLO_BAL) interleaved, TDP solo variants on cfg5.  usage: bash scripts/r02_s1.sh TAG
TAG=${1:-r02s1}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/${TAG}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
timeout 600 python bench.py > $OUT/${TAG}_bench2.json 2> $OUT/${TAG}_bench2.err
for rep in 1 2; do
  for v in 2 5 10 11 12 13 14 15 16 17; do
    MAGUS_SOLO_BAL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 \
        > $OUT/${TAG}_v${v}_$rep.json 2>> $OUT/${TAG}_ab.err
  done
done
for c in 3 5; do
  timeout 600 python scripts/probe_cfg.py $c 0 > $OUT/${TAG}_probe$c.txt 2>&1
done
for t in 0 1 2; do
  MAGUS_TDP_SOLO=$t timeout 600 python scripts/probe_cfg.py 5 0 > $OUT/${TAG}_cfg5_tdp$t.txt 2>&1
done
python - "$TAG" <<'PY' > $OUT/${TAG}_summary.txt
import json, sys, glob
tag = sys.argv[1]
for v in (2, 5, 10, 11, 12, 13, 14, 15, 16, 17):
    ms = []
    for f in sorted(glob.glob(f"gpurun_out/{tag}_v{v}_*.json")):
        try:
            d = json.load(open(f)); ms.append((round(d["roofline"]["replay_ms"], 4), round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"]))
        except Exception as e:
            ms.append(str(e)[:60])
    print("v", v, ms)
for f in sorted(glob.glob(f"gpurun_out/{tag}_probe*.txt") + glob.glob(f"gpurun_out/{tag}_cfg5_tdp*.txt")):
    print(f, open(f).read().strip()[:300])
PY
cat $OUT/${TAG}_summary.txt
tail -3 $OUT/${TAG}_pytest_gpu.log
