#!/bin/bash
# L-stage (MAGUS_SOLO_BAL=20: level in the cmd word, lock = sign of the biased count, |d| flag test when symmetric):
# full GPU suite, then interleaved cfg2 / cfg5 / cfg4 A/B against variant 2.  usage: bash scripts/r02_l1.sh TAG
TAG=${1:-r02l1}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/${TAG}_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/${TAG}_pytest.log 2>&1 <<< ""
echo "rc=$?" >> $OUT/${TAG}_pytest.log
tail -3 $OUT/${TAG}_pytest.log
for rep in 1 2 3; do
  for v in 2 20; do
    MAGUS_SOLO_BAL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 \
        > $OUT/${TAG}_c2_v${v}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for rep in 1 2; do
  for v in 2 20; do
    MAGUS_SOLO_BAL=$v timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 20 --preroll-ms 300 \
        > $OUT/${TAG}_c5_v${v}_$rep.json 2>> $OUT/${TAG}.err
  done
done
for v in 2 20; do
  MAGUS_SOLO_BAL=$v timeout 600 python bench.py --config 4 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 --preroll-ms 300 \
      > $OUT/${TAG}_c4_v${v}.json 2>> $OUT/${TAG}.err
done
python - "$TAG" <<'PY' > $OUT/${TAG}_summary.txt
import json, sys, glob
tag = sys.argv[1]
for c in ("c2", "c5", "c4"):
    for v in (2, 20):
        ms = []
        for f in sorted(glob.glob(f"gpurun_out/{tag}_{c}_v{v}_*.json") + glob.glob(f"gpurun_out/{tag}_{c}_v{v}.json")):
            try:
                d = json.load(open(f))
                ms.append((round(d["roofline"]["replay_ms"], 4), round(d["ms_per_step"], 4), round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"]))
            except Exception as e:
                ms.append(("err", f, str(e)[:80]))
        print(c, "v", v, ms)
PY
cat $OUT/${TAG}_summary.txt
