#!/bin/bash
# GPU tests, then the bench of configs 2-5 with MAGUS_WALK_SPLIT=1 / 0 (split vs lockstep chain walk; the
# worklist-rounds fix-up it compared against was removed after the A/B in profiles/r01_fixup_walk_ab.txt).
TAG=${1:-fix}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for c in 5 3 4 2; do
  for v in 1 0; do  # MAGUS_FIX_WALK
    MAGUS_WALK_SPLIT=$v timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 \
        > $OUT/${TAG}_cfg${c}_walk$v.json 2>> $OUT/${TAG}.err
  done
done
python - $TAG <<'PY' > $OUT/${TAG}_summary.txt
import json, sys, glob
for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}_cfg*_walk*.json")):
    try:
        d = json.load(open(f)); sg = d["segmentation"]
        print(f.split("/")[-1], "step %.3f replay %.3f" % (d["ms_per_step"], d["roofline"]["replay_ms"]),
              "segs", sg["n_segments"], "mism", sg["mismatched_segments"], "rounds", sg["fixup_rounds"],
              "mhz", d["clocks"]["sm_mhz"])
    except Exception as e:
        print(f, "ERR", e)
PY
cat $OUT/${TAG}_summary.txt
