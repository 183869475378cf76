#!/bin/bash
# wide L stage (cfg 3) A/B + round evidence of the L-stage solo kernel: GPU suite, default bench line, ncu launch
# list and one ncu --set full capture of the replay kernel.  usage: bash scripts/r02_l2.sh TAG
TAG=${1:-r02l2}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/${TAG}_smi.txt
(nproc; lscpu | grep "Model name") > $OUT/${TAG}_host.txt
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout 600 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
tail -2 $OUT/${TAG}_pytest_gpu.log
for rep in 1 2; do
  for l in 0 1; do
    MAGUS_WIDE_L=$l timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 --preroll-ms 300 \
        > $OUT/${TAG}_c3_l${l}_$rep.json 2>> $OUT/${TAG}.err
  done
done
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay -s 3 -c 1 \
    -o $OUT/${TAG}_replay python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > $OUT/${TAG}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay_wide -s 4 -c 1 \
    -o $OUT/${TAG}_wide python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > $OUT/${TAG}_ncu_wide.log 2>&1
python - "$TAG" <<'PY' > $OUT/${TAG}_summary.txt
import json, sys, glob
tag = sys.argv[1]
for l in (0, 1):
    ms = []
    for f in sorted(glob.glob(f"gpurun_out/{tag}_c3_l{l}_*.json")):
        try:
            d = json.load(open(f))
            ms.append((round(d["roofline"]["replay_ms"], 4), round(d["ms_per_step"], 4), round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"]))
        except Exception as e:
            ms.append(("err", f, str(e)[:80]))
    print("c3 wide_L", l, ms)
d = json.load(open(f"gpurun_out/{tag}_bench.json"))
print("c2 bench", d["roofline"]["replay_ms"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"])
PY
cat $OUT/${TAG}_summary.txt
