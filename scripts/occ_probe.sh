#!/bin/bash
# replay-kernel time vs resident one-warp CTAs per SM (dynamic smem padding), 1 GPU
TAG=${1:-occ}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
for pad in 0 2000 6000 10000 0; do
  MAGUS_SOLO_SMEM_PAD=$pad timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $OUT/${TAG}_pad$pad.json 2>> $OUT/${TAG}.err
done
MAGUS_SOLO=0 timeout 300 python bench.py --no-e2e --no-cpu-baseline > $OUT/${TAG}_nosolo.json 2>> $OUT/${TAG}.err
echo done
