#!/bin/bash
# round evidence of the L-stage kernels (outputs kept under 64 MiB: ncu reports exported to CSV on the box):
# default bench lines, ncu launch list, ncu --set full of the solo replay kernel (cfg 2) and the wide kernel (cfg 3)
TAG=${1:-r02l3}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/${TAG}_smi.txt
(nproc; lscpu | grep "Model name") > $OUT/${TAG}_host.txt
for rep in 1 2; do
  timeout 900 python bench.py > $OUT/${TAG}_bench_$rep.json 2> $OUT/${TAG}_bench.err
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --preroll-ms 300 > $OUT/${TAG}_ab_$rep.json 2>> $OUT/${TAG}.err
done
cp $OUT/${TAG}_bench_2.json $OUT/${TAG}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay -s 3 -c 1 \
    -o $OUT/${TAG}_replay python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > $OUT/${TAG}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay_wide -s 4 -c 1 \
    -o $OUT/${TAG}_wide python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > $OUT/${TAG}_ncu_wide.log 2>&1
for r in replay wide; do
  ncu -i $OUT/${TAG}_$r.ncu-rep --page raw --csv > $OUT/${TAG}_${r}_raw.csv 2>/dev/null
  ncu -i $OUT/${TAG}_$r.ncu-rep --page source --csv > $OUT/${TAG}_${r}_source.csv 2>/dev/null
  gzip -f $OUT/${TAG}_${r}_source.csv
done
ls -la $OUT/${TAG}_* | awk '{print $5, $9}'
rm -f $OUT/${TAG}_wide.ncu-rep $OUT/${TAG}_replay.ncu-rep
du -sh $OUT
for f in $OUT/${TAG}_bench_*.json $OUT/${TAG}_ab_*.json; do
  python -c "import json,sys; d=json.load(open('$f')); print('$f', d['roofline']['replay_ms'], d['ms_per_step'], round(d['roofline']['frac'],3), d['clocks'])"
done
