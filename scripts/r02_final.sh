#!/bin/bash
# round-2 final evidence: default bench lines (config 2 twice, configs 3-5, reference arm), the config-2 ncu launch
# list, ncu --set full of the config-2 solo kernel, the config-3 wide kernel (P stage) and the config-5 fused kernel
# (reports exported to CSV on the box; the .ncu-rep files are deleted to stay under gpurun's 64 MiB)
TAG=${1:-r02fin}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version,power.limit --format=csv > $OUT/${TAG}_smi.txt
(nproc; lscpu | grep "Model name") > $OUT/${TAG}_host.txt
timeout 900 python bench.py > $OUT/${TAG}_bench_1.json 2> $OUT/${TAG}_bench.err
for c in 3 4 5; do timeout 900 python bench.py --config $c > $OUT/${TAG}_bench_cfg$c.json 2>> $OUT/${TAG}_bench.err; done
timeout 900 python bench.py > $OUT/${TAG}_bench_2.json 2>> $OUT/${TAG}_bench.err
timeout 900 python bench.py --impl reference > $OUT/${TAG}_bench_reference.json 2>> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay_solo -s 3 -c 1 \
    -o $OUT/${TAG}_replay python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > $OUT/${TAG}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay_wide -s 4 -c 1 \
    -o $OUT/${TAG}_wide python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > $OUT/${TAG}_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay_fused -s 3 -c 1 \
    -o $OUT/${TAG}_fused python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > $OUT/${TAG}_ncu3.log 2>&1
for r in replay wide fused; do
  ncu -i $OUT/${TAG}_$r.ncu-rep --page raw --csv > $OUT/${TAG}_${r}_raw.csv 2>/dev/null
  ncu -i $OUT/${TAG}_$r.ncu-rep --page source --csv > $OUT/${TAG}_${r}_source.csv 2>/dev/null
  gzip -f $OUT/${TAG}_${r}_source.csv
  rm -f $OUT/${TAG}_$r.ncu-rep
done
du -sh $OUT
for f in $OUT/${TAG}_bench_*.json; do python -c "import json; d=json.load(open('$f')); r=d.get('roofline',{}); print('$f', d.get('impl','ours'), d['value'], r.get('replay_ms'), d['ms_per_step'], r.get('frac'), d.get('clocks'))" 2>&1 | tail -1; done
