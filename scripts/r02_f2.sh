#!/bin/bash
# ncu --set full of the fused MAGUS + TDP kernel (config 5) and the cfg5 launch list; reports exported to CSV on the box
TAG=${1:-r02f2}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file $OUT/${TAG}_c5_launches.csv python bench.py --config 5 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:magus_replay_fused -s 3 -c 1 \
    -o $OUT/${TAG}_fused python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --preroll-ms 0 \
    > $OUT/${TAG}_ncu_fused.log 2>&1
ncu -i $OUT/${TAG}_fused.ncu-rep --page raw --csv > $OUT/${TAG}_fused_raw.csv 2>/dev/null
ncu -i $OUT/${TAG}_fused.ncu-rep --page source --csv > $OUT/${TAG}_fused_source.csv 2>/dev/null
gzip -f $OUT/${TAG}_fused_source.csv
rm -f $OUT/${TAG}_fused.ncu-rep
python scripts/launch_summary.py $OUT/${TAG}_c5_launches.csv
