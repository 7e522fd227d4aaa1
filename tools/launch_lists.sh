#!/bin/bash
# ncu launch lists (timed region only) of the c2 and c5 bench commands -> gpurun_out/$R/
R=${R:-r1}
O=gpurun_out/$R
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --config c5 --batch 256 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c5.log 2>&1
ls -la $O
