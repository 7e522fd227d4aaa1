#!/bin/bash
# per-launch time + DRAM bytes for one solve of a config (ncu), plain run first
set -e
CFG=$1; CNT=$2; OUT=$3
python tools/prof_run.py $CFG $CNT > gpurun_out/plain_$OUT.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none --csv --log-file gpurun_out/$OUT.csv python tools/prof_run.py $CFG $CNT > gpurun_out/ncu_$OUT.log 2>&1
