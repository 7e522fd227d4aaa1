#!/bin/bash
# FFT launch list (durations) of one solve: tools/ncu_fft_list.sh <cfg> <count> <out>
CFG=$1; CNT=$2; OUT=$3
mkdir -p gpurun_out/fl
python tools/prof_run.py $CFG $CNT > gpurun_out/fl/plain_$OUT.log 2>&1 || exit 1
timeout 1200 ncu --profile-from-start off -k regex:fft --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/fl/$OUT.csv python tools/prof_run.py $CFG $CNT > gpurun_out/fl/ncu_$OUT.log 2>&1
