#!/bin/bash
set -e
python tools/prof_run.py c5 64 > gpurun_out/plain_f2.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:fft_fast_kernel --launch-skip 300 -c 6 -o gpurun_out/fft_c5 python tools/prof_run.py c5 64 > gpurun_out/ncu_f2.log 2>&1
