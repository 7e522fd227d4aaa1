#!/bin/bash
set -e
python tools/prof_run.py c2 64 > gpurun_out/plain_fft.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"fft_fast_kernel" -s 40 -c 4 -o gpurun_out/fft_c2 python tools/prof_run.py c2 64 > gpurun_out/ncu_fft.log 2>&1
