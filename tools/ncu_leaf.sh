#!/bin/bash
# full ncu capture of one leaf launch + one big FFT launch of the c5 x 64 solve
set -e
python tools/prof_run.py c5 64 > gpurun_out/plain.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:leaf_kernel -c 1 -o gpurun_out/leaf_c5 python tools/prof_run.py c5 64 > gpurun_out/ncu_leaf.log 2>&1
