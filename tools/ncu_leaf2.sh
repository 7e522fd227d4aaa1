#!/bin/bash
set -e
python tools/prof_run.py c2 64 > gpurun_out/plain_l2.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"leaf_(pivot3|build)_kernel" -c 2 -o gpurun_out/leaf_c2 python tools/prof_run.py c2 64 > gpurun_out/ncu_l2.log 2>&1
