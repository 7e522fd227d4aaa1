#!/bin/bash
set -e
python tools/prof_run.py c2 64 > gpurun_out/plain_l3.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"leaf_build_row_kernel" -c 1 -o gpurun_out/brow_c2 python tools/prof_run.py c2 64 > gpurun_out/ncu_l3.log 2>&1
