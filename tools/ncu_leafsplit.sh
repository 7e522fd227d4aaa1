#!/bin/bash
set -e
python tools/prof_run.py c5 64 > gpurun_out/plain_ls.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"leaf_(pivot|build|check)_kernel" -c 3 -o gpurun_out/leafsplit python tools/prof_run.py c5 64 > gpurun_out/ncu_ls.log 2>&1
