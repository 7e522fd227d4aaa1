#!/bin/bash
# usage: tools/ncu_kernel.sh <kernel-regex> <out-name> [prof_run args]
set -e
K=$1; OUT=$2; shift 2
python tools/prof_run.py "$@" > gpurun_out/plain_$OUT.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:$K -c 1 -o gpurun_out/$OUT python tools/prof_run.py "$@" > gpurun_out/ncu_$OUT.log 2>&1
