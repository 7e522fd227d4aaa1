#!/bin/bash
# --set full captures of the three leaf kernels (first leaf, round 0) for c2 x64
O=gpurun_out/r1
mkdir -p $O
python tools/prof_run.py c2 64 > $O/plain_leaf.log 2>&1 || exit 1
for K in leaf_build_row leaf_pivot_relay leaf_check; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:$K -c 1 -o $O/full_c2_$K python tools/prof_run.py c2 64 > $O/ncu_full_$K.log 2>&1
done
ls -la $O
