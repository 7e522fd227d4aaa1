#!/bin/bash
# --set full captures of the fast leaf kernels (first leaf, round 0), c2 x64
O=gpurun_out/fast
mkdir -p $O
python tools/prof_run.py c2 64 > $O/plain.log 2>&1 || exit 1
for K in leaf_chain leaf_basis; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:$K -c 1 -o $O/$K python tools/prof_run.py c2 64 > $O/ncu_$K.log 2>&1
done
ls -la $O
