#!/bin/bash
# --set full of the leaf kernels at round 0 of the 3rd leaf (bench timed region, c2)
O=gpurun_out/${R:-r1}; mkdir -p $O
for K in leaf_chain2 leaf_basis; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K -s 8 -c 1 \
      -o $O/full_c2_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_c2_$K.log 2>&1
done
