#!/bin/bash
# Round profile artifacts (run under gpurun): bench lines first (no profiler),
# then ncu launch lists of the same bench commands (timed region only, via
# cudaProfilerStart/Stop in bench.py), then --set full captures of the top
# kernels.  Output: gpurun_out/$R/.
R=${R:-r1}
O=gpurun_out/$R
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err || exit 1
python bench.py --config c5 --batch 256 --steps 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
for K in leaf_chain2 leaf_basis fft_reg_kernel fft_col_kernel trim_fused pointwise_matmul; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K -s 5 -c 1 \
      -o $O/full_c2_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_c2_$K.log 2>&1
done
ls -la $O
