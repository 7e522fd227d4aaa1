#!/bin/bash
# Round profile artifacts for tag $R: bench lines (no profiler), ncu launch
# list of the default bench (timed region), --set full captures of the top kernels.
R=${R:-s4}
O=gpurun_out/$R
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err || exit 1
python bench.py --config c5 --batch 256 --steps 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 1200 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
for K in leaf_fused3 fft_col_kernel fft_reg_kernel trim_cl pointwise_matmul cg_update twist_fold; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K -s 20 -c 1 \
      -o $O/full_c2_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_c2_$K.log 2>&1
done
ls -la $O
