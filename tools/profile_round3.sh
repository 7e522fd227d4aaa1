#!/bin/bash
# Round-end check for tag $R: gpu tests, smoke, bench lines (no profiler),
# ncu launch list of the default bench, --set full captures of the top kernels.
R=${R:-s7}
O=gpurun_out/$R
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
for K in leaf_fused3 fft_col_kernel; do
  timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K -s 20 -c 1 \
      -o $O/full_c2_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_c2_$K.log 2>&1
done
ls -la $O
