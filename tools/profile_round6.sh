#!/bin/bash
# Round check for tag $R: gpu tests, smoke, bench lines (c2 default with the CPU arm, c5, c3, c4, c1,
# c5b, the reference arm), then ncu: launch list of the c2 timed region and --set full captures of the
# top kernels.  Every ncu command runs only after the same command line exited 0 without ncu.
R=${R:-r2g}
O=gpurun_out/$R
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c5 --batch 256 --steps 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --config c3 --steps 2 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c4 --steps 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 1500 python bench.py --config c5b --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_c5b.json 2> $O/bench_c5b.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/plain_c2.log 2>&1 && \
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
for K in leaf_fused3 "fft_col_kernel" update_small combine_small; do
  N=$(echo $K | tr -cd 'a-z0-9_')
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K -s 6 -c 1 \
      -o $O/full_c2_$N python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_c2_$N.log 2>&1
  timeout 120 ncu -i $O/full_c2_$N.ncu-rep --page raw --csv > $O/full_c2_$N.csv 2>/dev/null
done
rm -f $O/*.ncu-rep.tmp
ls -la $O
