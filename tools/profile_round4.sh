#!/bin/bash
# Final check for tag $R: gpu tests, smoke, bench lines (c2 default, c5), ncu launch list.
R=${R:-s8}
O=gpurun_out/$R
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c5 --batch 256 --steps 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
ls -la $O
