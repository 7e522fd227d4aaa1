#!/bin/bash
# Round check for tag $R: gpu tests, smoke, bench lines (c2 default, c5, reference arm),
# ncu launch lists of the bench timed region (c2 and c5).  Each ncu command runs only
# after the same command line exited 0 without ncu.
R=${R:-r2}
O=gpurun_out/$R
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c5 --batch 256 --steps 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/plain_c2.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
python bench.py --config c5 --batch 256 --steps 1 --warmup 3 --no-cpu-baseline > $O/plain_c5.log 2>&1 && \
timeout 2400 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --config c5 --batch 256 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c5.log 2>&1
ls -la $O
