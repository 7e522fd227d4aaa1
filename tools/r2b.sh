#!/bin/bash
# fused two-pass FFT: shape sweep by mode, gpu tests, bench A/B
O=gpurun_out/r2c
mkdir -p $O
timeout 600 python tools/fft_c2.py 8192x800 12288x32 12288x64 16384x800 32768x32 32768x256 32768x3200 65536x256 > $O/fft_c2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for v in 1 0 2; do
TR_FFT_C2=$v timeout 300 python bench.py --no-cpu-baseline > $O/bench_c2_v$v.json 2> $O/bench_c2_v$v.err
TR_FFT_C2=$v timeout 600 python bench.py --config c5 --batch 256 --steps 3 --no-cpu-baseline > $O/bench_c5_v$v.json 2> $O/bench_c5_v$v.err
done
ls -la $O
