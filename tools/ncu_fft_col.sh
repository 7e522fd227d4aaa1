#!/bin/bash
O=gpurun_out/fftcol; mkdir -p $O
for n in 16384 32768; do
  python tools/fft_one.py $n > $O/plain_$n.log 2>&1 || exit 1
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:fft_col -c 2 -o $O/col_$n python tools/fft_one.py $n > $O/ncu_$n.log 2>&1
done
ls -la $O
