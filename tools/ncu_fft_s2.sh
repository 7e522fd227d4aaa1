#!/bin/bash
# --set full captures of the dominant FFT kernels at config 5 (batch 256)
O=gpurun_out/s2
mkdir -p $O
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"fft_col_kernel|fft_reg_kernel|pointwise|trim_fused|twist_fold" -s 20 -c 12 -o $O/fft_c5 python tools/prof_run.py c5 256 > $O/ncu_fft_c5.log 2>&1
tail -3 $O/ncu_fft_c5.log
