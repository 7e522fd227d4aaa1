#!/bin/bash
# A/B: fft_col_kernel register budget (3 vs 4 resident CTAs per SM)
mkdir -p gpurun_out/ab
for rep in 1 2; do
 for v in base reg2; do
  for c in "" "--config c5 --batch 256 --steps 3"; do
   if [ $v = reg2 ]; then export TR_LIB_PATH=tools/libvar/lib_reg2.so; else unset TR_LIB_PATH; fi
   timeout 300 python bench.py --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['config'], 'solves/s %.1f'%d['value'], 'fft ms %.2f'%d['kernels']['fft']['ms_per_step'])"
  done
 done
done 2>&1 | tee gpurun_out/ab/col.txt
