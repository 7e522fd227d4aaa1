#!/bin/bash
O=gpurun_out/r2e
mkdir -p $O
rm -f $O/phases.txt
for g in 1 2; do
for only in 0 8192 12288 16384; do
for cl in 0 4 8; do
echo "== g$g only=$only cl=$cl" >> $O/phases.txt
TR_PHASE_TIMES=1 TR_GROUPS=$g TR_FFT_C2=1 TR_FFT_C2_ONLY=$only TR_FFT_C2_CL=$cl timeout 300 python bench.py --no-cpu-baseline --steps 4 2>&1 >/dev/null | grep phases | tail -3 | head -1 >> $O/phases.txt
done
done
done
cat $O/phases.txt
