#!/bin/bash
O=gpurun_out/r2g
mkdir -p $O
rm -f $O/summary.txt
run() { # name, config args, env...
  name=$1; shift; cfg=$1; shift
  env "$@" timeout 600 python bench.py $cfg --no-cpu-baseline 2> $O/$name.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$name', round(d['value'],2), round(d['ms_per_step'],2), {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items() if k in('fft','leaf_pivot','combine','update')})
" >> $O/summary.txt 2>&1
}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for v in 0 2; do
run c2_v$v "" TR_FFT_C2=$v
run c5_v$v "--config c5 --batch 256 --steps 3" TR_FFT_C2=$v
run c4_v$v "--config c4 --steps 3" TR_FFT_C2=$v
run c3_v$v "--config c3 --steps 2" TR_FFT_C2=$v
run c1_v$v "--config c1" TR_FFT_C2=$v
run c5_b16_v$v "--config c5 --batch 16 --steps 3" TR_FFT_C2=$v
done
cat $O/summary.txt; tail -3 $O/pytest_gpu.log
