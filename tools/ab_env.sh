#!/bin/bash
# ab_env.sh VAR: bench lines (c2, c5 at 256 systems, c3, c1) with VAR unset and VAR=0, twice
V=$1
for rep in 1 2; do
for val in on 0; do
 for c in "" "--config c5 --batch 256 --steps 3" "--config c3 --steps 2" "--config c1"; do
  if [ $val = on ]; then unset $V; else export $V=0; fi
  python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$V=$val', d['config']['config'], 'solves/s %.2f'%d['value'], 'ms/step %.2f'%d['ms_per_step'])"
 done
done
done
