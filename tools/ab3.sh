#!/bin/bash
# ab3.sh <tag...>: c2 / c1 / c5 (256 systems) / c4 bench lines for the default library and tools/libvar/lib_<tag>.so
for rep in 1 2; do
for v in default "$@"; do
 for c in "" "--config c1" "--config c5 --batch 256 --steps 3" "--config c4 --steps 3"; do
  if [ $v = default ]; then L=paper_1302_6945_b200/libtoepreg_b200.so; else L="tools/libvar/lib_$v.so"; fi
  TR_LIB_PATH=$L python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['config'], 'solves/s %.2f'%d['value'], 'ns/cond %.0f'%d['chain']['ns_per_condition'])"
 done
done
done
