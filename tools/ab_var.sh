#!/bin/bash
# ab_var.sh <tag...>: c2 (and c1) bench lines for the default library and tools/libvar/lib_<tag>.so, twice each
for rep in 1 2; do
for v in default "$@"; do
 for c in "" "--config c1"; do
  if [ $v = default ]; then L=""; else L="tools/libvar/lib_$v.so"; fi
  TR_LIB_PATH=${L:-paper_1302_6945_b200/libtoepreg_b200.so} python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['config'], 'solves/s %.1f'%d['value'], 'ns/cond %.0f'%d['chain']['ns_per_condition'])"
 done
done
done
