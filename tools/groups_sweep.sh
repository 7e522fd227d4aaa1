#!/bin/bash
# c2 step time vs the number of stream groups the 64 right-hand sides are split into
for r in 1 0; do
for g in ${GROUPS_LIST:-1 2 3 4 6 8}; do
  echo "== refine=$r groups=$g"
  TR_GROUPS=$g timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --refine $r 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done; done
