#!/bin/bash
# c2 (direct solve only) step time and per-class device time vs batch size
for b in ${BATCHES:-1 4 16 64}; do
  echo "== batch=$b"
  timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --refine ${REFINE:-0} --batch $b 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])
for k,v in d['kernels'].items(): print('   %-12s %8.3f ms %6d launches' % (k, v['ms_per_step'], v['launches_per_step']))"
done
