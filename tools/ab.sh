for rep in 1 2; do
for v in s0 s16 s64 s256; do
 for c in "" "--config c5 --batch 256"; do
  TR_LIB_PATH=tools/libvar/lib_$v.so python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['config'], 'solves/s %.1f'%d['value'], 'ns/cond %.0f'%d['chain']['ns_per_condition'])"
 done
done
done
