timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "TR_TRIM=new" "TR_TRIM=old"; do
 for c in "" "--config c5 --batch 256"; do
  env $v python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['config'], 'solves/s %.1f'%d['value'], {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
 done
done
