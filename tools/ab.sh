for v in 1 0; do
 for c in "" "--config c5 --batch 128"; do
  TR_F3=$v python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('F3=$v', d['config']['config'], 'solves/s %.1f'%d['value'], {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
 done
done
