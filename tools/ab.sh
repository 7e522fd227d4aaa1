timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
for v in 1 0; do
 for c in "" "--config c5 --batch 256"; do
  TR_WRAP=$v python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('WRAP=$v', d['config']['config'], 'solves/s %.1f'%d['value'])"
 done
done
