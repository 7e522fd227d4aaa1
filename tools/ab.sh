timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/ab_check.py c2 64 /tmp/a2.npz; TR_GROUPS=1 python tools/ab_check.py c2 64 /tmp/b2.npz; python tools/ab_check.py --cmp /tmp/a2.npz /tmp/b2.npz
for v in 1 2 3 4; do
  TR_GROUPS=$v python bench.py --steps 10 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('G=$v', d['config']['config'], 'solves/s %.1f'%d['value'], 'e2e %.1f'%d['e2e']['value'])"
done
