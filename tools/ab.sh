TR_PHASE_TIMES=1 python tools/ab_check.py c5 256 /tmp/a.npz 2>&1 | tail -2 | head -1
for c in "" "--config c5 --batch 256"; do
  python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['config'], 'solves/s %.1f'%d['value'])"
done
