timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
for v in 1 0; do
 for c in "" "--config c5 --batch 256"; do
  TR_FFT_2STREAM=$v python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('2STREAM=$v', d['config']['config'], 'solves/s %.1f'%d['value'])"
 done
done
TR_PHASE_TIMES=1 python tools/ab_check.py c5 256 /tmp/a.npz 2>&1 | tail -2 | head -1
