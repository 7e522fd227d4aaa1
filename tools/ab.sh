TR_F3_PAIR=0 python tools/f3_trace.py c2 64 2>&1 | tail -4
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
python bench.py --steps 5 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['config'], 'solves/s %.1f'%d['value'])"
