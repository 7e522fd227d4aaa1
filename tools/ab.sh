python tools/cg_iterations.py 2>&1 | tail -5
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in "" "--config c5 --batch 256" "--config c1" "--config c4"; do
  python bench.py --steps 3 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['config'], 'solves/s %.2f'%d['value'])"
done
