timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
for c in "" "--config c5 --batch 256"; do
  python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['config'], 'solves/s %.1f'%d['value'])"
done
python -c "import __graft_entry__ as g; g.smoke()"
