timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in "TR_TREE_L2MB=0" "TR_TREE_L2MB=16" "TR_TREE_L2MB=24" "TR_TREE_L2MB=40"; do
 for c in "--config c5 --batch 256" ""; do
  env $v python bench.py --steps 5 --no-cpu-baseline $c | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['config'], 'solves/s %.1f'%d['value'])"
 done
done
