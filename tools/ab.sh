python bench.py --config c5 --batch 512 --steps 2 --warmup 2 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['config'], d['config']['systems_per_rank'], 'solves/s %.1f'%d['value'])"
python - <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl
sys.path.insert(0,'oracle')
for count in (160, 300):
    raw = wl.c5_random(n=2048, count=count, seed=5)
    probs = [wl.to_problem(raw, tb, i) for i in range(count)]
    reps = tb.solve_tikhonov_batch(probs)
    single = tb.solve_tikhonov(probs[count - 1])
    import toepreg_oracle as O
    ex = O.dense_solution(probs[count - 1])
    print(count, "batch-vs-single equal:", np.array_equal(reps[-1].x_hat, single.x_hat),
          "err vs dense %.2e" % (np.linalg.norm(reps[-1].x_hat - ex) / np.linalg.norm(ex)),
          "max resid %.1e" % max(r.relative_residual for r in reps))
PY
