"""A/B check: solve a workload, save x + diagnostics to an .npz (run twice under
different env settings, then compare with --cmp a.npz b.npz)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        d = np.max(np.abs(a[k] - b[k])) if a[k].size else 0.0
        print(k, "max|diff|", d, "rel", d / max(np.max(np.abs(a[k])), 1e-300))
    sys.exit(0)
import torch
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl
cfg, count, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = wl.c2_rect(nrhs=count, seed=0) if cfg == "c2" else wl.c5_random(n=16384, count=count, seed=0)
probs = [wl.to_problem(raw, tb, i) for i in range(count)]
db = tb.DeviceBatch(probs, tb.SolverConfig(refine=int(os.environ.get("REFINE", "1")))).stage()
for _ in range(3):
    db.run()
torch.cuda.synchronize()
t0 = time.time()
for _ in range(3):
    db.run()
torch.cuda.synchronize()
print(cfg, count, "s/run %.4f" % ((time.time() - t0) / 3))
reps = db.reports(db.fetch())
np.savez(out, x=np.stack([r.x_hat for r in reps]),
         deg=np.stack([np.asarray(r.final_col_degrees) for r in reps]),
         res=np.array([r.relative_residual for r in reps]),
         scale=np.array([r.diagnostics.max_column_scale for r in reps]))
