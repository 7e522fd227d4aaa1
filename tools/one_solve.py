"""One batched solve (for launch-list profiling): config c2 or c5, count systems."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 32
refine = int(sys.argv[3]) if len(sys.argv) > 3 else 0
raw = wl.c2_rect(nrhs=count, seed=0) if cfg == "c2" else wl.c5_random(n=16384, count=count, seed=0)
probs = [wl.to_problem(raw, tb, i) for i in range(count)]
db = tb.DeviceBatch(probs, tb.SolverConfig(refine=refine)).stage()
db.run(with_diag=False); torch.cuda.synchronize()
torch.cuda.profiler.start()
db.run(with_diag=False); torch.cuda.synchronize()
torch.cuda.profiler.stop()
