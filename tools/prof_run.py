"""Run one warm solve, then one solve between cudaProfilerStart/Stop (for
ncu --profile-from-start off)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 64
if cfg == "c5":
    raw = wl.c5_random(n=16384, count=count, seed=0)
else:
    raw = wl.c2_rect(nrhs=count, seed=0)
probs = [wl.to_problem(raw, tb, i) for i in range(count)]
db = tb.DeviceBatch(probs).stage()
db.run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
db.run(with_diag=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
