"""Warm per-class device time (CUDA events around every launch, eager) and
the graph-mode time of the same batched solve."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import _lib, workloads as wl
lib = _lib.load()
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 32
refine = int(sys.argv[3]) if len(sys.argv) > 3 else 0
raw = wl.c2_rect(nrhs=count, seed=0) if cfg == "c2" else wl.c5_random(n=16384, count=count, seed=0)
probs = [wl.to_problem(raw, tb, i) for i in range(count)]
db = tb.DeviceBatch(probs, tb.SolverConfig(refine=refine)).stage()
for _ in range(3):
    db.run(with_diag=False)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); 
for _ in range(5):
    db.run(with_diag=False)
b.record(); torch.cuda.synchronize()
print(f"graph mode: {a.elapsed_time(b)/5:.2f} ms per solve of {count}")
lib.tr_kernel_timing(1)
db.run(with_diag=False); torch.cuda.synchronize()
st = _lib.kernel_stats()
lib.tr_kernel_timing(0)
tot = sum(v[0] for v in st.values())
print(f"eager kernel sum: {tot:.2f} ms")
for k, v in sorted(st.items(), key=lambda x: -x[1][0]):
    if v[1]:
        print(f"  {k:12s} {v[0]:8.3f} ms {v[1]:6d} launches {1e3*v[0]/v[1]:7.1f} us avg")
