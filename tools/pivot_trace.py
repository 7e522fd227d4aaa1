import ctypes as C, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import _lib, workloads as wl
lib = _lib.load()
f = lib.tr_debug_pivot_trace
f.argtypes = [C.c_int, C.c_void_p, C.c_int]
raw = wl.c2_rect(nrhs=64, seed=0)
probs = [wl.to_problem(raw, tb, i) for i in range(64)]
db = tb.DeviceBatch(probs, tb.SolverConfig(refine=0)).stage()
db.run(); torch.cuda.synchronize()
f(1, None, 0)
import os as _o
_o.environ["TR_GRAPHS"] = "0"
db.run(); torch.cuda.synchronize()
buf = (C.c_longlong * 4096)()
f(0, C.addressof(buf), 4096)
a = np.frombuffer(buf, dtype=np.int64).reshape(-1, 4)[1:192]
d_row = a[:, 1] - a[:, 0]; d_dec = a[:, 2] - a[:, 1]; d_pub = a[:, 3] - a[:, 2]
step = np.diff(a[:, 0])
print("per step cycles: total=%.0f  rows(start->c1)=%.0f decide=%.0f publish=%.0f  barrier+rest=%.0f" % (
    step.mean(), d_row.mean(), d_dec.mean(), d_pub.mean(), step.mean() - (d_row + d_dec + d_pub)[:-1].mean()))
