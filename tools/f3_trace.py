"""Phase clock trace of leaf_fused3_kernel (system 0, round 0, last leaf)."""
import ctypes as C, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["TR_GRAPHS"] = "0"
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import _lib, workloads as wl
lib = _lib.load()
f = lib.tr_debug_chain_trace
f.argtypes = [C.c_int, C.c_void_p, C.c_int]
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 64
raw = wl.c2_rect(nrhs=count, seed=0) if cfg == "c2" else wl.c5_random(n=16384, count=count, seed=0)
probs = [wl.to_problem(raw, tb, i) for i in range(count)]
db = tb.DeviceBatch(probs, tb.SolverConfig(refine=0)).stage()
db.run(); torch.cuda.synchronize()
f(1, None, 0)
db.run(); torch.cuda.synchronize()
buf = (C.c_longlong * 4096)()
f(0, C.addressof(buf), 4096)
b = np.frombuffer(buf, dtype=np.int64)[3072:3072 + 24].copy()
t0 = b[0]
print("block starts:", [int(x - t0) for x in b[:9] if x > 0])
print("decider end %d; loop end decider %d; basis ends %s; finish end %d" % (
    b[9] - t0, b[10] - t0, [int(x - t0) for x in b[11:18] if x > 0], b[20] - t0))
