"""Per-step clock trace of the leaf chain kernel (system 0, round 0, last leaf)."""
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
K = tb.plan_info(probs[0])["max_leaf_conditions"]
a = np.frombuffer(buf, dtype=np.int64).reshape(-1, 4)[:K]
step = np.diff(a[:, 0])
a = a[1:K - 1]; step = step[1:K - 2]
dec = a[:, 1] - a[:, 0]; upd = a[:, 2] - a[:, 1]; pub = a[:, 3] - a[:, 2]
print("K", K, "mean step cycles %.0f  decide+ci %.0f  log+arrive+sync-wait %.0f  pre+front %.0f" % (
    step.mean(), dec.mean(), upd.mean(), pub.mean()))
print("per-step:", step.tolist())
print("handover steps (32k-1 -> 32k):", [int(step[i]) for i in range(31, K - 1, 32)])
b = np.frombuffer(buf, dtype=np.int64)[3072:3078]
print("basis kernel phases (cycles from start): load %d build %d norm+write %d check %d" % (
    b[1] - b[0], b[2] - b[1], b[3] - b[2], b[4] - b[3]))
b = np.frombuffer(buf, dtype=np.int64)[3072:3083]
if b[1] > b[0] > 0:
    print("fused3 phases (cycles from start): decider done %d, basis rows done %s, finish done %d" % (
        b[1] - b[0], [int(x - b[0]) for x in b[2:9] if x > 0], b[10] - b[0]))
