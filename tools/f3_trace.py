"""Phase clock trace of leaf_fused3_kernel (system 0, last leaf): per round
[start, decider end, basis end, normalise, residual] and the commit."""
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
b = np.frombuffer(buf, dtype=np.int64)[3072:3072 + 130].copy()
print("kernel entry to the first chain step: %d cycles" % (b[0] - b[129]))
t0 = b[0]
for r in range(4):
    x = b[32 * r:32 * r + 24]
    if x[0] > 0 and abs(x[0] - t0) < 1e8:
        blocks = [int(v - x[0]) for v in x[:12] if 0 < v - x[0] < 1e8]
        print("round %d: start %d, block starts %s, decider end %d, chain+basis %d, normalised %d, residual %d"
              % (r, x[0] - t0, blocks, x[12] - x[0], x[13] - x[0], x[14] - x[0], x[15] - x[0]))
        print("   residual detail (fold, dft, rows per coset):", [int(v - x[0]) for v in x[16:22]])
        print("   hand-over waits of blocks 1..7 (cycles):", [int(v) for v in b[32 * r + 25:32 * r + 32]])
        print("   epilogue done %d, normalised rows written %d" % (x[22] - x[0], x[23] - x[0]))
print("commit at %d" % (b[128] - t0))
