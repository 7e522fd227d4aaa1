"""Phase clock trace of the cluster FFT (cluster 0, CTA 0): cycles per phase
per line: wait(TMA) passA sync1 exchange sync2 passB."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_6945_b200 import _lib
lib = _lib.load()
f = lib.tr_debug_cl_trace
f.argtypes = [C.c_int, C.c_void_p]
n, lines = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32768x256").split("x"))
x = torch.randn(lines, n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
lib.tr_fft(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), n, lines, -1, None)
torch.cuda.synchronize()
f(1, None)
lib.tr_fft(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), n, lines, -1, None)
torch.cuda.synchronize()
buf = np.zeros(8 * 64, dtype=np.int64)
f(0, buf.ctypes.data)
t = buf.reshape(64, 8)
rows = [r for r in t if r[0] > 0]
print("it   wait  passA  sync  recv  passB  cwait  (cycles)  next-iter")
for i, r in enumerate(rows):
    d = np.diff(r[:7])
    nxt = rows[i + 1][0] - r[6] if i + 1 < len(rows) else 0
    print(i, *[f"{v:6d}" for v in d], f"{nxt:6d}")
