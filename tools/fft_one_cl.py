import ctypes as C, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_6945_b200 import _lib
lib = _lib.load()
n, lines = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32768x256").split("x"))
x = torch.randn(lines, n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    lib.tr_fft(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), n, lines, -1, None)
torch.cuda.synchronize()
