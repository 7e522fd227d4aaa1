"""Run tr_fft(n, lines) a few times (for ncu)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_6945_b200 import _lib
lib = _lib.load()
n = int(sys.argv[1]); lines = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, (1 << 24) // n)
x = torch.randn(lines, n, dtype=torch.complex128, device="cuda"); y = torch.empty_like(x)
for _ in range(3):
    assert lib.tr_fft(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), n, lines, -1, None) == 0
torch.cuda.synchronize()
print("ok")
