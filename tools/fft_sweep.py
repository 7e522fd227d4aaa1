"""Time tr_fft for every length 2^a q (q in 1,3,5,7,9,15) in [lo, hi]; prints
'n ms_per_Gelem' lines used to rank FFT lengths (fft_good_len cost table)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_6945_b200 import _lib
lib = _lib.load()
lo = int(sys.argv[1]) if len(sys.argv) > 1 else 16
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 17
TOT = 1 << 23
sizes = sorted({q << a for q in (1, 3, 5, 7, 9, 15) for a in range(0, 18) if lo <= (q << a) <= hi})
x = torch.randn(TOT, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
for n in sizes:
    lines = max(1, TOT // n)
    xp, yp = C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr())
    for _ in range(3):
        lib.tr_fft(xp, yp, n, lines, -1, None)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 10
    a.record()
    for _ in range(it):
        lib.tr_fft(xp, yp, n, lines, -1, None)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / it
    print(f"{n} {ms / (lines * n) * 1e9 / 1e3:.4f}")  # us per million elements
