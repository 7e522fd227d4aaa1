"""Batched complex128 FFT throughput: this library's tr_fft vs cuFFT (torch.fft)
on the same lengths (GB/s counting one read + one write of the data)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_6945_b200 import _lib  # noqa: E402

lib = _lib.load()
torch.cuda.set_device(0)
sizes = [int(s) for s in sys.argv[1:]] or [128, 256, 512, 1024, 2048, 4096, 3 * 1024, 5 * 512,
                                           8192, 16384, 32768, 65536, 3 * 16384, 131072]
TOT = 1 << 24  # complex elements per call (256 MiB)
print(f"{'n':>8s} {'lines':>7s} {'ours GB/s':>10s} {'cufft GB/s':>11s} {'ratio':>6s} {'maxerr':>9s}")
for n in sizes:
    lines = max(1, TOT // n)
    x = torch.randn(lines, n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    xp = C.c_void_p(torch.view_as_real(x).data_ptr())
    yp = C.c_void_p(torch.view_as_real(y).data_ptr())

    def ours():
        assert lib.tr_fft(xp, yp, n, lines, -1, None) == 0

    def cufft():
        return torch.fft.fft(x, dim=1)

    res = {}
    for name, f in (("ours", ours), ("cufft", cufft)):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 10
        a.record()
        for _ in range(it):
            f()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / it
        res[name] = 2 * 16 * lines * n / (ms * 1e-3) / 1e9
    ref = torch.fft.fft(x, dim=1)
    ours()
    torch.cuda.synchronize()
    err = ((y - ref).abs().max() / ref.abs().max()).item()
    print(f"{n:8d} {lines:7d} {res['ours']:10.0f} {res['cufft']:11.0f} {res['ours']/res['cufft']:6.2f} {err:9.1e}")
