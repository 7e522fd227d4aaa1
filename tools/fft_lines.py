"""tr_fft throughput (GB/s, one read + one write per element) at given
(n, lines) shapes, with the cluster/TMA path on and off (TR_FFT_CL is read
once per process, so each setting runs in its own process)."""
import ctypes as C
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_1302_6945_b200 import _lib
    lib = _lib.load()
    for spec in sys.argv[2:]:
        n, lines = (int(v) for v in spec.split("x"))
        x = torch.randn(lines, n, dtype=torch.complex128, device="cuda")
        y = torch.empty_like(x)
        xp, yp = C.c_void_p(torch.view_as_real(x).data_ptr()), C.c_void_p(torch.view_as_real(y).data_ptr())
        for _ in range(3):
            assert lib.tr_fft(xp, yp, n, lines, -1, None) == 0
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 20
        a.record()
        for _ in range(it):
            lib.tr_fft(xp, yp, n, lines, -1, None)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / it * 1e3
        err = ((y - torch.fft.fft(x, dim=1)).abs().max() / torch.fft.fft(x, dim=1).abs().max()).item()
        print(f"{n:7d} x {lines:5d}: {us:9.1f} us  {32 * n * lines / (us * 1e-6) / 1e9:7.0f} GB/s  err {err:.1e}",
              flush=True)
else:
    shapes = sys.argv[1:] or ["32768x256", "32768x512", "12288x64", "12288x1365", "16384x256", "8192x256",
                              "65536x256"]
    for env in ("1", "0"):
        print(f"TR_FFT_CL={env}", flush=True)
        subprocess.run([sys.executable, __file__, "child"] + shapes, env=dict(os.environ, TR_FFT_CL=env))
