"""tr_fft throughput (GB/s, one read + one write per element) at given
(n, lines) shapes with the fused two-pass cluster kernel on and off
(TR_FFT_C2 is read once per process, so each setting runs in its own process)."""
import ctypes as C
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_1302_6945_b200 import _lib
    lib = _lib.load()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for spec in sys.argv[2:]:
        n, lines = (int(v) for v in spec.split("x"))
        x = torch.randn(lines, n, dtype=torch.complex128, device="cuda")
        y = torch.empty_like(x)
        xp, yp = C.c_void_p(torch.view_as_real(x).data_ptr()), C.c_void_p(torch.view_as_real(y).data_ptr())
        for _ in range(3):
            assert lib.tr_fft(xp, yp, n, lines, -1, None) == 0
        torch.cuda.synchronize()
        it = 10
        tot = 0.0
        for _ in range(it):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            lib.tr_fft(xp, yp, n, lines, -1, None)
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        us = tot / it * 1e3
        ref = torch.fft.fft(x, dim=1)
        err = ((y - ref).abs().max() / ref.abs().max()).item()
        # in place, inverse sign
        z = x.clone()
        zp = C.c_void_p(torch.view_as_real(z).data_ptr())
        assert lib.tr_fft(zp, zp, n, lines, 1, None) == 0
        ref2 = torch.fft.ifft(x, dim=1) * n
        err2 = ((z - ref2).abs().max() / ref2.abs().max()).item()
        print(f"{n:7d} x {lines:5d}: {us:9.1f} us  {32 * n * lines / (us * 1e-6) / 1e9:7.0f} GB/s  "
              f"err {err:.1e} inplace/inv {err2:.1e}", flush=True)
        del x, y, z, ref, ref2
else:
    shapes = sys.argv[1:] or ["8192x64", "8192x800", "12288x32", "12288x64", "12288x1365", "16384x64", "16384x800",
                              "32768x32", "32768x256", "32768x3200", "65536x256", "24576x256", "20480x256",
                              "28672x256", "18432x256", "30720x256", "10240x256", "131072x64"]
    for env in ("1", "2", "0"):
        print(f"TR_FFT_C2={env}", flush=True)
        subprocess.run([sys.executable, __file__, "child"] + shapes, env=dict(os.environ, TR_FFT_C2=env))
