"""Latency of a dependent chain of tr_fft calls replayed from a CUDA graph
(the solver's execution mode), by fused-two-pass mode (TR_FFT_C2, TR_FFT_C2_CL)."""
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
        x = torch.randn(lines, n, dtype=torch.complex128, device="cuda") / n
        y = torch.empty_like(x)
        xp, yp = C.c_void_p(torch.view_as_real(x).data_ptr()), C.c_void_p(torch.view_as_real(y).data_ptr())
        s = torch.cuda.Stream()
        sp = C.c_void_p(s.cuda_stream)
        with torch.cuda.stream(s):
            for _ in range(3):
                assert lib.tr_fft(xp, yp, n, lines, -1, sp) == 0
                assert lib.tr_fft(yp, xp, n, lines, 1, sp) == 0
            x.mul_(1.0 / n / n / n)
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            reps = 32
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    assert lib.tr_fft(xp, yp, n, lines, -1, sp) == 0
                    assert lib.tr_fft(yp, xp, n, lines, 1, sp) == 0
                    x.mul_(1.0 / n)
            g.replay()
            s.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(5):
                g.replay()
            b.record(s)
            s.synchronize()
            us = a.elapsed_time(b) * 1e3 / (5 * reps * 2)
        print(f"{n:7d} x {lines:5d}: {us:8.2f} us per transform (incl. 1/2 scale kernel)  "
              f"{32 * n * lines / (us * 1e-6) / 1e9:7.0f} GB/s", flush=True)
else:
    shapes = sys.argv[1:] or ["12288x32", "12288x64", "12288x800", "12288x1600", "6144x800", "24576x800", "16384x800",
                              "32768x3200"]
    for env in ({"TR_FFT_C2": "0"}, {"TR_FFT_C2": "1"}, {"TR_FFT_C2": "1", "TR_FFT_C2_CL": "4"},
                {"TR_FFT_C2": "1", "TR_FFT_C2_CL": "8"}, {"TR_FFT_C2": "2"}):
        print(env, flush=True)
        subprocess.run([sys.executable, __file__, "child"] + shapes, env=dict(os.environ, **env))
