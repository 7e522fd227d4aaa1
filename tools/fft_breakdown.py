"""FFT device time by (length, lines) for one solve of a config (eager, per-launch CUDA events)."""
import ctypes as C, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import _lib, workloads as wl
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 256
raw = wl.c5_random(n=16384, count=count, seed=0) if cfg == "c5" else wl.c2_rect(nrhs=count, seed=0)
probs = [wl.to_problem(raw, tb, i) for i in range(count)]
db = tb.DeviceBatch(probs).stage()
db.run(); torch.cuda.synchronize()
lib = _lib.load()
lib.tr_kernel_timing(1)
db.run(with_diag=False); torch.cuda.synchronize()
rows = (C.c_int64 * 300)(); ms = (C.c_double * 100)()
k = lib.tr_fft_breakdown(rows, ms, 100)
tot = sum(ms[i] for i in range(k))
print(f"{cfg} x{count}: FFT total {tot:.2f} ms in {sum(rows[3*i+2] for i in range(k))} launches")
for i in range(min(k, 25)):
    n, lines, cnt = rows[3 * i], rows[3 * i + 1], rows[3 * i + 2]
    gb = 2 * 16 * n * lines * cnt / 1e9
    print(f"  n={n:6d} lines={lines:6d} calls={cnt:5d} ms={ms[i]:8.2f}  {gb / (ms[i] / 1e3):7.0f} GB/s (in+out once)")
lib.tr_kernel_timing(0)
