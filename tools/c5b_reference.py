"""CPU baseline for BASELINE config 5b (one l2 system, n = 2^22): runs the
REFERENCE package itself (read-only import from /root/reference) on one core
and records its wall time, ledger and residual.  Hours of CPU time; run in
the background:  python tools/c5b_reference.py [log2n] > profiles/r2_c5b_reference.json"""
import json
import os
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
import toepreg  # noqa: E402
from paper_1302_6945_b200 import workloads as wl  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 22
raw = wl.c5_random(n=1 << log2n, count=1, seed=0)
prob = wl.to_problem(raw, toepreg, 0)
t0 = time.perf_counter()
rep = toepreg.solve_tikhonov(prob)
t1 = time.perf_counter()
print(json.dumps({
    "config": "c5b" if log2n == 22 else f"c5-like n=2^{log2n}",
    "n": 1 << log2n,
    "impl": "reference (toepreg.solve_tikhonov, 1 core)",
    "wall_time_s": rep.wall_time,
    "outer_wall_s": t1 - t0,
    "relative_residual": rep.relative_residual,
    "final_col_degrees": [int(v) for v in rep.final_col_degrees],
    "diagnostics": rep.diagnostics.as_dict() if hasattr(rep.diagnostics, "as_dict") else str(rep.diagnostics),
    "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t"),
}), flush=True)
