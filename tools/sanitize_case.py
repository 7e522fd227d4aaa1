"""Small solves for compute-sanitizer (racecheck / synccheck / memcheck):
config 1 (n = 256, 4 leaves) and config-5 shape at n = 512 (batch of 2),
refinement on (CG + final residual), through the public API.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import paper_1302_6945_b200 as tb  # noqa: E402
from paper_1302_6945_b200 import workloads as wl  # noqa: E402

which = sys.argv[1:] or ["c1", "c5"]
if "c1" in which:
    raw = wl.c1_blur(256)
    r = tb.solve_tikhonov(wl.to_problem(raw, tb))
    print("c1 ok", r.final_col_degrees, r.relative_residual)
if "c5" in which:
    raw = wl.c5_random(n=512, count=2, seed=1)
    reps = tb.solve_tikhonov_batch([wl.to_problem(raw, tb, i) for i in range(2)])
    print("c5 n=512 ok", [r.relative_residual for r in reps])
if "c2" in which:
    raw = wl.c2_rect(m=1024, n=512, nrhs=2, seed=0)
    reps = tb.solve_tikhonov_batch([wl.to_problem(raw, tb, i) for i in range(2)])
    print("c2 mini ok", [r.relative_residual for r in reps])
