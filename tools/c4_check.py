"""Config-4 status check: direct solve diagnostics under a few settings."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl
raw = wl.c4_nufft(seed=0)
p = wl.to_problem(raw, tb)
for refine in (0, 1):
    try:
        r = tb.solve_tikhonov(p, tb.SolverConfig(refine=refine))
        xt = raw["x_true"]
        print(os.environ.get("TAG", ""), "refine", refine, "ok dp", r.diagnostics.difficult_points, "res %.3e" % r.relative_residual,
              "err %.3e" % (np.linalg.norm(r.x_hat - xt) / np.linalg.norm(xt)), "deg", r.final_col_degrees.tolist())
    except Exception as e:
        print(os.environ.get("TAG", ""), "refine", refine, "FAILED", type(e).__name__, e)
