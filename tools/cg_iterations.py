import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl
for cfg, raw, k in (("c2", wl.c2_rect(nrhs=8, seed=0), 8), ("c5", wl.c5_random(n=16384, count=8, seed=0), 8),
                    ("c1", wl.c1_blur(256, seed=0), 1), ("c3", wl.c3_firstdiff(n=4096, lam=1e-2, seed=0), 1),
                    ("c4mini", wl.c4_nufft(m=1024, n=2048, seed=0), 1)):
    probs = [wl.to_problem(raw, tb, i) for i in range(k)] if k > 1 else [wl.to_problem(raw, tb)]
    reps = tb.solve_tikhonov_batch(probs)
    print(cfg, "cg iterations", [r.diagnostics.refine_cg_iterations for r in reps], "resid", ["%.1e" % r.relative_residual for r in reps][:3])
