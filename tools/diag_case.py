"""Diagnostic: solve one golden fixture on the GPU and print the raw per-system
tr_diag (status, deferred count, ledger, truncations) without raising.

    python tools/diag_case.py <fixture name> [refine]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_1302_6945_b200 as tb  # noqa: E402
from conftest import case_config, load_case, rel  # noqa: E402
from paper_1302_6945_b200 import workloads as wl  # noqa: E402

name = sys.argv[1]
refine = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw, d = load_case(os.path.join(ROOT, "tests", "golden", "cases", name + ".npz"))
prob = wl.to_problem(raw, tb)
db = tb.DeviceBatch([prob], case_config(tb, d, refine)).stage().run()
x = db.fetch()[0]
g = db.diag[0]
p = len(d["final_col_degrees"])
print(f"{name} refine={refine} rc={db.rc} status={g.status} dp={g.difficult_points} (ref {int(d['difficult_points'])})"
      f" ledger={list(g.final_col_degrees[:p])} (ref {list(d['final_col_degrees'])}) trim_overflow={g.trim_overflow}"
      f" retried={g.retried_leaves} resid={g.relative_residual:.3e} (ref {float(d['relative_residual']):.3e})"
      f" cg_it={g.refine_cg_iterations} gpu<->exact={rel(x, d['x_exact']):.3e}"
      f" ref<->exact={rel(d['x_hat'], d['x_exact']):.3e} gpu<->ref={rel(x, d['x_hat']):.3e}")
