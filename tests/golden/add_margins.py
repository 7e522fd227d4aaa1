"""Annotate every golden fixture with how close the reference's discrete
decisions were to flipping under rounding, and with the reference's own
rounding-path spread.

    python tests/golden/add_margins.py [pattern]

The oracle reproduces the reference bit for bit (tests/test_oracle.py), so
its instrumented run (toepreg_oracle.MARGINS) sees the reference's decisions:

* ``margin_pivot``  min over pivot decisions of 1 - |phi_2nd| / |phi_1st|
                    among the candidate columns (0 = an exact tie);
* ``margin_defer``  min over decisions of |log10(|phi_j| / (thr max|phi|))|
                    (0 = on the deferral threshold, ref tanint.py:200-205);
* ``margin_check``  min over leaf attempts of |log10(res / 1e-11)|
                    (0 = on the self-check tolerance that triggers a retry
                    with another absorption order, ref tanint.py:423-429).

A GPU run whose arithmetic differs in rounding reproduces the reference's
degree ledger exactly when these margins exceed the rounding difference of
the quantities compared; when a leaf self-check sits within a factor of a
few of its tolerance, a retry may happen on one side only and the two runs
absorb that leaf in different orders (both valid).

* ``spread_exact``  distance to the exact solution of the reference's
                    algorithm with its long-double tree products replaced by
                    float64 ones: how far the reference's own
                    answer moves under a rounding change;
* ``spread_col_degrees``  that variant's final degree ledger.
"""

from __future__ import annotations

import glob
import multiprocessing as mp
import os
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]


def annotate(path):
    import toepreg_oracle as O
    import paper_1302_6945_b200 as tb
    from paper_1302_6945_b200 import workloads as wl
    from conftest import load_case
    raw, d = load_case(path)
    prob = wl.to_problem(raw, tb)
    fill = str(d["cfg_fill"]) if "cfg_fill" in d else "auto"
    O.MARGINS = []
    O.COMBINE_EXTENDED = True
    r = O.solve(prob, fill=fill)
    same = np.array_equal(r["x_hat"], d["x_hat"])
    m = O.MARGINS
    O.MARGINS = None

    def mins(kind, f):
        v = [f(x) for k, x in m if k == kind]
        return float(min(v)) if v else float("inf")

    out = dict(d)
    out["margin_pivot"] = np.array(mins("pivot", lambda x: x))
    # an exactly zero pivot candidate is deferred by any rounding: no margin issue
    out["margin_defer"] = np.array(mins("defer", lambda x: abs(np.log10(x)) if x > 0 else np.inf))
    out["margin_check"] = np.array(mins("check", lambda x: abs(np.log10(x)) if x > 0 else np.inf))
    O.COMBINE_EXTENDED = False
    try:
        rv = O.solve(prob, fill=fill)
        ex = d["x_exact"]
        out["spread_exact"] = np.array(float(np.linalg.norm(rv["x_hat"] - ex) / np.linalg.norm(ex)))
        out["spread_col_degrees"] = rv["final_col_degrees"]
    except Exception:  # the variant may fail where the reference barely succeeds
        out["spread_exact"] = np.array(float("inf"))
    O.COMBINE_EXTENDED = True
    np.savez_compressed(path, **out)
    flip = "spread_col_degrees" in out and not np.array_equal(out["spread_col_degrees"],
                                                              d["final_col_degrees"])
    return (os.path.basename(path), same, float(out["margin_pivot"]), float(out["margin_defer"]),
            float(out["margin_check"]), float(out["spread_exact"]), flip)


if __name__ == "__main__":
    pat = sys.argv[1] if len(sys.argv) > 1 else "*"
    paths = sorted(glob.glob(os.path.join(HERE, "cases", pat + ".npz")))
    paths.sort(key=lambda p: -os.path.getsize(p) if "c3_full" not in p else -1e12)
    with mp.get_context("spawn").Pool(8) as pool:
        for name, same, mp_, md, mc, sp, flip in pool.imap_unordered(annotate, paths):
            print(f"{name:32s} oracle==ref {same}  pivot {mp_:.2e}  defer {md:.2f}  check {mc:.2f}"
                  f"  spread {sp:.2e}  ledger flips under FP64 combine: {flip}", flush=True)
