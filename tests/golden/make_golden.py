"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference lives at /root/reference and is
read-only; it is not present on the GPU box, which only sees the committed
.npz files):

    python tests/golden/make_golden.py

Every fixture stores the inputs (or the seed recipe that regenerates them
bit-for-bit with numpy's SeedSequence streams), the reference's outputs
(``x_hat``, ``final_col_degrees``, diagnostics, ``relative_residual``) and,
where the size allows, an exact solution from the reference's own dense
oracle (``dense_oracle``, ref: pkg/src/toepreg/solver.py:81-101) or
tight-tolerance CG (``cg_solve``, ref: solver.py:181-215).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import toepreg  # noqa: E402  (the reference, read-only)
from toepreg import extension as rext  # noqa: E402
from toepreg import fftpoly as rfft  # noqa: E402
from toepreg import tanint as rtan  # noqa: E402

from paper_1302_6945_b200 import workloads as wl  # noqa: E402

OUT = os.path.join(HERE, "cases")
STAGE = os.path.join(HERE, "stages")


def _exact(problem, n):
    if n <= 2048:
        return toepreg.dense_oracle(problem, max_n=2048), "dense"
    x, it = toepreg.cg_solve(problem, toepreg.CGConfig(tolerance=1e-15,
                                                       max_iterations=20000))
    return x, f"cg{it}"


def _save_case(name, raw, problem, store_inputs=True, recipe=None):
    t0 = time.perf_counter()
    rep = toepreg.solve_tikhonov(problem)
    dt = time.perf_counter() - t0
    n = problem.n
    exact, how = _exact(problem, n)
    out = {
        "variant": np.array(raw["variant"]),
        "m": np.array(raw["m"]),
        "n": np.array(raw["n"]),
        "x_hat": rep.x_hat,
        "final_col_degrees": rep.final_col_degrees,
        "relative_residual": np.array(rep.relative_residual),
        "conditions_total": np.array(rep.diagnostics.conditions_total),
        "difficult_points": np.array(rep.diagnostics.difficult_points),
        "recursion_depth": np.array(rep.diagnostics.recursion_depth),
        "max_column_scale": np.array(rep.diagnostics.max_column_scale),
        "x_exact": exact,
        "exact_how": np.array(how),
        "ref_seconds": np.array(dt),
    }
    if store_inputs:
        for key in ("T_gen", "L_gen", "G_col", "b", "normal_rhs"):
            v = raw.get(key)
            if v is not None:
                out[key] = np.asarray(v)
        for key in ("beta", "L_rows"):
            if raw.get(key) is not None:
                out[key] = np.array(raw[key])
    if recipe is not None:
        out["recipe"] = np.array(recipe)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    err = np.linalg.norm(rep.x_hat - exact) / np.linalg.norm(exact)
    print(f"{name:28s} n={n:6d} ref={dt:7.3f}s dp={rep.diagnostics.difficult_points}"
          f" ref<->exact={err:.3e} ({how})", flush=True)


def _pick(raw, i):
    d = dict(raw)
    for key in ("T_gen", "b", "normal_rhs", "x_true"):
        v = d.get(key)
        if v is not None and np.asarray(v).ndim == 2:
            d[key] = np.asarray(v)[i]
    return d


def solves():
    os.makedirs(OUT, exist_ok=True)
    # known-answer cases (ref tests/test_solver.py:48-61)
    ident = {"variant": "general", "m": 4, "n": 4,
             "T_gen": np.eye(1, 7, 3, dtype=np.complex128)[0],
             "L_rows": 4, "L_gen": np.eye(1, 7, 3, dtype=np.complex128)[0],
             "b": np.array([4.0, 8.0, 12.0, 16.0], dtype=np.complex128)}
    _save_case("known_identity_general4", ident, wl.to_problem(ident, toepreg))
    ridge = {"variant": "l2", "m": 1, "n": 1, "T_gen": np.array([2.0 + 0j]),
             "beta": 1.0, "b": np.array([10.0 + 0j])}
    _save_case("known_scalar_ridge", ridge, wl.to_problem(ridge, toepreg))
    # rectangular general (ref tests/test_solver.py:64-79 shape)
    rng = np.random.default_rng(12)
    cn = lambda k: (rng.standard_normal(k) + 1j * rng.standard_normal(k)) / np.sqrt(2)
    rect = {"variant": "general", "m": 24, "n": 16, "T_gen": cn(39), "L_rows": 10,
            "L_gen": cn(25), "b": rng.standard_normal(24) + 1j * rng.standard_normal(24)}
    _save_case("rect_general_24x16_L10", rect, wl.to_problem(rect, toepreg))
    # small corpus subset (ref tests/test_acceptance.py:65-83 stream)
    for code, variant in enumerate(("general", "l2", "gramian")):
        for n in (4, 8, 16, 32, 64):
            for trial in range(2):
                rng = np.random.default_rng(np.random.SeedSequence((8801, code, n, trial)))
                raw = wl.random_problem(variant, n, rng)
                _save_case(f"small_{variant}_n{n}_t{trial}", raw, wl.to_problem(raw, toepreg))
    # n = 512 random instances, one per variant
    for code, variant in enumerate(("general", "l2", "gramian")):
        rng = np.random.default_rng(np.random.SeedSequence((2024, code, 512)))
        raw = wl.random_problem(variant, 512, rng)
        _save_case(f"rand512_{variant}", raw, wl.to_problem(raw, toepreg))
    # BASELINE config 1 at full size
    raw = wl.c1_blur(256, seed=0)
    _save_case("c1_full", raw, wl.to_problem(raw, toepreg))
    # config 2 shape, reduced and one full RHS (inputs regenerated from the seed)
    raw = wl.c2_rect(m=1024, n=512, nrhs=2, seed=0)
    for i in range(2):
        _save_case(f"c2_mini_rhs{i}", _pick(raw, i), wl.to_problem(raw, toepreg, i))
    raw = wl.c2_rect(nrhs=1, seed=0)
    _save_case("c2_full_rhs0", _pick(raw, 0), wl.to_problem(raw, toepreg, 0),
               store_inputs=False, recipe="c2_rect(nrhs=1, seed=0)[0]")
    # config 3 shape, reduced
    for lam in (1e-2, 1.0):
        raw = wl.c3_firstdiff(n=1024, lam=lam, seed=0)
        _save_case(f"c3_mini_lam{lam:g}", raw, wl.to_problem(raw, toepreg))
    # config 4 shape, reduced
    raw = wl.c4_nufft(m=512, n=1024, seed=0)
    _save_case("c4_mini", raw, wl.to_problem(raw, toepreg))
    # config 5 shape, reduced, and one full-size system
    raw = wl.c5_random(n=2048, count=2, seed=0)
    for i in range(2):
        _save_case(f"c5_mini_sys{i}", _pick(raw, i), wl.to_problem(raw, toepreg, i))
    raw = wl.c5_random(n=16384, count=1, seed=0)
    _save_case("c5_full_sys0", _pick(raw, 0), wl.to_problem(raw, toepreg, 0),
               store_inputs=False, recipe="c5_random(n=16384, count=1, seed=0)[0]")


def stages():
    """Stage-level fixtures: assembled weights, coset evaluation, the
    long-double product, and one leaf's basis, all from the reference."""
    os.makedirs(STAGE, exist_ok=True)
    rng = np.random.default_rng(np.random.SeedSequence((8801, 1, 64, 0)))
    raw = wl.random_problem("l2", 64, rng)
    prob = wl.to_problem(raw, toepreg)
    sysm = rext.assemble(prob)
    np.savez_compressed(os.path.join(STAGE, "assemble_l2_n64.npz"),
                        weights=sysm.weights, order=sysm.order, tau=sysm.tau,
                        T_gen=raw["T_gen"], b=raw["b"], beta=raw["beta"])
    for variant, code in (("general", 0), ("gramian", 2)):
        rng = np.random.default_rng(np.random.SeedSequence((8801, code, 32, 0)))
        raw = wl.random_problem(variant, 32, rng)
        sysm = rext.assemble(wl.to_problem(raw, toepreg))
        extra = {k: raw[k] for k in ("T_gen", "L_gen", "G_col", "b", "normal_rhs")
                 if raw.get(k) is not None}
        np.savez_compressed(os.path.join(STAGE, f"assemble_{variant}_n32.npz"),
                            weights=sysm.weights, order=sysm.order, tau=sysm.tau,
                            L_rows=raw["L_rows"], **extra)
    # coset evaluation of a random cube
    rng = np.random.default_rng(77)
    cube = rng.standard_normal((2, 2, 300)) + 1j * rng.standard_normal((2, 2, 300))
    ev = {}
    for (N, off, st) in ((512, 3, 8), (512, 0, 4), (12288, 5, 64), (1024, 7, 1)):
        ev[f"N{N}_o{off}_s{st}"] = rfft.grid_eval(cube, N, offset=off, stride=st)
    np.savez_compressed(os.path.join(STAGE, "grid_eval.npz"), cube=cube, **ev)
    # long-double matrix-polynomial product
    a = rng.standard_normal((5, 5, 65)) + 1j * rng.standard_normal((5, 5, 65))
    b = rng.standard_normal((5, 5, 97)) + 1j * rng.standard_normal((5, 5, 97))
    np.savez_compressed(os.path.join(STAGE, "matpoly.npz"), a=a, b=b,
                        ld=rfft.matpoly_multiply(a, b, extended=True),
                        f64=rfft.matpoly_multiply(a, b, extended=False))
    # the first leaf of config 1 through the reference's serial driver
    raw = wl.c1_blur(256, seed=0)
    sysm = rext.assemble(wl.to_problem(raw, toepreg))
    ts = rtan.TauState.from_tau(sysm.tau)
    idx = np.sort(np.concatenate([np.arange(0, sysm.order, 8), np.arange(1, sysm.order, 8)]))
    idx = idx[rtan._stride_order(idx.size)]
    conds = [sysm.condition(r, int(k)) for k in idx for r in range(sysm.rows)]
    basis, deferred = rtan.serial_tan_int(conds, ts)
    np.savez_compressed(os.path.join(STAGE, "leaf_c1_first.npz"),
                        weights=sysm.weights, order=sysm.order, tau=sysm.tau,
                        basis=basis.coeffs, degs=ts.col_degrees,
                        deferred=len(deferred))


if __name__ == "__main__":
    which = sys.argv[1:] or ["solves", "stages"]
    if "stages" in which:
        stages()
    if "solves" in which:
        solves()
