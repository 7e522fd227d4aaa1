"""The CPU oracle against the reference's own outputs (golden fixtures made
by tests/golden/make_golden.py from /root/reference), the reference tests'
known answers, and the extension-size hand traces."""

import glob
import os

import numpy as np
import pytest

import toepreg_oracle as O
from conftest import GOLDEN, case_paths, decisions_robust, load_case, rel
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl

SMALL = [p for p in case_paths() if "full" not in os.path.basename(p)]


@pytest.mark.parametrize("path", SMALL, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_reproduces_reference_bitwise(path):
    raw, d = load_case(path)
    fill = str(d["cfg_fill"]) if "cfg_fill" in d else "auto"
    r = O.solve(wl.to_problem(raw, tb), fill=fill)
    assert np.array_equal(r["x_hat"], d["x_hat"])
    assert np.array_equal(r["final_col_degrees"], d["final_col_degrees"])
    dg = r["diagnostics"]
    assert dg["difficult_points"] == int(d["difficult_points"])
    assert dg["recursion_depth"] == int(d["recursion_depth"])
    assert dg["conditions_total"] == int(d["conditions_total"])
    assert dg["max_column_scale"] == float(d["max_column_scale"])
    assert r["relative_residual"] == float(d["relative_residual"])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2_full_rhs0"])
def test_oracle_reproduces_reference_full_size(name):
    raw, d = load_case(os.path.join(GOLDEN, "cases", name + ".npz"))
    r = O.solve(wl.to_problem(raw, tb))
    assert np.array_equal(r["x_hat"], d["x_hat"])


def test_known_answers():
    # identity T = L = I -> x = b / 2 (ref tests/test_solver.py:48-54)
    b = np.array([4.0, 8.0, 12.0, 16.0])
    p = tb.ProblemSpec.general(tb.identity_spec(4), tb.identity_spec(4), b)
    assert np.allclose(O.solve(p)["x_hat"], b / 2, atol=1e-12)
    # (4 + 1) x = 2 * 10 -> 4 (ref :57-61)
    p = tb.ProblemSpec.l2(tb.ToeplitzSpec(1, 1, np.array([2.0])), 1.0, [10.0])
    assert np.allclose(O.solve(p)["x_hat"], [4.0], atol=1e-12)


def test_extension_hand_traces():
    # ref tests/test_extension.py:34-45
    assert O.extend_detail(1000, 256, rows=3, paired=False, force_even=False) == (8, 4, 63)
    assert O.extend_detail(128, 256, rows=3, paired=False) == (0, 1, 64)
    k1, p1, _ = O.extend_detail(512, 256, rows=2, paired=False)
    k2, p2, _ = O.extend_detail(512, 256, rows=2, paired=True)
    assert p2 == p1 + 1 and k1 == k2 == 0
    with pytest.raises(ValueError):
        O.extend_detail(0, 256)
    with pytest.raises(ValueError):
        O.extend_detail(100, 2, rows=3)


def test_stage_grid_eval_matches_reference():
    g = np.load(os.path.join(GOLDEN, "stages", "grid_eval.npz"))
    for key in g.files:
        if key.startswith("N"):
            N, off, st = [int(s[1:]) for s in key.split("_")]
            assert np.array_equal(O.grid_eval(g["cube"], N, off, st), g[key])


def test_stage_matpoly_matches_reference():
    m = np.load(os.path.join(GOLDEN, "stages", "matpoly.npz"))
    assert np.array_equal(O.matpoly_product(m["a"], m["b"], extended=True), m["ld"])
    assert np.array_equal(O.matpoly_product(m["a"], m["b"], extended=False), m["f64"])


@pytest.mark.parametrize("name", ["assemble_l2_n64", "assemble_general_n32", "assemble_gramian_n32"])
def test_stage_assembly_matches_reference(name):
    a = dict(np.load(os.path.join(GOLDEN, "stages", name + ".npz")))
    variant = name.split("_")[1]
    n = 64 if variant == "l2" else 32
    raw = {"variant": variant, "m": n, "n": n}
    for k in ("T_gen", "L_gen", "G_col", "b", "normal_rhs"):
        if k in a:
            raw[k] = a[k]
    if "beta" in a:
        raw["beta"] = float(a["beta"])
    if "L_rows" in a:
        raw["L_rows"] = int(a["L_rows"])
    asm = O.assemble(wl.to_problem(raw, tb))
    assert asm.order == int(a["order"])
    assert np.array_equal(asm.tau, a["tau"])
    assert np.array_equal(asm.weights, a["weights"])


def test_stage_serial_leaf_matches_reference():
    f = np.load(os.path.join(GOLDEN, "stages", "leaf_c1_first.npz"))
    W, order = f["weights"], int(f["order"])
    nodes = O.unit_roots(order)
    idx = np.sort(np.concatenate([np.arange(0, order, 8), np.arange(1, order, 8)]))
    idx = idx[(np.arange(idx.size) * O.golden_stride(idx.size)) % idx.size]
    rows, _, p = W.shape
    wrows = W[:, idx, :].swapaxes(0, 1).reshape(idx.size * rows, -1)
    z = np.repeat(nodes[idx], rows)
    refs = [(int(k), r) for k in idx for r in range(rows)]
    cube = np.zeros((p, p, z.size + 1), dtype=np.complex128)
    cube[:, :, 0] = np.eye(p)
    degs = -f["tau"].copy()
    length, deferred = O.sweep(cube, 1, z, wrows, refs, degs, 1e-8, True, {"scale": 1.0})
    basis = cube[:, :, :length].copy()
    O.normalize_columns(basis)
    assert len(deferred) == int(f["deferred"])
    assert np.array_equal(degs, f["degs"])
    assert np.array_equal(basis, f["basis"])


def test_oracle_matches_dense_and_cg_exact():
    raw, d = load_case(os.path.join(GOLDEN, "cases", "rand512_l2.npz"))
    p = wl.to_problem(raw, tb)
    x = O.dense_solution(p)
    assert rel(x, d["x_exact"]) < 1e-12
    xc = O.cg_exact(p, tol=1e-14)
    assert rel(xc, x) < 1e-11


CG_CASES = sorted(glob.glob(os.path.join(GOLDEN, "stages", "cg_*_n96.npz")))


def _cg_problem(path, mod):
    from paper_1302_6945_b200 import workloads as wl
    d = dict(np.load(path))
    raw = {k: (v.item() if v.ndim == 0 else v) for k, v in d.items()}
    raw["variant"] = str(d["variant"])
    return wl.to_problem(raw, mod), d


@pytest.mark.parametrize("path", CG_CASES, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_normal_operator_and_cg_match_reference(path):
    """Oracle NormalOperator.apply and cg_solve against the reference's own
    outputs (tests/golden/make_golden_cg.py): same iteration counts."""
    import paper_1302_6945_b200 as tb
    prob, d = _cg_problem(path, tb)
    assert rel(O.normal_apply(prob, d["x"]), d["ax"]) < 1e-13
    x, it = O.cg_solve(prob)
    assert it == int(d["it_cg"])
    assert rel(x, d["x_cg"]) < 1e-12
    x5, it5 = O.cg_solve(prob, max_iterations=5)
    assert it5 == int(d["it_cg5"]) == 5
    assert rel(x5, d["x_cg5"]) < 1e-12


def test_oracle_nufft_setup_matches_reference():
    """Gramian column, samples and rhs of the NUFFT setup against the
    reference (tests/golden/make_golden_nufft.py); host helpers identical."""
    from paper_1302_6945_b200 import nufft as nf
    g = np.load(os.path.join(GOLDEN, "stages", "nufft.npz"))
    assert rel(O.nufft_gramian_col(g["freqs"], g["weights"], 256), g["gram"]) < 1e-14
    s, r = O.nufft_samples_and_rhs(g["freqs"], g["weights"], g["x"])
    assert rel(s, g["samples"]) < 1e-14 and rel(r, g["rhs"]) < 1e-14
    assert np.array_equal(nf.voronoi_weights(g["freqs"]), g["weights"])
    rng = np.random.default_rng(np.random.SeedSequence((7, 93)))
    rng.triangular(-0.5, 0.0, 0.5, size=300)
    assert np.array_equal(nf.make_signal(256, 3, 0.02, rng), g["x"])
    reg = nf.second_difference_regularizer(5, 2.0)
    assert reg.gen[4] == 4.0 and reg.gen[3] == -2.0 and reg.gen[5] == -2.0


def test_fixture_decision_margins_recorded():
    """Every fixture carries the reference's decision margins
    (tests/golden/add_margins.py); most are robust, so the GPU tests compare
    their degree ledgers position by position."""
    cases = case_paths()
    for p in cases:
        d = dict(np.load(p))
        for key in ("margin_pivot", "margin_defer", "margin_check", "spread_exact"):
            assert key in d, (p, key)
    robust = [decisions_robust(dict(np.load(p))) for p in cases]
    assert sum(robust) >= 0.6 * len(cases), sum(robust)
