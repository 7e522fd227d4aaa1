"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs, the oracle, and exact solutions.

Tolerances (relative 2-norm unless stated):
  * accuracy default (SolverConfig.refine=1): GPU <-> exact <= 1e-12 on
    well-conditioned fixtures (reference <-> exact <= 1e-9), hence
    GPU <-> reference == reference <-> exact <= 1e-9; never farther from the
    exact solution than the reference itself.
  * single pass (refine=0, the reference's own algorithm): within 6x the
    reference's distance to the exact solution, or of that distance under a
    rounding change of the reference (an FP64 leaf lands
    at ~sqrt(2) x the reference's floor; measured <= 3x on most fixtures).
  * integer outputs: recursion depth and condition count exact; degree
    ledger and deferred count exact wherever the reference's decisions are
    robust to rounding (conftest.decisions_robust), a valid final profile
    elsewhere; no truncated products.
  * ill-conditioned fixtures where the reference itself fails (ILL): no
    exception, residual no worse than the reference's.
"""

import ctypes as C
import glob
import os

import numpy as np
import pytest

import toepreg_oracle as O
from conftest import GOLDEN, case_config, case_paths, decisions_robust, load_case, rel
from paper_1302_6945_b200 import workloads as wl

pytestmark = pytest.mark.gpu

CASES = case_paths()
# the reference itself fails on these (cond ~ 1e8 .. 7e8): its normal residual
# is 1e-2 .. 0.24, so only "no exception, residual no worse" is meaningful
ILL = ("c4_mini", "c4_full")


def _solve(tb, raw, refine, d=None):
    cfg = case_config(tb, d, refine) if d is not None else tb.SolverConfig(refine=refine)
    return tb.solve_tikhonov(wl.to_problem(raw, tb), cfg)


def _integers_exact(rep, d, name):
    """Integer outputs of the direct solve: the recursion depth and condition
    count always equal the reference's, and no product was truncated.  Where
    the reference's decisions are robust to rounding (decisions_robust) the
    degree ledger (position by position) and the deferred count are equal
    too; elsewhere (a leaf self-check within a factor of 3 of its 1e-11
    tolerance retries on one side only, etc.) the ledger is still a valid
    final profile: one column of degree 0, the others 1."""
    assert rep.diagnostics.recursion_depth == int(d["recursion_depth"]), name
    assert rep.diagnostics.conditions_total == int(d["conditions_total"]), name
    assert rep.diagnostics.trim_overflow == 0, name
    if decisions_robust(d):
        assert np.array_equal(rep.final_col_degrees, d["final_col_degrees"]), \
            (name, rep.final_col_degrees, d["final_col_degrees"])
        assert rep.diagnostics.difficult_points == int(d["difficult_points"]), name
    else:
        assert sorted(rep.final_col_degrees.tolist()) == sorted(d["final_col_degrees"].tolist()), name


@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[:-4])
def test_parity_with_reference_refined(gpu, path):
    tb = gpu
    raw, d = load_case(path)
    name = os.path.basename(path)[:-4]
    rep = _solve(tb, raw, 1, d)
    ref_exact = rel(d["x_hat"], d["x_exact"])
    gpu_exact = rel(rep.x_hat, d["x_exact"])
    gpu_ref = rel(rep.x_hat, d["x_hat"])
    assert rep.x_hat.dtype == np.complex128 and rep.x_hat.shape == d["x_hat"].shape
    assert np.all(np.isfinite(rep.x_hat))
    assert rep.relative_residual <= float(d["relative_residual"]) * 1.0001 + 1e-13, \
        (name, rep.relative_residual, float(d["relative_residual"]))
    if name in ILL:
        # the reference's integer decisions here are chaotic (its own ledger
        # and deferral count change under a rounding change: add_margins.py)
        # the FP64 direct solve fails here (the reference's long-double tree
        # products are what keep its own direct solve from failing, App. B):
        # x must come from the CG rescue, closer to the exact solution than 0
        assert rep.diagnostics.rescued or rep.diagnostics.trim_overflow == 0
        assert gpu_exact < 1.0, (name, gpu_exact)
        return
    _integers_exact(rep, d, name)
    assert gpu_exact <= ref_exact * 1.0001 + 1e-15, (name, gpu_exact, ref_exact)
    if ref_exact <= 1e-9:
        assert gpu_exact <= 1e-12, (name, gpu_exact)
        assert gpu_ref <= 1e-9, (name, gpu_ref)
        assert rep.relative_residual <= 1e-12


@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[:-4])
def test_single_pass_matches_reference_error_level(gpu, path):
    tb = gpu
    raw, d = load_case(path)
    name = os.path.basename(path)[:-4]
    if name in ILL:
        pytest.skip("reference fails on this conditioning; see the refined test")
    rep = _solve(tb, raw, 0, d)
    ref_exact = rel(d["x_hat"], d["x_exact"])
    # the reference's own error moves under a rounding change (spread_exact:
    # its algorithm with float64 tree products); a single FP64
    # pass (float64 leaves AND products) lands within 6x of the larger of the
    # two (measured: <= 3x on 61 of 64 fixtures, 3-5x on c3 lambda=1e-2,
    # ext_general_k24, ext_l2_k1_echo)
    floor = max(ref_exact, float(d["spread_exact"]))
    assert rel(rep.x_hat, d["x_exact"]) <= 6 * floor + 1e-13, (name, rel(rep.x_hat, d["x_exact"]), floor)
    _integers_exact(rep, d, name)
    assert rep.relative_residual <= 6 * max(float(d["relative_residual"]), floor) + 1e-14


def test_known_answers(gpu):
    tb = gpu
    b = np.array([4.0, 8.0, 12.0, 16.0])
    p = tb.ProblemSpec.general(tb.identity_spec(4), tb.identity_spec(4), b)
    assert np.allclose(tb.solve_tikhonov(p).x_hat, b / 2, atol=1e-12)
    p = tb.ProblemSpec.l2(tb.ToeplitzSpec(1, 1, np.array([2.0])), 1.0, [10.0])
    assert np.allclose(tb.solve_tikhonov(p).x_hat, [4.0], atol=1e-12)
    # zero right-hand side -> zero solution
    p = tb.ProblemSpec.l2(tb.ToeplitzSpec(4, 4, np.arange(1, 8.0)), 1.0, np.zeros(4))
    r = tb.solve_tikhonov(p)
    assert not r.x_hat.any() and r.relative_residual == 0.0


def test_singular_system_raises(gpu):
    tb = gpu
    z = np.zeros(7)
    p = tb.ProblemSpec.general(tb.ToeplitzSpec(4, 4, z), tb.ToeplitzSpec(4, 4, z), np.ones(4))
    with pytest.raises(tb.SingularSystemError):
        tb.solve_tikhonov(p)


def test_deterministic_and_batch_invariant(gpu):
    tb = gpu
    raw = wl.c5_random(n=1024, count=5, seed=11)
    probs = [wl.to_problem(raw, tb, i) for i in range(5)]
    a = tb.solve_tikhonov_batch(probs)
    b = tb.solve_tikhonov_batch(probs)
    c = tb.solve_tikhonov(probs[3])
    assert all(np.array_equal(x.x_hat, y.x_hat) for x, y in zip(a, b))
    assert np.array_equal(a[3].x_hat, c.x_hat)


def test_shared_operator_batch(gpu):
    tb = gpu
    raw = wl.c2_rect(m=1024, n=512, nrhs=6, seed=3)
    probs = [wl.to_problem(raw, tb, i) for i in range(6)]
    reps = tb.solve_tikhonov_batch(probs)
    for i, r in enumerate(reps):
        single = tb.solve_tikhonov(probs[i])
        assert np.array_equal(r.x_hat, single.x_hat)
        x = O.dense_solution(probs[i])
        assert rel(r.x_hat, x) < 1e-12


@pytest.mark.parametrize("count", [40, 300])
def test_batch_groups_invariant(gpu, count):
    """Batches split into 2-4 stream groups (>= 32 systems), with the leaf
    attempts paired in 2-CTA clusters (40: 20 systems per group) and
    unpaired (300: 3 groups of 100, 200 CTAs > 148 SMs), give bit-identical
    solutions to one-system solves, and match the dense solution."""
    tb = gpu
    raw = wl.c5_random(n=256, count=count, seed=29)
    probs = [wl.to_problem(raw, tb, i) for i in range(count)]
    reps = tb.solve_tikhonov_batch(probs)
    for i in sorted({0, 1, count // 4, count // 2 - 1, count // 2, count - 1}):
        single = tb.solve_tikhonov(probs[i])
        assert np.array_equal(reps[i].x_hat, single.x_hat), i
        assert np.array_equal(reps[i].final_col_degrees, single.final_col_degrees)
        assert rel(reps[i].x_hat, O.dense_solution(probs[i])) < 1e-10


def test_split_leaf_path_bit_identical_to_fused(gpu):
    """More than 8 x 148 systems: the groups no longer fit one CTA per SM and
    the leaves run the split path (chain kernel + row-parallel basis kernel,
    leaf_fast.cu).  Its multipliers mu_i = f_i c_i are formed by the same
    pinned rounding sequence as the fused kernel's mu warp (cmul_mu), so a
    system's solution does not depend on the batch it is solved in."""
    tb = gpu
    count = 1300
    raw = wl.c5_random(n=64, count=count, seed=31)
    probs = [wl.to_problem(raw, tb, i) for i in range(count)]
    reps = tb.solve_tikhonov_batch(probs)
    for i in (0, 1, 647, 1299):
        single = tb.solve_tikhonov(probs[i])
        assert np.array_equal(reps[i].x_hat, single.x_hat), i
        assert np.array_equal(reps[i].final_col_degrees, single.final_col_degrees)
        assert rel(reps[i].x_hat, O.dense_solution(probs[i])) < 1e-10


def test_shared_operator_groups(gpu):
    """Config-2 shape (one T, many right-hand sides) across stream groups."""
    tb = gpu
    raw = wl.c2_rect(m=1024, n=512, nrhs=40, seed=8)
    probs = [wl.to_problem(raw, tb, i) for i in range(40)]
    reps = tb.solve_tikhonov_batch(probs)
    for i in (0, 19, 20, 39):
        assert np.array_equal(reps[i].x_hat, tb.solve_tikhonov(probs[i]).x_hat), i
        assert rel(reps[i].x_hat, O.dense_solution(probs[i])) < 1e-12


@pytest.mark.parametrize("variant", ["general", "l2", "gramian"])
def test_small_corpus_against_dense(gpu, variant):
    """The reference acceptance gate (ref tests/test_acceptance.py:107-113):
    < 1e-8 vs dense for n in {4..64}."""
    tb = gpu
    code = {"general": 0, "l2": 1, "gramian": 2}[variant]
    for n in (4, 8, 16, 32, 64):
        for trial in range(4):
            rng = np.random.default_rng(np.random.SeedSequence((8801, code, n, trial)))
            raw = wl.random_problem(variant, n, rng)
            for refine in (0, 1):
                rep = _solve(tb, raw, refine)
                x = O.dense_solution(wl.to_problem(raw, tb))
                assert rel(rep.x_hat, x) < 1e-8
                assert sorted(rep.final_col_degrees.tolist()) == [0] + [1] * (rep.final_col_degrees.size - 1)


@pytest.mark.parametrize("variant", ["general", "l2", "gramian"])
def test_planted_solution_n512(gpu, variant):
    """ref tests/test_acceptance.py:116-122: max-abs < 1e-9 at n = 512."""
    tb = gpu
    rng = np.random.default_rng(np.random.SeedSequence((2024, 7, 512)))
    raw = wl.random_problem(variant, 512, rng)
    base = wl.to_problem(raw, tb)
    x_true = (rng.standard_normal(512) + 1j * rng.standard_normal(512)) / np.sqrt(2.0)
    y = O.normal_apply(base, x_true)
    planted = tb.ProblemSpec(variant=variant, T=base.T, L=base.L, G=base.G, beta=base.beta,
                             b=None, normal_rhs=y)
    for refine in (0, 1):
        rep = tb.solve_tikhonov(planted, tb.SolverConfig(refine=refine))
        assert np.abs(rep.x_hat - x_true).max() < 1e-9


def test_full_size_c5_properties(gpu):
    """Size-independent checks at BASELINE config-5 size (n = 16384)."""
    tb = gpu
    raw = wl.c5_random(n=16384, count=3, seed=5)
    probs = [wl.to_problem(raw, tb, i) for i in range(3)]
    reps = tb.solve_tikhonov_batch(probs)
    for p, r in zip(probs, reps):
        assert r.relative_residual < 1e-13
        assert sorted(r.final_col_degrees.tolist()) == [0, 1, 1, 1, 1]
        # residual recomputed independently on the CPU
        res = np.linalg.norm(O.normal_apply(p, r.x_hat) - O.normal_rhs(p))
        assert res / np.linalg.norm(O.normal_rhs(p)) < 1e-12


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128).view(np.float64).copy()).cuda()


def test_stage_fft_against_numpy(gpu):
    import torch
    from paper_1302_6945_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(0)
    for n in (1, 2, 3, 48, 64, 96, 1024, 12288, 32768, 98304, 1 << 20, 3 << 18, 1 << 21):
        lines = max(1, min(4, (1 << 21) // n))
        x = rng.standard_normal((lines, n)) + 1j * rng.standard_normal((lines, n))
        dx = _dev(x)
        out = torch.empty_like(dx)
        for sign in (-1, 1):
            assert lib.tr_fft(C.c_void_p(dx.data_ptr()), C.c_void_p(out.data_ptr()), n, lines, sign, None) == 0
            got = out.cpu().numpy().view(np.complex128).reshape(lines, n)
            ref = np.fft.fft(x, axis=-1) if sign < 0 else n * np.fft.ifft(x, axis=-1)
            assert rel(got, ref) < 2e-15 * np.log2(max(n, 2))


def test_stage_grid_eval_and_product(gpu):
    import torch
    from paper_1302_6945_b200 import _lib
    lib = _lib.load()
    g = np.load(os.path.join(GOLDEN, "stages", "grid_eval.npz"))
    cube = g["cube"]
    lines = cube.shape[0] * cube.shape[1]
    src = _dev(cube.reshape(lines, -1))
    for key in g.files:
        if not key.startswith("N"):
            continue
        N, off, st = [int(s[1:]) for s in key.split("_")]
        out = torch.empty((lines, N // st, 2), dtype=torch.float64, device="cuda")
        assert lib.tr_grid_eval(C.c_void_p(src.data_ptr()), lines, cube.shape[2], N, off, st,
                                C.c_void_p(out.data_ptr()), None) == 0
        got = out.cpu().numpy().view(np.complex128).reshape(g[key].shape)
        assert rel(got, g[key]) < 1e-14
    m = np.load(os.path.join(GOLDEN, "stages", "matpoly.npz"))
    a, b = _dev(m["a"]), _dev(m["b"])
    L = m["a"].shape[2] + m["b"].shape[2] - 1
    out = torch.empty((25, L, 2), dtype=torch.float64, device="cuda")
    assert lib.tr_matpoly_mul(C.c_void_p(a.data_ptr()), m["a"].shape[2], C.c_void_p(b.data_ptr()),
                              m["b"].shape[2], 5, C.c_void_p(out.data_ptr()), None) == 0
    got = out.cpu().numpy().view(np.complex128).reshape(5, 5, L)
    # the reference product is long double; FP64 FFT products carry eps*log(R) error
    assert np.abs(got - m["ld"]).max() / np.abs(m["ld"]).max() < 1e-14


@pytest.mark.parametrize("name", ["assemble_l2_n64", "assemble_general_n32", "assemble_gramian_n32"])
def test_stage_assembly(gpu, name):
    import torch
    tb = gpu
    from paper_1302_6945_b200 import _lib
    lib = _lib.load()
    a = dict(np.load(os.path.join(GOLDEN, "stages", name + ".npz")))
    W = a["weights"]
    rows, N, P = W.shape
    variant = name.split("_")[1]
    n = 64 if variant == "l2" else 32
    pl = int(a.get("L_rows", n))
    d = tb.solver.make_desc(variant, n, n, pl, tb.SolverConfig())
    out = torch.zeros((N, rows, P, 2), dtype=torch.float64, device="cuda")
    keep = {}
    def ptr(key):
        if key not in a:
            return None
        keep[key] = _dev(a[key])
        return C.c_void_p(keep[key].data_ptr())
    bsq = None
    if "beta" in a:
        keep["beta"] = torch.tensor([abs(float(a["beta"])) ** 2], dtype=torch.float64, device="cuda")
        bsq = C.c_void_p(keep["beta"].data_ptr())
    rhs = ptr("normal_rhs") if "normal_rhs" in a else ptr("b")
    assert lib.tr_assemble(C.byref(d), ptr("T_gen"), ptr("L_gen"), ptr("G_col"), bsq, rhs,
                           int("normal_rhs" in a), C.c_void_p(out.data_ptr()), None) == 0
    got = np.transpose(out.cpu().numpy().view(np.complex128).reshape(N, rows, P), (1, 0, 2))
    assert np.abs(got - W).max() <= 1e-12 * max(1.0, np.abs(W).max())


@pytest.mark.parametrize("label", ["c1", "c2", "c3", "general64"])
def test_stage_leaf_against_oracle(gpu, label):
    """The first leaf (weights from the oracle's assembly) vs the oracle's
    serial leaf: same degree ledger and deferrals, basis within FP64 sweep
    noise."""
    import torch
    tb = gpu
    from paper_1302_6945_b200 import _lib
    lib = _lib.load()
    raw = {"c1": lambda: wl.c1_blur(256),
           "c2": lambda: wl.c2_rect(m=1024, n=512, nrhs=1),
           "c3": lambda: wl.c3_firstdiff(n=512, lam=1e-2),
           "general64": lambda: wl.random_problem("general", 64, np.random.default_rng(5))}[label]()
    idx0 = 0 if np.asarray(raw.get("b", [0])).ndim == 2 else None
    prob = wl.to_problem(raw, tb, idx0)
    asm = O.assemble(prob)
    v, m, n, pl = tb.solver._shape(prob)
    d = tb.solver.make_desc(v, m, n, pl, tb.SolverConfig())
    W = asm.weights
    rows, N, P = W.shape
    offsets, stride = (0,), 1
    while rows * len(offsets) * (N // stride) > 256:
        offsets, _, stride = O.split_rule(N, offsets, stride, True)
    idx = O.coset_indices(N, offsets, stride)
    K = rows * idx.size
    degs = -asm.tau.copy()
    coeffs, d_ref, deferred, _, _, _ = O.leaf_basis(W, asm.nodes, idx, degs.copy(), 1e-8)
    Wd = _dev(np.transpose(W, (1, 0, 2)))
    cd = (C.c_int64 * 8)(*([int(x) for x in degs] + [0] * (8 - P)))
    out = torch.zeros((P * P * (K + 1) * 2,), dtype=torch.float64, device="cuda")
    nd, att = C.c_int32(), C.c_int32()
    rr = C.c_double()
    assert lib.tr_leaf(C.byref(d), C.c_void_p(Wd.data_ptr()), 0, cd, C.c_void_p(out.data_ptr()),
                       K + 1, C.byref(nd), C.byref(rr), C.byref(att), None) == 0
    g = out.cpu().numpy().view(np.complex128).reshape(P, P, K + 1)
    assert list(cd)[:P] == [int(x) for x in d_ref]
    assert nd.value == len(deferred)
    L = coeffs.shape[2]
    assert np.abs(g[:, :, :L] - coeffs).max() <= 1e-9 * np.abs(coeffs).max()
    assert rr.value < 1e-11


CG_CASES = sorted(glob.glob(os.path.join(GOLDEN, "stages", "cg_*_n96.npz")))


def _cg_problem(tb, path):
    d = dict(np.load(path))
    raw = {k: (v.item() if v.ndim == 0 else v) for k, v in d.items()}
    raw["variant"] = str(d["variant"])
    return wl.to_problem(raw, tb), d


@pytest.mark.parametrize("path", CG_CASES, ids=lambda p: os.path.basename(p)[:-4])
def test_normal_operator_matches_reference(gpu, path):
    tb = gpu
    prob, d = _cg_problem(tb, path)
    op = tb.NormalOperator(prob)
    assert rel(op.apply(d["x"]), d["ax"]) < 1e-12
    assert op.transforms == int(d["transforms"])
    assert rel(tb.apply_normal_operator(prob, d["x"]), d["ax"]) < 1e-12


@pytest.mark.parametrize("path", CG_CASES, ids=lambda p: os.path.basename(p)[:-4])
def test_cg_matches_reference(gpu, path):
    """GPU CG against the reference's cg_solve: the same stopping rule, so the
    iteration count agrees up to rounding (+-2) and x to the CG tolerance."""
    tb = gpu
    prob, d = _cg_problem(tb, path)
    x, it = tb.cg_solve(prob)
    assert abs(it - int(d["it_cg"])) <= 2, (it, int(d["it_cg"]))
    assert rel(x, d["x_cg"]) < 1e-9
    x5, it5 = tb.cg_solve(prob, tb.CGConfig(max_iterations=5))
    assert it5 == 5
    assert rel(x5, d["x_cg5"]) < 1e-10
    op = tb.NormalOperator(prob)
    _, it_op = tb.cg_solve(prob, tb.CGConfig(max_iterations=3), operator=op)
    assert it_op == 3 and op.transforms == 3 * int(d["transforms"])


def test_cg_edge_cases(gpu):
    tb = gpu
    rng = np.random.default_rng(5)
    raw = wl.random_problem("l2", 64, rng)
    raw["b"] = np.zeros_like(raw["b"])
    x, it = tb.cg_solve(wl.to_problem(raw, tb))
    assert it == 0 and not np.any(x)
    raw = wl.random_problem("l2", 64, rng)
    x, it = tb.cg_solve(wl.to_problem(raw, tb), tb.CGConfig(time_budget=1e-9))
    assert it == 1  # the budget is checked after a completed iteration
    x, it = tb.cg_solve(wl.to_problem(raw, tb), tb.CGConfig(time_budget=0.0))
    assert it == 1  # a zero budget still runs one iteration (ref solver.py:211)
    # the operator applies to THIS problem's right-hand side (ref solver.py:181-215):
    # an operator of the same matrix built for another rhs gives the same result,
    # one of another matrix is refused
    mine = wl.to_problem(raw, tb)
    twin = dict(raw, b=np.asarray(raw["b"]) * 2.0)
    xa, ita = tb.cg_solve(mine, tb.CGConfig(max_iterations=7), operator=tb.NormalOperator(wl.to_problem(twin, tb)))
    xb, itb = tb.cg_solve(mine, tb.CGConfig(max_iterations=7))
    assert ita == itb == 7 and np.array_equal(xa, xb)
    other = wl.to_problem(wl.random_problem("l2", 64, rng), tb)
    with pytest.raises(ValueError):
        tb.cg_solve(mine, operator=tb.NormalOperator(other))
    x, it = tb.cg_solve(wl.to_problem(raw, tb), tb.CGConfig(max_iterations=0))
    assert it == 0


def test_cg_batch_per_system_stopping(gpu):
    tb = gpu
    raw = wl.c5_random(n=512, count=4, seed=3)
    probs = [wl.to_problem(raw, tb, i) for i in range(4)]
    out = tb.cg_solve_batch(probs)
    for p, (x, it) in zip(probs, out):
        xo, ito = O.cg_solve(p)
        assert abs(it - ito) <= 2
        assert rel(x, xo) < 1e-9
        assert rel(x, tb.solve_tikhonov(p).x_hat) < 1e-9


def test_cg_full_size_c5_agrees_with_direct_solve(gpu):
    tb = gpu
    raw = wl.c5_random(n=16384, count=1, seed=0)
    p = wl.to_problem(raw, tb, 0)
    x, it = tb.cg_solve(p)
    assert 0 < it < 10 * 16384
    assert rel(x, tb.solve_tikhonov(p).x_hat) < 1e-9


def test_nufft_setup_matches_reference(gpu):
    from paper_1302_6945_b200 import nufft as nf
    g = np.load(os.path.join(GOLDEN, "stages", "nufft.npz"))
    col = nf.weighted_fourier_gramian(g["freqs"], g["weights"], 256).gen
    assert rel(col, g["gram"]) < 1e-12
    big = nf.weighted_fourier_gramian(g["freqs"][:64], g["weights"][:64], 20000).gen
    assert rel(big, g["gram_big"]) < 1e-10  # phases up to 2 pi 0.5 2e4: reference rounding ~1e-12
    assert rel(nf.nufft_samples(g["freqs"], g["x"]), g["samples"]) < 1e-12
    assert rel(nf.nufft_normal_rhs(g["freqs"], g["weights"] * g["samples"], 256), g["rhs"]) < 1e-12
    # against the oracle at the c4 shape ratio (K = n / 2)
    rng = np.random.default_rng(11)
    f = rng.uniform(0.0, 1.0, 512)
    b = rng.standard_normal(512) + 1j * rng.standard_normal(512)
    assert rel(nf.nufft_normal_rhs(f, b, 1024), np.exp(2j * np.pi * np.outer(np.arange(1024), f)) @ b) < 1e-12
    assert rel(nf.weighted_fourier_gramian(f, np.abs(b), 1024).gen, O.nufft_gramian_col(f, np.abs(b), 1024)) < 1e-12


def test_run_nufft_matches_reference(gpu):
    from paper_1302_6945_b200 import nufft as nf
    g = np.load(os.path.join(GOLDEN, "stages", "nufft.npz"))
    out = nf.run_nufft(nf.NufftConfig(n=256, samples=320))
    assert out["weights_sum"] == float(g["run_wsum"])
    assert out["difficult_points"] == int(g["run_dp"])
    x = np.array(out["x_direct_re"]) + 1j * np.array(out["x_direct_im"])
    # the regularised problem is ill-conditioned (reg_scale 1e-4): judge both
    # solves against the exact solution of the same problem (dense oracle)
    rng = np.random.default_rng(np.random.SeedSequence((0, 93)))
    f = rng.triangular(-0.5, 0.0, 0.5, size=320)
    w = nf.voronoi_weights(f)
    xt = nf.make_signal(256, 3, 0.02, rng)
    _, rhs = O.nufft_samples_and_rhs(f, w, xt)
    prob = gpu.ProblemSpec.gramian(gpu.HermitianToeplitzSpec(256, O.nufft_gramian_col(f, w, 256)),
                                   nf.second_difference_regularizer(256, 1e-4), rhs)
    exact = O.dense_solution(prob)
    assert rel(x, exact) <= rel(g["run_x"], exact) * 1.01 + 1e-12
    assert out["rel_err_direct"] <= float(g["run_err"]) * 1.01
    assert out["cg_iterations"] >= 1 and out["rel_residual_direct"] < 1e-6


@pytest.mark.parametrize("name", ["c2_mini_rhs0", "c5_mini_sys0", "rand512_general", "c3_mini_lam0.01"])
def test_direct_refinement_path(gpu, name):
    """refine_cg=0: refinement by a second superfast solve (the path CG
    falls back to) reaches the same accuracy as the CG refinement."""
    tb = gpu
    raw, d = load_case(os.path.join(GOLDEN, "cases", name + ".npz"))
    prob = wl.to_problem(raw, tb)
    a = tb.solve_tikhonov(prob, tb.SolverConfig(refine=1, refine_cg=0)).x_hat
    b = tb.solve_tikhonov(prob, tb.SolverConfig(refine=1)).x_hat
    ex = d["x_exact"]
    ra, rb = rel(a, ex), rel(b, ex)
    assert ra < 1e-11 and rb < 1e-11, (ra, rb)


def test_run_accuracy_matches_reference(gpu):
    """GPU run_accuracy on the reference's seeded cells: same rows, errors at
    least as small as the reference's (refinement) and tiny in absolute terms."""
    import json
    from paper_1302_6945_b200 import experiments as ex
    g = json.load(open(os.path.join(GOLDEN, "stages", "experiments.json")))
    rows = ex.run_accuracy(ex.ExperimentConfig(sizes=(16, 32), trials=2, seed=2024))
    assert [(r["variant"], r["n"]) for r in rows] == [(r["variant"], r["n"]) for r in g["accuracy"]]
    for ours, ref in zip(rows, g["accuracy"]):
        assert ours["max_err"] <= max(ref["max_err"], 1e-12), (ours, ref)


def test_run_cg_equivalence_and_complexity_rows(gpu):
    from paper_1302_6945_b200 import experiments as ex
    cfg = ex.ExperimentConfig(variants=("l2",), sizes=(64, 128), trials=1)
    rows = ex.run_cg_equivalence(cfg)
    assert len(rows) == 2 and all(r["mean_iters"] >= 1 and r["direct_max_err"] < 1e-9 for r in rows)
    rows, fits = ex.run_complexity(cfg)
    assert len(rows) == 2 and rows[0]["params"] == 127 and "l2" in fits


def test_reference_five_field_config_accepted(gpu):
    """The reference's SolverConfig has five fields (ref solver.py:39-45);
    passing an object of exactly that shape works and equals refine=1."""
    import dataclasses
    tb = gpu

    @dataclasses.dataclass(frozen=True)
    class RefSolverConfig:  # stand-in with the reference's exact fields
        n_lim: int = 256
        pivot_threshold: float = 1e-8
        fill: str = "auto"
        paired: bool = True
        force_even: bool = True

    raw, d = load_case(os.path.join(GOLDEN, "cases", "c5_mini_sys0.npz"))
    prob = wl.to_problem(raw, tb)
    a = tb.solve_tikhonov(prob, RefSolverConfig())
    b = tb.solve_tikhonov(prob, tb.SolverConfig())
    c = tb.solve_tikhonov(prob)
    assert np.array_equal(a.x_hat, b.x_hat) and np.array_equal(a.x_hat, c.x_hat)
    assert np.array_equal(a.final_col_degrees, d["final_col_degrees"])
    info = tb.plan_info(prob, RefSolverConfig())
    assert info["order"] == 4096


def test_wall_time_covers_the_solve_only(gpu):
    """wall_time is the device time of assemble -> extract (+ refinement);
    it excludes staging, the copy back and the residual evaluation
    (ref solver.py:62-71) and is positive and below the host-observed time."""
    import time
    tb = gpu
    raw = wl.c5_random(n=2048, count=1, seed=2)
    prob = wl.to_problem(raw, tb, 0)
    tb.solve_tikhonov(prob)  # warm (plan, graph capture)
    t0 = time.perf_counter()
    rep = tb.solve_tikhonov(prob)
    host = time.perf_counter() - t0
    assert 0.0 < rep.wall_time < host


def test_host_abi_binding_from_integration_doc(gpu):
    """Run the ctypes binding exactly as INTEGRATION.md prints it (the block
    is extracted from the document and executed) on host buffers."""
    import re
    from conftest import ROOT
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"### ctypes binding a non-torch caller would use\s*```python\n(.*?)```", text, re.S)
    assert block, "INTEGRATION.md lost its ctypes example"
    code = block.group(1).replace('"paper_1302_6945_b200/libtoepreg_b200.so"',
                                  repr(os.path.join(ROOT, "paper_1302_6945_b200", "libtoepreg_b200.so")))
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)  # noqa: S102 (the documented binding)
    raw, d = load_case(os.path.join(GOLDEN, "cases", "c5_mini_sys0.npz"))
    x = ns["solve_l2_host"](raw["T_gen"], raw["beta"], raw["b"], int(raw["m"]), int(raw["n"]))
    tb = gpu
    ref = tb.solve_tikhonov(wl.to_problem(raw, tb)).x_hat
    assert np.array_equal(x, ref)
    assert rel(x, d["x_exact"]) < 1e-12


def test_full_size_c5b_single_system(gpu):
    """BASELINE config 5b: one l2 system of n = 2^22 (N = 2^23, 17 levels).
    Checked through size-independent properties: the normal-equation residual
    recomputed on the CPU by the oracle's FFT operator, the final degree
    ledger, and agreement with an independent GPU solve (conjugate gradients
    from zero to 1e-14)."""
    tb = gpu
    n = 1 << 22
    raw = wl.c5_random(n=n, count=1, seed=0)
    prob = wl.to_problem(raw, tb, 0)
    rep = tb.solve_tikhonov(prob)
    assert rep.diagnostics.trim_overflow == 0
    assert rep.diagnostics.conditions_total == 2 * 2 * n
    assert sorted(rep.final_col_degrees.tolist()) == [0, 1, 1, 1, 1]
    y = O.normal_rhs(prob)
    res = np.linalg.norm(O.normal_apply(prob, rep.x_hat) - y) / np.linalg.norm(y)
    assert res < 1e-11 and abs(res - rep.relative_residual) < 1e-12, (res, rep.relative_residual)
    x_cg, it = tb.cg_solve(prob, tb.CGConfig(tolerance=1e-14))
    assert 0 < it < 10 * n
    assert rel(rep.x_hat, x_cg) < 1e-10


def test_real_cg_refinement_matches_complex_path(gpu):
    """Real l2 data refines by CG on real vectors with half-length transforms
    (csrc/cg.cu pm_spectra_kernel; needs a two-pass half-length plan: c2's
    shape).  The same systems with one right-hand side entry carrying a 1e-300
    imaginary part take the complex path; both must agree to rounding, match
    the exact (dense) solution, and batch == single bit for bit."""
    tb = gpu
    raw = wl.c2_rect(m=8192, n=4096, nrhs=3, seed=5)
    probs = [wl.to_problem(raw, tb, i) for i in range(3)]
    reps = tb.solve_tikhonov_batch(probs)
    tagged = []
    for p in probs:
        b = np.array(p.b, dtype=np.complex128)
        b[0] += 1e-300j
        tagged.append(tb.ProblemSpec(variant="l2", T=p.T, beta=p.beta, b=b))
    reps_c = tb.solve_tikhonov_batch(tagged)
    single = tb.solve_tikhonov(probs[1])
    assert np.array_equal(single.x_hat, reps[1].x_hat)
    exact = O.dense_solution(probs[1])
    for r, rc in zip(reps, reps_c):
        assert r.diagnostics.refine_cg_iterations > 0 and rc.diagnostics.refine_cg_iterations > 0
        assert not r.x_hat.imag.any()          # real state: no imaginary rounding noise
        assert rel(r.x_hat, rc.x_hat) < 1e-13
        assert abs(r.diagnostics.refine_cg_iterations - rc.diagnostics.refine_cg_iterations) <= 2
    assert rel(reps[1].x_hat, exact) < 1e-12
    assert rel(reps_c[1].x_hat, exact) < 1e-12


@pytest.mark.parametrize("mode", ["1", "2"])
def test_fused_two_pass_fft_modes(gpu, mode):
    """The opt-in fused two-pass transform (csrc/fft_col.cu fft_col2_kernel:
    TR_FFT_C2 = 1 per-line clusters with the scratch-slot mailboxes, 2
    persistent clusters) against numpy-class accuracy, out of place / in place,
    both signs, line counts below and above the slot count.  The mode is read
    once per process, so each runs in its own."""
    import subprocess
    import sys
    from conftest import ROOT
    shapes = ["12288x40", "8192x100", "32768x90", "20480x33"]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fft_c2.py"), "child"] + shapes,
                         env=dict(os.environ, TR_FFT_C2=mode), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if " err " in l]
    assert len(lines) == len(shapes), out.stdout
    for l in lines:
        err = float(l.split(" err ")[1].split()[0])
        err2 = float(l.split("inplace/inv ")[1].split()[0])
        assert err < 5e-15 and err2 < 5e-15, l


_SPEC_CODE = r"""
import hashlib, sys
import numpy as np
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl
import toepreg_oracle as O
h = hashlib.sha1()
errs = []
for n, count, seed in ((4096, 3, 3), (256, 3, 7)):      # CG refinement / direct refinement
    raw = wl.c5_random(n=n, count=count, seed=seed)
    probs = [wl.to_problem(raw, tb, i) for i in range(count)]
    for p, r in zip(probs, tb.solve_tikhonov_batch(probs)):
        h.update(r.x_hat.tobytes())
        h.update(r.final_col_degrees.tobytes())
        if n == 256:
            x = O.dense_solution(p)
            errs.append(float(np.linalg.norm(r.x_hat - x) / np.linalg.norm(x)))
print(h.hexdigest(), max(errs))
"""


def test_speculative_direct_phase_reruns_with_the_exact_fallback(gpu):
    """The direct phase leaves the exact-fallback leaf launches out and runs
    again with them only when a leaf was handed over (csrc/solver.cu
    run_solve).  TR_TEST_VIOL makes system 0 hand a leaf over: the result must
    equal the non-speculative run (TR_SPEC_LEAF=0) bit for bit, with and
    without a hand-over, on the CG and the direct refinement paths."""
    import subprocess
    import sys
    from conftest import ROOT

    def go(**env):
        e = dict(os.environ, **env)
        e["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "oracle"), e.get("PYTHONPATH", "")])
        out = subprocess.run([sys.executable, "-c", _SPEC_CODE], env=e, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        digest, err = out.stdout.split()
        return digest, float(err)

    base_on, e1 = go(TR_SPEC_LEAF="1")
    base_off, e2 = go(TR_SPEC_LEAF="0")
    assert base_on == base_off and max(e1, e2) < 1e-12
    for leaf in ("0", "2"):
        on, e3 = go(TR_SPEC_LEAF="1", TR_TEST_VIOL=leaf)
        off, e4 = go(TR_SPEC_LEAF="0", TR_TEST_VIOL=leaf)
        assert on == off, leaf
        assert max(e3, e4) < 1e-12
