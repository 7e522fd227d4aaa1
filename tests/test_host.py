"""Host-side API mirror: problem containers behave like the reference's
(ref: pkg/src/toepreg/toeplitz.py:37-233) and the reference's own
ProblemSpec objects are accepted by duck typing."""

import os

import numpy as np
import pytest

import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import workloads as wl


def test_toeplitz_layout_and_validation():
    t = tb.ToeplitzSpec(2, 3, [1, 2, 3, 4])  # gen top-right -> bottom-left
    assert t.entry(0, 2) == 1 and t.entry(0, 0) == 3 and t.entry(1, 0) == 4
    assert t.gen.dtype == np.complex128 and not t.gen.flags.writeable
    with pytest.raises(ValueError):
        tb.ToeplitzSpec(2, 3, [1, 2, 3])
    with pytest.raises(ValueError):
        tb.ToeplitzSpec(0, 3, [])
    a = tb.adjoint_spec(tb.ToeplitzSpec(2, 2, [1j, 2, 3]))
    assert np.array_equal(a.gen, np.array([3, 2, -1j]))


def test_hermitian_spec():
    h = tb.HermitianToeplitzSpec(3, [2.0, 1 + 1j, 3j])
    assert np.array_equal(h.full_gen, [-3j, 1 - 1j, 2, 1 + 1j, 3j])
    with pytest.raises(ValueError):
        tb.HermitianToeplitzSpec(2, [1j, 0])
    with pytest.raises(ValueError):
        tb.HermitianToeplitzSpec(3, [1, 2])


def test_problem_constructors_validate_like_the_reference():
    T = tb.ToeplitzSpec(3, 2, np.ones(4))
    L = tb.ToeplitzSpec(2, 2, np.ones(3))
    with pytest.raises(ValueError):
        tb.ProblemSpec.general(T, tb.ToeplitzSpec(2, 3, np.ones(4)), np.ones(3))
    with pytest.raises(ValueError):
        tb.ProblemSpec.general(T, L, np.ones(2))
    with pytest.raises(ValueError):
        tb.ProblemSpec.l2(T, 0, np.ones(3))
    with pytest.raises(ValueError):
        tb.ProblemSpec.gramian(tb.HermitianToeplitzSpec(3, [1, 0, 0]), L, np.ones(3))
    p = tb.ProblemSpec.l2(T, 2j, np.ones(3))
    assert p.beta_sq == 4.0 and p.n == 2 and p.m == 3 and p.reg_rows == 2


def test_workloads_are_seed_deterministic():
    a = wl.c5_random(n=64, count=2, seed=7)
    b = wl.c5_random(n=64, count=2, seed=7)
    assert np.array_equal(a["T_gen"], b["T_gen"]) and np.array_equal(a["b"], b["b"])
    c = wl.c2_rect(m=64, n=32, nrhs=3)
    assert c["b"].shape == (3, 64) and c["T_gen"].shape == (95,)
    g = wl.c4_nufft(m=32, n=64)
    assert g["G_col"][0].imag == 0.0 and abs(g["G_col"][0] - 32) < 1e-9


def test_reference_problem_objects_are_accepted_by_shape_logic():
    ref = pytest.importorskip("toepreg", reason="reference package not importable here")
    raw = wl.random_problem("general", 8, np.random.default_rng(1))
    rp = wl.to_problem(raw, ref)
    assert tb.solver._shape(rp) == ("general", 8, 8, 8)


def test_json_formats_roundtrip_like_the_reference():
    """Interchange formats of ref toeplitz.py:236-263 (README:68-72)."""
    import json
    import sys
    import numpy as np
    import paper_1302_6945_b200 as tb
    g = np.array([1 + 2j, 3.5, -1j, 0.25, 7.0])
    spec = tb.ToeplitzSpec(3, 3, g)
    obj = json.loads(json.dumps(tb.spec_to_json(spec)))
    assert obj["rows"] == 3 and obj["cols"] == 3 and obj["gen_re"][0] == 1.0
    back = tb.spec_from_json(json.dumps(obj))
    assert np.array_equal(back.gen, spec.gen)
    assert np.array_equal(tb.spec_from_json({"rows": 1, "cols": 2, "gen_re": [1.0, 2.0]}).gen,
                          np.array([1.0, 2.0], dtype=np.complex128))
    v = np.array([1.0 - 1j, 2.0, 1e-300j])
    assert np.array_equal(tb.vector_from_json(json.dumps(tb.vector_to_json(v))), v)
    assert np.array_equal(tb.vector_from_json({"re": [1.0, 2.0]}), np.array([1.0, 2.0], dtype=complex))


def test_experiment_drivers_host_parts_match_reference():
    """Seeded streams, generators and the complexity fit of the experiment
    drivers against the reference (tests/golden/make_golden_experiments.py)."""
    import json
    import os
    import numpy as np
    from paper_1302_6945_b200 import experiments as ex
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "stages", "experiments.json")))
    for variant in ex.VARIANTS:
        rng = ex._stream(2024, "accuracy", variant, 16, 1)
        p = ex.random_problem(variant, 16, rng)
        x = ex.complex_normal(rng, 16)
        parts = [p.T.gen if p.T is not None else np.zeros(0), p.L.gen if p.L is not None else np.zeros(0),
                 p.G.gen if p.G is not None else np.zeros(0), p.b if p.b is not None else np.zeros(0), x]
        assert float(np.abs(np.concatenate([np.ravel(q) for q in parts])).sum()) == g["draws"][variant][0]
        assert (float(abs(p.beta)) if p.beta is not None else 0.0) == g["draws"][variant][1]
    fit = ex.fit_complexity([256, 512, 1024, 2048], [0.011, 0.026, 0.060, 0.135])
    assert np.allclose([fit.c1, fit.c2, fit.r_squared], g["fit"], rtol=1e-12, atol=0)
    assert {v: ex.free_parameters(v, 100) for v in ex.VARIANTS} == g["free_parameters"]


def test_bench_reference_arm_runs_on_cpu():
    """`bench.py --impl reference` (the driver's reference arm) needs no GPU:
    it times the oracle on the host cores and prints one JSON line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    for key in ("metric", "unit", "cpu_baseline", "e2e", "config", "higher_is_better"):
        assert key in line
