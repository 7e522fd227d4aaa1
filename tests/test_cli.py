"""CLI wiring (paper_1302_6945_b200/cli.py; reference behaviour:
pkg/src/toepreg/cli.py and its tests pkg/tests/test_cli.py): argument and
input errors exit 2 before any solve (CPU), solves run on the GPU and match
the dense Tikhonov solution, numerical failures exit 3."""

import json

import numpy as np
import pytest

from paper_1302_6945_b200 import cli
from paper_1302_6945_b200.experiments import dense_solution
from paper_1302_6945_b200.toeplitz import (HermitianToeplitzSpec, ProblemSpec, ToeplitzSpec,
                                           spec_to_json, vector_to_json)


def _dump(path, obj):
    path.write_text(json.dumps(obj))
    return str(path)


def _vec(path):
    obj = json.loads(path.read_text())
    return np.asarray(obj["re"]) + 1j * np.asarray(obj["im"])


def _cvec(rng, k):
    return rng.standard_normal(k) + 1j * rng.standard_normal(k)


def _spec(rng, m, n):
    return ToeplitzSpec(m, n, _cvec(rng, m + n - 1))


# ---------------------------------------------------------------- CPU: errors

def test_usage_errors_exit_two(capsys):
    assert cli.main([]) == 2
    assert cli.main(["solve", "--variant", "l2", "--n", "8", "--no-such-flag"]) == 2
    assert "usage" in capsys.readouterr().err
    assert cli.main(["accuracy", "--sizes", "16,-4"]) == 2
    assert cli.main(["complexity", "--sizes", "a,b"]) == 2
    assert cli.main(["solve", "--variant", "l2", "--beta-sq", "huge", "--n", "8"]) == 2


def test_input_errors_exit_two_before_solving(tmp_path, capsys):
    t = _dump(tmp_path / "T.json", {"rows": 2, "cols": 2, "gen_re": [0, 1, 0]})
    assert cli.main(["solve", "--variant", "general", "--input", t]) == 2
    assert cli.main(["solve", "--variant", "general", "--input", t,
                     "--reg", t]) == 2                      # no --b
    assert cli.main(["solve", "--variant", "l2", "--input", t]) == 2
    assert cli.main(["solve", "--variant", "gramian", "--input", t, "--reg", t]) == 2
    missing = str(tmp_path / "absent.json")
    assert cli.main(["solve", "--variant", "l2", "--input", missing, "--b", missing]) == 2
    assert cli.main(["solve", "--variant", "l2"]) == 2     # neither --input nor --n
    assert cli.main(["solve", "--variant", "l2", "--n", "8", "--beta-sq", "-1"]) == 2
    assert cli.main(["solve", "--variant", "l2", "--n", "8", "--count", "0"]) == 2
    assert cli.main(["solve", "--variant", "l2", "--input", t, "--b", t, "--count", "2"]) == 2
    assert "error:" in capsys.readouterr().err


def test_gramian_input_must_be_square_hermitian(tmp_path):
    rng = np.random.default_rng(7)
    reg = _dump(tmp_path / "L.json", spec_to_json(_spec(rng, 6, 6)))
    rhs = _dump(tmp_path / "r.json", vector_to_json(np.ones(6)))
    for bad in (_spec(rng, 6, 6), _spec(rng, 5, 6)):
        g = _dump(tmp_path / "G.json", spec_to_json(bad))
        assert cli.main(["solve", "--variant", "gramian", "--input", g,
                         "--reg", reg, "--rhs", rhs]) == 2


def test_hermitian_conversion_keeps_first_column():
    h = HermitianToeplitzSpec(4, [5.0, 1 + 2j, -1j, 0.5])
    full = ToeplitzSpec(4, 4, h.full_gen)
    back = cli._as_hermitian(full)
    assert back.order == 4 and np.array_equal(back.gen, h.gen)
    assert np.array_equal(back.full_gen, h.full_gen)


def test_seeded_problem_stream_and_beta_default():
    ns = cli.build_parser().parse_args(["solve", "--variant", "l2", "--n", "16", "--m", "24"])
    a = cli._seeded_problem(ns, 3)
    b = cli._seeded_problem(ns, 3)
    assert a.variant == "l2" and a.m == 24 and a.n == 16
    assert np.array_equal(a.T.gen, b.T.gen) and np.array_equal(a.b, b.b)
    assert abs(a.beta - 16 ** 0.25) < 1e-15
    ns = cli.build_parser().parse_args(["solve", "--variant", "l2", "--n", "16",
                                        "--beta-sq", "4"])
    assert abs(cli._seeded_problem(ns, 0).beta - 2.0) < 1e-15


# ---------------------------------------------------------------- GPU: solves

@pytest.mark.gpu
def test_cli_solve_random_matches_dense(gpu, tmp_path, capsys):
    out = tmp_path / "x.json"
    for variant in ("general", "l2", "gramian"):
        assert cli.main(["solve", "--variant", variant, "--n", "40", "--seed", "5",
                         "--out", str(out)]) == 0
        assert f"variant={variant}" in capsys.readouterr().out
        ns = cli.build_parser().parse_args(["solve", "--variant", variant, "--n", "40"])
        x_ref = dense_solution(cli._seeded_problem(ns, 5))
        x = _vec(out)
        assert x.shape == (40,)
        assert np.linalg.norm(x - x_ref) <= 1e-9 * np.linalg.norm(x_ref)


@pytest.mark.gpu
def test_cli_solve_from_files_matches_dense(gpu, tmp_path):
    rng = np.random.default_rng(61)
    t, reg, b = _spec(rng, 28, 20), _spec(rng, 12, 20), _cvec(rng, 28)
    out = tmp_path / "x.json"
    assert cli.main(["solve", "--variant", "general",
                     "--input", _dump(tmp_path / "T.json", spec_to_json(t)),
                     "--reg", _dump(tmp_path / "L.json", spec_to_json(reg)),
                     "--b", _dump(tmp_path / "b.json", vector_to_json(b)),
                     "--out", str(out)]) == 0
    x_ref = dense_solution(ProblemSpec.general(t, reg, b))
    assert np.linalg.norm(_vec(out) - x_ref) <= 1e-9 * np.linalg.norm(x_ref)

    t2, b2 = _spec(rng, 16, 16), _cvec(rng, 16)
    assert cli.main(["solve", "--variant", "l2",
                     "--input", _dump(tmp_path / "T2.json", spec_to_json(t2)),
                     "--b", _dump(tmp_path / "b2.json", vector_to_json(b2)),
                     "--beta-sq", "auto", "--out", str(out)]) == 0
    x_ref = dense_solution(ProblemSpec.l2(t2, 16 ** 0.25, b2))
    assert np.linalg.norm(_vec(out) - x_ref) <= 1e-9 * np.linalg.norm(x_ref)


@pytest.mark.gpu
def test_cli_batch_count_equals_single_solves(gpu, tmp_path, capsys):
    out = tmp_path / "xs.json"
    assert cli.main(["solve", "--variant", "l2", "--n", "48", "--seed", "10",
                     "--count", "3", "--out", str(out)]) == 0
    assert capsys.readouterr().out.count("variant=l2") == 3
    batch = json.loads(out.read_text())
    one = tmp_path / "x.json"
    for k in range(3):
        assert cli.main(["solve", "--variant", "l2", "--n", "48", "--seed", str(10 + k),
                         "--out", str(one)]) == 0
        single = _vec(one)
        xb = np.asarray(batch[k]["re"]) + 1j * np.asarray(batch[k]["im"])
        assert np.array_equal(xb, single)       # batch-invariant results


@pytest.mark.gpu
def test_cli_singular_system_exits_three(gpu, tmp_path, capsys):
    zeros = {"rows": 4, "cols": 4, "gen_re": [0.0] * 7}
    assert cli.main(["solve", "--variant", "gramian",
                     "--input", _dump(tmp_path / "G.json", zeros),
                     "--reg", _dump(tmp_path / "L.json", zeros),
                     "--rhs", _dump(tmp_path / "r.json", vector_to_json(np.ones(4)))]) == 3
    assert "numerical failure" in capsys.readouterr().err
