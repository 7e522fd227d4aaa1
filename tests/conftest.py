import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


def load_case(path):
    """Golden fixture -> (raw problem dict, fixture dict).  Cases stored by
    recipe regenerate their inputs from the seeded workload generators."""
    from paper_1302_6945_b200 import workloads as wl
    d = dict(np.load(path))
    raw = {k: (v.item() if v.ndim == 0 else v) for k, v in d.items()}
    raw["variant"] = str(d["variant"])
    if "recipe" in d:
        # "<generator call>[index]" or "<generator call>": regenerate the inputs
        r = str(d["recipe"])
        call, idx = r, None
        if r.endswith("]"):
            call, idx = r[:r.rindex("[")], int(r[r.rindex("[") + 1:-1])
        name = call[:call.index("(")]
        if name not in wl.__all__:
            raise ValueError(r)
        src = eval(call, {"__builtins__": {}}, {name: getattr(wl, name)})  # noqa: S307 (fixture recipe)
        for key in ("T_gen", "L_gen", "G_col", "b", "normal_rhs", "beta", "L_rows"):
            v = src.get(key)
            if v is None:
                continue
            if idx is not None and isinstance(v, np.ndarray) and v.ndim == 2:
                v = v[idx]
            raw[key] = v
    return raw, d


def case_config(tb, d, refine=1):
    """SolverConfig of a fixture (fill policy recorded by make_golden_big)."""
    fill = str(d["cfg_fill"]) if "cfg_fill" in d else "auto"
    return tb.SolverConfig(fill=fill, refine=refine)


def decisions_robust(d):
    """True when every discrete decision of the reference on this fixture is
    far from its threshold (tests/golden/add_margins.py): no near-tie between
    pivot candidates (exact structural ties, margin 0, are broken the same way
    by both), no |phi_j| within 3x of the deferral threshold, no leaf
    self-residual within 3x of the retry tolerance, and the reference's own
    ledger survives a rounding change (float64 instead of long-double tree
    products).  Then a run that differs from it only in rounding takes the
    same decisions, and its integer outputs must equal the reference's."""
    mp_ = float(d["margin_pivot"])
    if not (mp_ == 0.0 or mp_ > 1e-6):
        return False
    if float(d["margin_defer"]) < 0.5 or float(d["margin_check"]) < 0.5:
        return False
    if "spread_col_degrees" in d and not np.array_equal(d["spread_col_degrees"], d["final_col_degrees"]):
        return False
    return True


def case_paths(pattern="*"):
    return sorted(glob.glob(os.path.join(GOLDEN, "cases", pattern + ".npz")))


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0))


@pytest.fixture(scope="session")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1302_6945_b200 as tb
    return tb
