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
        r = str(d["recipe"])
        if r.startswith("c2_rect"):
            src = wl.c2_rect(nrhs=1, seed=0)
            raw["T_gen"], raw["b"], raw["beta"] = src["T_gen"], src["b"][0], src["beta"]
        elif r.startswith("c5_random"):
            src = wl.c5_random(n=16384, count=1, seed=0)
            raw["T_gen"], raw["b"], raw["beta"] = src["T_gen"][0], src["b"][0], src["beta"]
        else:
            raise ValueError(r)
    return raw, d


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
