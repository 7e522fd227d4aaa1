"""GPU normal operator and conjugate gradients (ref: pkg/src/toepreg/solver.py
:104-215 ``NormalOperator``, ``apply_normal_operator``, ``CGConfig``,
``cg_solve``).

Same signatures and conventions as the reference: ``NormalOperator(problem)``
with ``.apply(x)``, ``.n`` and the ``.transforms`` counter (forward plus
inverse FFTs: 7 per apply for the general variant, 4 for l2, 5 for gramian);
``cg_solve(problem, config=None, operator=None) -> (x, iterations)`` runs
plain CG from a zero start and stops at ``||r|| <= tolerance * ||rhs||``, the
iteration limit (default ``max(10 n, 100)``) or the time budget (checked
after completed iterations).  The arithmetic runs in libtoepreg_b200.so
(``tr_normal_apply`` / ``tr_cg_batch``: the FFT normal operator of the
solver plus one fused vector-update kernel per iteration); ``cg_solve_batch``
runs many same-shape systems at once with per-system stopping.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .solver import DeviceBatch, SolverConfig, _check, _torch

__all__ = ["NormalOperator", "apply_normal_operator", "CGConfig", "cg_solve", "cg_solve_batch"]

_TRANSFORMS = {"general": 7, "l2": 4, "gramian": 5}


class _Staged:
    """Problem inputs staged in HBM plus the operator / CG workspace."""

    def __init__(self, problems: Sequence):
        torch = _torch()
        self.db = DeviceBatch(list(problems), SolverConfig()).stage()
        lib = _lib.load()
        self.ws_bytes = lib.tr_cg_workspace_bytes(C.byref(self.db.desc), self.db.batch)
        if self.ws_bytes == 0:
            _check(2)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda")

    def ptr(self, k):
        d = self.db.dev.get(k)
        return C.c_void_p(d.data_ptr()) if d is not None else None

    def operands(self):
        bs = self.db.bs
        return (self.ptr("T"), bs.get("T", 0), self.ptr("L"), bs.get("L", 0),
                self.ptr("G"), bs.get("G", 0), self.ptr("beta"), bs.get("beta", 0))


class NormalOperator:
    """Matrix-free x -> (T^H T + L^H L) x on the GPU (ref solver.py:104-167)."""

    def __init__(self, problem):
        self.problem = problem
        self.transforms = 0
        self._st = _Staged([problem])
        self._per_apply = _TRANSFORMS[self._st.db.variant]

    @property
    def n(self) -> int:
        return self.problem.n

    def apply(self, x: np.ndarray) -> np.ndarray:
        torch = _torch()
        n = self.problem.n
        xv = np.ascontiguousarray(np.asarray(x, dtype=np.complex128).reshape(n))
        xd = torch.from_numpy(xv.view(np.float64).copy()).to("cuda")
        yd = torch.empty_like(xd)
        lib = _lib.load()
        st = torch.cuda.current_stream().cuda_stream
        rc = lib.tr_normal_apply(C.byref(self._st.db.desc), 1, *self._st.operands(),
                                 C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()),
                                 C.c_void_p(self._st.ws.data_ptr()), C.c_size_t(self._st.ws_bytes),
                                 C.c_void_p(st))
        _check(rc)
        self.transforms += self._per_apply
        return yd.cpu().numpy().view(np.complex128).reshape(n).copy()


def apply_normal_operator(problem, x: np.ndarray) -> np.ndarray:
    return NormalOperator(problem).apply(x)


@dataclass(frozen=True)
class CGConfig:
    max_iterations: Optional[int] = None
    tolerance: float = 1e-12
    time_budget: Optional[float] = None


def _cg(st: _Staged, cfg: CGConfig) -> Tuple[np.ndarray, np.ndarray]:
    torch = _torch()
    db = st.db
    lib = _lib.load()
    x = torch.empty((db.batch, db.n, 2), dtype=torch.float64, device="cuda")
    its = (C.c_int64 * db.batch)()
    s = torch.cuda.current_stream().cuda_stream
    rc = lib.tr_cg_batch(C.byref(db.desc), db.batch, *st.operands(),
                         st.ptr("rhs"), db.bs["rhs"], int(db.rhs_is_normal),
                         int(cfg.max_iterations or 0), float(cfg.tolerance),
                         -1.0 if cfg.time_budget is None else float(cfg.time_budget),
                         C.c_void_p(x.data_ptr()), its,
                         C.c_void_p(st.ws.data_ptr()), C.c_size_t(st.ws_bytes), C.c_void_p(s))
    _check(rc)
    xh = x.cpu().numpy().view(np.complex128).reshape(db.batch, db.n).copy()
    return xh, np.array(its[:], dtype=np.int64)


def _same_matrix(p, q) -> bool:
    def gen(spec):
        return None if spec is None else (spec.rows if hasattr(spec, "rows") else spec.order,
                                          np.asarray(spec.gen).tobytes())
    return (p.variant == q.variant and gen(p.T) == gen(q.T) and gen(p.L) == gen(q.L)
            and gen(p.G) == gen(q.G) and (p.beta or 0) == (q.beta or 0))


def cg_solve(problem, config: CGConfig = None, operator: NormalOperator = None):
    """Plain conjugate gradients from a zero start.  Returns (x, iterations)."""
    cfg = config or CGConfig()
    if cfg.max_iterations is not None and cfg.max_iterations <= 0:
        return np.zeros(problem.n, dtype=np.complex128), 0
    # ref solver.py:181-215 applies `operator` to `problem`'s right-hand side:
    # an operator of the same normal matrix (same T / L / G / beta) is
    # equivalent to staging `problem` itself; another matrix is refused
    if operator is not None and operator.problem is not problem:
        if not _same_matrix(operator.problem, problem):
            raise ValueError("operator was built for a different normal matrix")
    reuse = operator is not None and operator.problem is problem
    st = operator._st if reuse else _Staged([problem])
    x, its = _cg(st, cfg)
    if operator is not None:
        operator.transforms += operator._per_apply * int(its[0])
    return x[0], int(its[0])


def cg_solve_batch(problems: Sequence, config: CGConfig = None) -> List[Tuple[np.ndarray, int]]:
    """CG on many same-shape problems at once (per-system stopping)."""
    cfg = config or CGConfig()
    x, its = _cg(_Staged(problems), cfg)
    return [(x[i], int(its[i])) for i in range(len(problems))]
