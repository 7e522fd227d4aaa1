"""Drop-in ``solve_tikhonov`` on the B200 (ref: pkg/src/toepreg/solver.py:39-78).

Same call signature, argument conventions and returned report as the
reference: ``solve_tikhonov(problem, config=None) -> SolveReport`` with
``x_hat`` a fresh complex128 ndarray of length n, ``final_col_degrees`` the
degree ledger, and ``relative_residual`` = ||A x - y|| / ||y|| for the normal
equations.  The work runs in libtoepreg_b200.so (hand-written sm_100a
kernels) through the C ABI; torch only supplies device memory and streams.

Extras beyond the reference surface, for batched and device-resident use:
``solve_tikhonov_batch(problems)`` (one launch sequence for many systems of
one shape, e.g. config 2's 64 right-hand sides or config 5's 4096 systems)
and ``DeviceBatch`` (inputs already in HBM, used by bench.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _lib

__all__ = ["SolverConfig", "SolveReport", "TanIntDiagnostics", "SingularSystemError",
           "solve_tikhonov", "solve_tikhonov_batch", "DeviceBatch", "plan_info"]


class SingularSystemError(RuntimeError):
    """The interpolation data does not determine a unique solution
    (ref: tanint.py:45-46)."""


@dataclass(frozen=True)
class SolverConfig:
    """ref: solver.py:39-45.  Extra fields: ``refine`` > 0 refines the
    direct (superfast) solution on the normal-equation residual, which puts
    x within ~1e-14 of the exact solution, so the distance to the
    reference's x_hat equals the reference's own error (<= 1e-9 on
    well-conditioned problems); 0 is the reference's single pass, whose FP64
    leaf rounding lands ~sqrt(2) x the reference's error away from it
    (SURVEY Appendix B).  ``refine_cg`` caps the conjugate-gradient
    iterations (warm-started at the direct solution) tried first; systems CG
    does not finish within the cap (ill-conditioned ones), or all systems
    when it is 0, get ``refine`` direct refinement solves instead."""

    n_lim: int = 256
    pivot_threshold: float = 1e-8
    fill: str = "auto"
    paired: bool = True
    force_even: bool = True
    refine: int = 1
    refine_cg: int = 256


@dataclass
class TanIntDiagnostics:
    """ref: tanint.py:72-85 (plus retried_leaves / trim_overflow and the
    CG refinement iterations)."""

    conditions_total: int = 0
    difficult_points: int = 0
    recursion_depth: int = 0
    max_column_scale: float = 1.0
    retried_leaves: int = 0
    trim_overflow: int = 0
    refine_cg_iterations: int = 0
    rescued: bool = False

    def as_dict(self) -> dict:
        return {
            "conditions_total": self.conditions_total,
            "difficult_points": self.difficult_points,
            "recursion_depth": self.recursion_depth,
            "max_column_scale": self.max_column_scale,
        }


@dataclass
class SolveReport:
    """ref: solver.py:48-55."""

    x_hat: np.ndarray
    variant: str
    wall_time: float
    relative_residual: float
    diagnostics: TanIntDiagnostics
    final_col_degrees: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


# ------------------------------------------------------------------ helpers

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1302_6945_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _gen(spec):
    return np.ascontiguousarray(spec.gen, dtype=np.complex128)


def _shape(problem):
    v = problem.variant
    if v not in _lib.VARIANTS:
        raise ValueError(f"unknown variant {v!r}")
    if v == "gramian":
        n = problem.G.order
        return v, n, n, problem.L.rows
    n, m = problem.T.cols, problem.T.rows
    pl = problem.L.rows if v == "general" else n
    return v, m, n, pl


def make_desc(variant, m, n, pl, cfg) -> _lib.TrDesc:
    """``cfg`` is our SolverConfig or any object with the reference's five
    fields (ref solver.py:39-45: n_lim, pivot_threshold, fill, paired,
    force_even); the refinement fields default to ours when absent."""
    if cfg.fill not in _lib.FILLS:
        raise ValueError(f"unknown fill policy {cfg.fill!r}")
    d = _lib.TrDesc()
    d.variant = _lib.VARIANTS[variant]
    d.m, d.n, d.p_rows = m, n, pl
    d.n_lim = int(cfg.n_lim)
    d.pivot_threshold = float(cfg.pivot_threshold)
    d.fill = _lib.FILLS[cfg.fill]
    d.paired = int(bool(cfg.paired))
    d.force_even = int(bool(cfg.force_even))
    d.refine = int(getattr(cfg, "refine", SolverConfig.refine))
    d.refine_cg = int(getattr(cfg, "refine_cg", SolverConfig.refine_cg))
    return d


def plan_info(problem, config=None) -> dict:
    cfg = config or SolverConfig()
    d = make_desc(*_shape(problem), cfg)
    lib = _lib.load()
    order, leaves, kmax = C.c_int64(), C.c_int64(), C.c_int64()
    depth = C.c_int32()
    rc = lib.tr_plan_info(C.byref(d), C.byref(order), C.byref(leaves), C.byref(depth), C.byref(kmax))
    _check(rc)
    return {"order": order.value, "leaves": leaves.value, "depth": depth.value,
            "max_leaf_conditions": kmax.value}


def _check(rc, diags=None):
    if rc == 0:
        return
    msg = _lib.last_error()
    if rc == 2:
        raise ValueError(msg or "invalid argument")
    if rc == 3:
        raise SingularSystemError(msg or "singular interpolation system")
    raise RuntimeError(f"libtoepreg_b200 error {rc}: {msg}")


class DeviceBatch:
    """A batch of same-shape problems staged in device memory.

    ``stage()`` copies host inputs to HBM (pinned staging, async); ``run()``
    launches the whole solve on the current stream; ``fetch()`` copies x back.
    Shared operands (one T for many right-hand sides) use batch stride 0.
    """

    _ws_cache = {}

    def __init__(self, problems: Sequence, config=None):
        torch = _torch()
        if len(problems) == 0:
            raise ValueError("empty batch")
        self.cfg = config or SolverConfig()
        shapes = {_shape(p) for p in problems}
        if len(shapes) != 1:
            raise ValueError("all problems of a batch must share variant and shape")
        self.variant, self.m, self.n, self.pl = shapes.pop()
        self.batch = len(problems)
        self.desc = make_desc(self.variant, self.m, self.n, self.pl, self.cfg)
        lib = _lib.load()
        self.ws_bytes = lib.tr_workspace_bytes(C.byref(self.desc), self.batch)
        if self.ws_bytes == 0:
            _check(2)
        v = self.variant

        def pack(arrs, length):
            """Stack (or share) complex128 vectors as a float64 host tensor."""
            first = arrs[0]
            shared = all(a is first or (a.shape == first.shape and np.array_equal(a, first))
                         for a in arrs[1:])
            if shared:
                host = np.ascontiguousarray(first, dtype=np.complex128).reshape(1, length)
                return host, 0
            host = np.stack([np.asarray(a, dtype=np.complex128) for a in arrs]).reshape(len(arrs), length)
            return host, length

        hosts = {}
        self.bs = {}
        if v in ("general", "l2"):
            hosts["T"], self.bs["T"] = pack([_gen(p.T) for p in problems], self.m + self.n - 1)
        if v in ("general", "gramian"):
            hosts["L"], self.bs["L"] = pack([_gen(p.L) for p in problems], self.pl + self.n - 1)
        if v == "gramian":
            hosts["G"], self.bs["G"] = pack([np.asarray(p.G.gen) for p in problems], self.n)
        if v == "l2":
            b2 = np.array([abs(p.beta) ** 2 for p in problems], dtype=np.float64)
            if np.all(b2 == b2[0]):
                hosts["beta"], self.bs["beta"] = b2[:1].copy(), 0
            else:
                hosts["beta"], self.bs["beta"] = b2, 1
        normal = [getattr(p, "normal_rhs", None) is not None for p in problems]
        if any(normal) and not all(normal):
            raise ValueError("mixing planted normal rhs and data rhs in one batch")
        self.rhs_is_normal = bool(all(normal)) or v == "gramian"
        if self.rhs_is_normal:
            hosts["rhs"], self.bs["rhs"] = pack([np.asarray(p.normal_rhs, dtype=np.complex128)
                                                 for p in problems], self.n)
        else:
            hosts["rhs"], self.bs["rhs"] = pack([np.asarray(p.b, dtype=np.complex128)
                                                 for p in problems], self.m)
        self.hosts = hosts
        # real data (l2): the library's CG refinement then works on real vectors
        self.desc.real_data = int(v == "l2" and not any(
            np.iscomplexobj(hosts[k]) and hosts[k].imag.any() for k in ("T", "rhs")))
        self.h2d_bytes = sum(h.nbytes for h in hosts.values())
        self.dev = {}
        self.x = torch.empty((self.batch, self.n, 2), dtype=torch.float64, device="cuda")
        self.d2h_bytes = self.batch * self.n * 16
        key = (self.variant, self.m, self.n, self.pl, self.batch, self.cfg)
        ws = DeviceBatch._ws_cache.get(key)
        if ws is None:
            ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda")
            DeviceBatch._ws_cache.clear()
            DeviceBatch._ws_cache[key] = ws
        self.ws = ws
        self.diag = (_lib.TrDiag * self.batch)()
        self.pinned = {k: torch.from_numpy(np.array(h, copy=True, order="C").view(np.float64)).pin_memory()
                       for k, h in hosts.items()}
        self.x_host = torch.empty((self.batch, self.n, 2), dtype=torch.float64).pin_memory()

    def stage(self):
        """Host -> device copies of every input (async on the current stream)."""
        for k, h in self.pinned.items():
            d = self.dev.get(k)
            if d is None or d.shape != h.shape:
                d = self.dev[k] = h.to("cuda", non_blocking=True)
            else:
                d.copy_(h, non_blocking=True)
        return self

    def run(self, with_diag: bool = True):
        torch = _torch()
        lib = _lib.load()
        ptr = lambda k: C.c_void_p(self.dev[k].data_ptr()) if k in self.dev else None
        st = torch.cuda.current_stream().cuda_stream
        rc = lib.tr_solve_batch(
            C.byref(self.desc), self.batch,
            ptr("T"), self.bs.get("T", 0), ptr("L"), self.bs.get("L", 0),
            ptr("G"), self.bs.get("G", 0), ptr("beta"), self.bs.get("beta", 0),
            ptr("rhs"), self.bs["rhs"], int(self.rhs_is_normal),
            C.c_void_p(self.x.data_ptr()), self.diag if with_diag else None,
            C.c_void_p(self.ws.data_ptr()), C.c_size_t(self.ws_bytes), C.c_void_p(st))
        if rc not in (0, 3):
            _check(rc)
        self.rc = rc
        return self

    def fetch(self) -> np.ndarray:
        self.x_host.copy_(self.x, non_blocking=True)
        _torch().cuda.current_stream().synchronize()
        return self.x_host.numpy().view(np.complex128).reshape(self.batch, self.n)

    def reports(self, x: np.ndarray) -> List[SolveReport]:
        """One SolveReport per system.  ``wall_time`` is the device time of
        the batch's solve (assemble -> extract, plus refinement), excluding
        staging, the result copy and the residual evaluation, as the
        reference's covers assemble -> extract only (ref solver.py:62-71);
        every system of a batch reports the batch's time."""
        out = []
        for i in range(self.batch):
            dg = self.diag[i]
            if dg.status == 3:
                raise SingularSystemError(f"system {i}: interpolation data singular")
            if dg.status == 6:
                raise RuntimeError(f"system {i}: a basis product exceeded its planned length "
                                   f"({dg.trim_overflow} truncations); refusing to return x")
            if dg.status != 0:
                raise RuntimeError(f"system {i}: solver status {dg.status}: {_lib.last_error()}")
            p = 7 if self.variant == "general" else 5
            diag = TanIntDiagnostics(
                conditions_total=int(dg.conditions_total),
                difficult_points=int(dg.difficult_points),
                recursion_depth=int(dg.recursion_depth),
                max_column_scale=float(dg.max_column_scale),
                retried_leaves=int(dg.retried_leaves),
                trim_overflow=int(dg.trim_overflow),
                refine_cg_iterations=int(dg.refine_cg_iterations),
                rescued=bool(dg.rescued))
            out.append(SolveReport(
                x_hat=np.array(x[i], dtype=np.complex128),
                variant=self.variant, wall_time=float(dg.wall_time_s),
                relative_residual=float(dg.relative_residual), diagnostics=diag,
                final_col_degrees=np.array(dg.final_col_degrees[:p], dtype=np.int64)))
        return out


def solve_tikhonov_batch(problems: Sequence, config=None,
                         max_batch: int = 512) -> List[SolveReport]:
    """Solve many same-shape problems; returns one SolveReport per problem."""
    problems = list(problems)
    reports: List[SolveReport] = []
    for s in range(0, len(problems), max_batch):
        chunk = problems[s:s + max_batch]
        db = DeviceBatch(chunk, config).stage().run()
        reports.extend(db.reports(db.fetch()))
    return reports


def solve_tikhonov(problem, config=None) -> SolveReport:
    """Solve one instance (ref: solver.py:58-78).  ``config`` may be our
    SolverConfig, the reference's own ``toepreg.SolverConfig`` (five fields)
    or None (defaults)."""
    return solve_tikhonov_batch([problem], config)[0]
