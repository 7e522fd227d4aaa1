"""CPU oracle for the superfast Tikhonov-Toeplitz solve path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` leg may call it, and only as the checker or
the timed CPU baseline.  It is a numpy restatement of the reference package
``toepreg`` 0.1.0 (``/root/reference/pkg/src/toepreg``), written against the
reference's documented behaviour and pinned against the reference itself by
the golden fixtures in ``tests/golden`` (see ``tests/golden/make_golden.py``
and ``tests/test_oracle.py``): on every fixture the oracle reproduces the
reference's ``x_hat`` bit for bit, because it performs the same numpy
primitive operations in the same order.

Citations (``ref:`` = ``/root/reference/pkg/src/toepreg/``):
  fast_len            ref:fftpoly.py:43-56   (next_fast_len, 7-smooth)
  grid_eval           ref:fftpoly.py:64-89
  matpoly_product     ref:fftpoly.py:215-230 (long-double branch :222-226)
  trim_tail           ref:fftpoly.py:148-155, :211-212
  extend_detail       ref:extension.py:42-68
  extended_gen        ref:extension.py:76-102
  assemble            ref:extension.py:105-138, :190-273
  toeplitz_apply      ref:toeplitz.py:79-111
  golden_stride       ref:tanint.py:220-238
  attempt_orders      ref:tanint.py:247-259
  sweep               ref:tanint.py:137-217 (_Workspace + _serial_core)
  leaf                ref:tanint.py:395-434 (+ _self_residual :262-270)
  tree walk           ref:tanint.py:347-393 (_count/_indices/_split/_rec/_update_weights)
  cleanup             ref:tanint.py:438-454
  extract             ref:tanint.py:470-491
  normal_apply        ref:solver.py:104-167
  solve               ref:solver.py:58-78
"""

from __future__ import annotations

import functools
import math
import time

import numpy as np
import scipy.fft as _sfft

_LD_EXTENDS = np.finfo(np.longdouble).eps < np.finfo(np.float64).eps

RESCALE_TRIGGER = 1e8        # ref:tanint.py:41
RESCALE_PERIOD = 8           # ref:tanint.py:42
LEAF_CHECK_TOL = 1e-11       # ref:tanint.py:244
TRIM_TOL = 1e-14             # ref:fftpoly.py:211
GOLDEN = 0.6180339887498949  # ref:tanint.py:234


# Test-only instrumentation (None = off; never changes the arithmetic):
#   MARGINS: list receiving ("pivot", 1 - |phi_2nd| / |phi_1st|),
#            ("defer", |phi_j| / (thr max|phi|)) per decision and
#            ("check", self residual / tolerance) per leaf attempt, so the
#            fixtures can record how close each discrete decision of the
#            reference was to flipping under rounding;
#   COMBINE_EXTENDED: False runs the tree products in float64 instead of
#            long double (the reference's own rounding-path spread, SURVEY
#            App. B "ref <-> ref with FP64 combine").
MARGINS = None
COMBINE_EXTENDED = True


class OracleSingular(RuntimeError):
    """Mirror of ref:tanint.py:45 SingularSystemError."""


# ----------------------------------------------------------------- sizes

@functools.lru_cache(maxsize=None)
def fast_len(n: int) -> int:
    """Smallest 7-smooth integer >= n (ref:fftpoly.py:43-56)."""
    if n <= 1:
        return 1
    cand = n
    while True:
        r = cand
        for f in (2, 3, 5, 7):
            while r % f == 0:
                r //= f
        if r == 1:
            return cand
        cand += 1


def extend_detail(n_tilde, n_lim, rows=3, paired=True, force_even=True):
    """(k, levels, leaf_size) per ref:extension.py:42-68."""
    if n_tilde < 1:
        raise ValueError("system size must be positive")
    if n_lim < rows:
        raise ValueError("serial budget must allow at least one node per row")
    per = (2 if paired else 1) * rows
    levels, m = 0, n_tilde
    while per * m > n_lim:
        if m <= (2 if force_even else 1):
            raise ValueError("serial budget too small to terminate the split")
        levels += 1
        m = (m + 1) // 2
        if force_even and (m & 1):
            m += 1
    return (m << levels) - n_tilde, levels, m


# ------------------------------------------------------ toeplitz helpers

def _gen(spec):
    return np.asarray(spec.gen, dtype=np.complex128)


def adjoint_gen(gen):
    """Generator of the conjugate transpose (ref:toeplitz.py:104-106)."""
    return np.conj(gen)[::-1]


def toeplitz_apply(gen, rows, cols, x):
    """T @ x by circulant embedding of 7-smooth order (ref:toeplitz.py:79-101)."""
    x = np.asarray(x, dtype=np.complex128)
    q = fast_len(rows + cols - 1)
    col = np.zeros(q, dtype=np.complex128)
    col[:rows] = gen[cols - 1:]
    if cols > 1:
        col[q - (cols - 1):] = gen[:cols - 1]
    return np.fft.ifft(np.fft.fft(col) * np.fft.fft(x, q))[:rows]


def hermitian_full_gen(first_col):
    """Top-right -> bottom-left generator of a Hermitian Toeplitz matrix
    given by its first column (ref:toeplitz.py:132-135)."""
    g = np.asarray(first_col, dtype=np.complex128)
    return np.concatenate([np.conj(g[:0:-1]), g])


def normal_rhs(problem):
    """T^H b unless a planted normal rhs is supplied (ref:toeplitz.py:229-233)."""
    if getattr(problem, "normal_rhs", None) is not None:
        return np.asarray(problem.normal_rhs, dtype=np.complex128)
    T = problem.T
    return toeplitz_apply(adjoint_gen(_gen(T)), T.cols, T.rows, problem.b)


def beta_sq(problem):
    return abs(problem.beta) ** 2


# ------------------------------------------------------------- grid eval

def grid_eval(coeffs, n_nodes, offset=0, stride=1):
    """Values at w**(offset + stride*t), w = exp(2 pi i / n_nodes)
    (ref:fftpoly.py:64-89): twist, fold mod count, count * ifft."""
    if n_nodes < 1:
        raise ValueError("grid size must be positive")
    if stride < 1 or n_nodes % stride:
        raise ValueError("stride must be a positive divisor of the grid size")
    count = n_nodes // stride
    c = np.asarray(coeffs, dtype=np.complex128)
    length = c.shape[-1]
    off = offset % n_nodes
    if off:
        c = c * np.exp(2j * np.pi * off * np.arange(length) / n_nodes)
    if length > count:
        extra = (-length) % count
        if extra:
            c = np.pad(c, [(0, 0)] * (c.ndim - 1) + [(0, extra)])
        c = c.reshape(c.shape[:-1] + (-1, count)).sum(axis=-2)
    return count * np.fft.ifft(c, n=count, axis=-1)


# ------------------------------------------------------------- assembly

def extended_gen(gen, k, fill):
    """Prepend k outward diagonals: zeros, or the generator echoed
    (ref:extension.py:76-102)."""
    if k < 0:
        raise ValueError("extension count must be nonnegative")
    if k == 0:
        return gen.copy()
    if fill == "auto":
        mode = "zero" if k <= 1 else "echo"
    elif fill in ("zero", "echo"):
        mode = fill
    else:
        raise ValueError(f"unknown fill policy {fill!r}")
    if mode == "zero":
        head = np.zeros(k, dtype=np.complex128)
    else:
        head = gen[np.arange(k) % gen.size][::-1]
    return np.concatenate([head, gen])


def aligned_spectrum(gen, order, fill):
    """ref:extension.py:105-116."""
    k = order - gen.size
    if k < 0:
        raise ValueError("circulant order smaller than the block generator")
    return grid_eval(extended_gen(gen, k, fill), order)


def rhs_spectrum(rhs, order):
    """ref:extension.py:134-138 (bottom-aligned, negated)."""
    c = np.zeros(order, dtype=np.complex128)
    c[order - rhs.size:] = -rhs
    return grid_eval(c, order)


def unit_roots(n):
    """ref:fftpoly.py:59-61."""
    return np.exp(2j * np.pi * np.arange(n) / n)


class Assembled:
    """weights (rows, N, p), tau, nodes; ref:extension.py:151-187."""

    def __init__(self, variant, n, order, bounds, weights):
        self.variant = variant
        self.n = n
        self.order = order
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.tau = self.bounds - 1
        self.weights = weights
        self.nodes = unit_roots(order)
        self.rows, _, self.p = weights.shape


def assemble(problem, n_lim=256, fill="auto", paired=True, force_even=True):
    """Interpolation weights per variant (ref:extension.py:190-273)."""
    variant = problem.variant
    if variant == "l2":
        T = problem.T
        n, m = T.cols, T.rows
        order = m + n + extend_detail(m + n, n_lim, 2, paired, force_even)[0]
        z = unit_roots(order)
        g = _gen(T)
        w = np.zeros((2, order, 5), dtype=np.complex128)
        w[0, :, 0] = beta_sq(problem) * z ** (order - n)
        w[0, :, 1] = aligned_spectrum(adjoint_gen(g), order, fill)
        w[0, :, 2] = 1.0
        w[0, :, 4] = rhs_spectrum(normal_rhs(problem), order)
        w[1, :, 0] = -aligned_spectrum(g, order, fill)
        w[1, :, 1] = z ** (order - m)
        w[1, :, 3] = 1.0
        return Assembled("l2", n, order, [n, m, order - n, order - m, 1], w)
    if variant == "general":
        T, L = problem.T, problem.L
        n, m, pl = T.cols, T.rows, L.rows
        nt = max(m, pl) + n
        order = nt + extend_detail(nt, n_lim, 3, paired, force_even)[0]
        z = unit_roots(order)
        gt, gl = _gen(T), _gen(L)
        w = np.zeros((3, order, 7), dtype=np.complex128)
        w[0, :, 1] = aligned_spectrum(adjoint_gen(gt), order, fill)
        w[0, :, 2] = aligned_spectrum(adjoint_gen(gl), order, fill)
        w[0, :, 3] = 1.0
        w[0, :, 6] = rhs_spectrum(normal_rhs(problem), order)
        w[1, :, 0] = -aligned_spectrum(gt, order, fill)
        w[1, :, 1] = z ** (order - m)
        w[1, :, 4] = 1.0
        w[2, :, 0] = -aligned_spectrum(gl, order, fill)
        w[2, :, 2] = z ** (order - pl)
        w[2, :, 5] = 1.0
        bounds = [n, m, pl, order - n, order - m, order - pl, 1]
        return Assembled("general", n, order, bounds, w)
    if variant == "gramian":
        G, L = problem.G, problem.L
        n, pl = G.order, L.rows
        nt = max(n, pl) + n
        order = nt + extend_detail(nt, n_lim, 2, paired, force_even)[0]
        z = unit_roots(order)
        gl = _gen(L)
        w = np.zeros((2, order, 5), dtype=np.complex128)
        w[0, :, 0] = aligned_spectrum(hermitian_full_gen(G.gen), order, fill)
        w[0, :, 1] = aligned_spectrum(adjoint_gen(gl), order, fill)
        w[0, :, 2] = 1.0
        w[0, :, 4] = rhs_spectrum(normal_rhs(problem), order)
        w[1, :, 0] = -aligned_spectrum(gl, order, fill)
        w[1, :, 1] = z ** (order - pl)
        w[1, :, 3] = 1.0
        return Assembled("gramian", n, order, [n, pl, order - n, order - pl, 1], w)
    raise ValueError(f"unknown variant {variant!r}")


# ----------------------------------------------------- leaf serial sweep

def golden_stride(count):
    """Coprime stride near 0.618*count (ref:tanint.py:220-238)."""
    s = int(round(GOLDEN * count))
    while math.gcd(s, count) != 1:
        s += 1
    return s


def attempt_orders(count):
    """ref:tanint.py:247-259: default order, two bumped strides, reversed."""
    if count <= 2:
        yield np.arange(count)
        return
    base = golden_stride(count)
    default = (np.arange(count) * base) % count
    yield default
    s = int(round(GOLDEN * count))
    for bump in (2, 5):
        t = s + bump
        while math.gcd(t, count) != 1:
            t += 1
        yield (np.arange(count) * t) % count
    yield default[::-1]


def sweep(cube, length, nodes, wrows, refs, degs, thr, may_defer, stats):
    """Absorb conditions one by one into cube[:, :, :length] in place
    (ref:tanint.py:137-217).  Returns (new length, deferred list)."""
    deferred = []
    for t in range(len(nodes)):
        z = nodes[t]
        phi = wrows[t] @ (cube[:, :, :length] @ (z ** np.arange(length)))
        amax = np.abs(phi).max()
        bad = amax == 0.0
        if not bad:
            cands = np.flatnonzero(degs == degs.min())
            j = int(cands[np.argmax(np.abs(phi[cands]))])
            bad = abs(phi[j]) < thr * amax
            if MARGINS is not None:
                a = np.sort(np.abs(phi[cands]))[::-1]
                if a.size > 1:
                    MARGINS.append(("pivot", float(1.0 - a[1] / a[0])))
                MARGINS.append(("defer", float(abs(phi[j]) / (thr * amax))))
        if bad:
            if not may_defer:
                raise OracleSingular("pivot underflow while absorbing a condition")
            deferred.append((z, np.array(wrows[t]), refs[t]))
            continue
        mu = -phi / phi[j]
        mu[j] = 0.0
        if length >= cube.shape[2]:
            raise RuntimeError("workspace capacity exceeded")
        head = cube[:, j, :length].copy()
        cube[:, :, :length] += mu[None, :, None] * head[:, None, :]
        cube[:, j, :length] = -z * head
        cube[:, j, 1:length + 1] += head
        length += 1
        degs[j] += 1
        if (t + 1) % RESCALE_PERIOD == 0:
            cm = np.abs(cube[:, :, :length]).max(axis=(0, 2))
            big = cm > RESCALE_TRIGGER
            if big.any():
                cube[:, big, :] /= cm[big][None, :, None]
                stats["scale"] = max(stats["scale"], float(cm[big].max()))
    return length, deferred


def normalize_columns(cube):
    """Divide each column by its max modulus; returns the largest divisor
    (ref:tanint.py:179-183, :382-384)."""
    cm = np.abs(cube).max(axis=(0, 2))
    safe = np.where(cm > 0.0, cm, 1.0)
    cube /= safe[None, :, None]
    return float(safe.max())


def leaf_basis(weights, nodes_all, idx, degs, thr):
    """One leaf with retries (ref:tanint.py:395-434).  Returns
    (basis, degrees, deferred, scale factor, self residual, attempts)."""
    rows, _, p = weights.shape
    w_in = weights[:, idx, :]
    scale = float(np.abs(w_in).max())
    best = None
    attempts = 0
    for perm in attempt_orders(len(idx)):
        attempts += 1
        order = idx[perm]
        wrows = weights[:, order, :].swapaxes(0, 1).reshape(len(order) * rows, -1)
        z = np.repeat(nodes_all[order], rows)
        refs = [(int(k), r) for k in order for r in range(rows)]
        cube = np.zeros((p, p, len(z) + 1), dtype=np.complex128)
        cube[:, :, 0] = np.eye(p)
        d = degs.copy()
        stats = {"scale": 1.0}
        length, deferred = sweep(cube, 1, z, wrows, refs, d, thr, True, stats)
        factor = normalize_columns(cube[:, :, :length])
        factor = max(factor, stats["scale"])
        coeffs = cube[:, :, :length].copy()
        res = self_residual(coeffs, nodes_all[idx], w_in, scale)
        if MARGINS is not None:
            MARGINS.append(("check", float(res / LEAF_CHECK_TOL)))
        if best is None or res < best[0]:
            best = (res, coeffs, d, deferred, factor)
        if best[0] <= LEAF_CHECK_TOL:
            break
    res, coeffs, d, deferred, factor = best
    return coeffs, d, deferred, factor, res, attempts


def self_residual(coeffs, z, w_in, scale):
    """ref:tanint.py:262-270."""
    if scale == 0.0:
        return 0.0
    zp = z[:, None] ** np.arange(coeffs.shape[2])[None, :]
    vals = np.einsum("ijl,kl->kij", coeffs, zp)
    res = np.einsum("rki,kij->rkj", w_in, vals)
    return float(np.abs(res).max() / scale)


# ------------------------------------------------------------- products

def trim_tail(coeffs, rel_tol=TRIM_TOL):
    """ref:fftpoly.py:148-155."""
    mx = np.abs(coeffs).max()
    if mx == 0.0:
        return coeffs[..., :1]
    prof = np.abs(coeffs).max(axis=(0, 1))
    keep = np.flatnonzero(prof > rel_tol * mx)
    return coeffs[..., :(int(keep[-1]) + 1 if keep.size else 1)]


def matpoly_product(a, b, extended=True):
    """(p,p,La) x (p,p,Lb) via 7-smooth FFTs; long double when the platform
    has it and ``extended`` (ref:fftpoly.py:215-230)."""
    la, lb = a.shape[-1], b.shape[-1]
    out = la + lb - 1
    if out == 1:
        return (a[:, :, 0] @ b[:, :, 0])[:, :, None]
    r = fast_len(out)
    if extended and _LD_EXTENDS:
        fa = np.moveaxis(_sfft.fft(a.astype(np.clongdouble), r, axis=-1), -1, 0)
        fb = np.moveaxis(_sfft.fft(b.astype(np.clongdouble), r, axis=-1), -1, 0)
        res = _sfft.ifft(np.moveaxis(fa @ fb, 0, -1), axis=-1)[:, :, :out]
        return np.ascontiguousarray(res.astype(np.complex128))
    fa = np.moveaxis(np.fft.fft(a, r, axis=-1), -1, 0)
    fb = np.moveaxis(np.fft.fft(b, r, axis=-1), -1, 0)
    prod = np.moveaxis(fa @ fb, 0, -1)
    return np.ascontiguousarray(np.fft.ifft(prod, axis=-1)[:, :, :out])


# ------------------------------------------------------------ tree plan

def split_rule(order, offsets, stride, paired):
    """ref:tanint.py:354-366."""
    if len(offsets) == 1:
        o = offsets[0]
        if paired and order % (4 * stride) == 0:
            return (o, o + stride), (o + 2 * stride, o + 3 * stride), 4 * stride
        if order % (2 * stride) == 0:
            return (o,), (o + stride,), 2 * stride
        return None
    o1, o2 = offsets
    if order % (2 * stride) == 0:
        return (o1, o2), (o1 + stride, o2 + stride), 2 * stride
    return (o1,), (o2,), stride


def coset_indices(order, offsets, stride):
    """ref:tanint.py:350-352."""
    parts = [np.arange(o, order, stride) for o in offsets]
    return parts[0] if len(parts) == 1 else np.sort(np.concatenate(parts))


class Trace:
    """Optional per-stage capture for stage-level parity tests."""

    def __init__(self):
        self.leaves = []
        self.combines = []


class _Run:
    def __init__(self, asm, degs, n_lim, thr, paired, trace):
        self.asm = asm
        self.w = asm.weights.copy()
        self.degs = degs
        self.n_lim = n_lim
        self.thr = thr
        self.paired = paired
        self.trace = trace
        self.deferred = []
        self.depth = 0
        self.scale = 1.0
        self.retried = 0

    def node(self, offsets, stride, depth):
        a = self.asm
        self.depth = max(self.depth, depth)
        cut = None
        if a.rows * len(offsets) * (a.order // stride) > self.n_lim:
            cut = split_rule(a.order, offsets, stride, self.paired)
        if cut is None:
            idx = coset_indices(a.order, offsets, stride)
            coeffs, d, deferred, factor, res, attempts = leaf_basis(
                self.w, a.nodes, idx, self.degs, self.thr)
            if self.trace is not None:
                self.trace.leaves.append(dict(offsets=offsets, stride=stride,
                                              w_in=self.w[:, idx, :].copy(),
                                              degs_in=self.degs.copy(),
                                              basis=coeffs.copy(), degs_out=d.copy(),
                                              res=res, attempts=attempts))
            self.retried += attempts > 1
            self.degs[:] = d
            self.deferred.extend(deferred)
            self.scale = max(self.scale, factor)
            return coeffs
        left, right, st = cut
        bl = self.node(left, st, depth + 1)
        for o in right:                                  # ref:tanint.py:387-393
            idx = np.arange(o, a.order, st)
            vals = np.moveaxis(grid_eval(bl, a.order, offset=o, stride=st), -1, 0)
            self.w[:, idx, :] = np.einsum("rji,jik->rjk", self.w[:, idx, :], vals)
        br = self.node(right, st, depth + 1)
        prod = trim_tail(matpoly_product(bl, br, extended=COMBINE_EXTENDED)).copy()
        if self.trace is not None:
            self.trace.combines.append(dict(a=bl, b=br, out_untrimmed_len=bl.shape[2] + br.shape[2] - 1))
        cm = np.abs(prod).max(axis=(0, 2))
        safe = np.where(cm > 0.0, cm, 1.0)
        prod /= safe[None, :, None]
        self.scale = max(self.scale, float(safe.max()))
        return prod

    def cleanup(self, basis):
        """ref:tanint.py:438-454."""
        if not self.deferred:
            return basis
        pts = sorted(self.deferred, key=lambda d: (d[2][0], d[2][1]))
        if len(pts) > 2:
            s = golden_stride(len(pts))
            pts = [pts[(i * s) % len(pts)] for i in range(len(pts))]
        p = basis.shape[0]
        cube = np.zeros((p, p, basis.shape[2] + len(pts) + 1), dtype=np.complex128)
        cube[:, :, :basis.shape[2]] = basis
        z = np.array([d[0] for d in pts])
        wrows = np.array([self.asm.weights[d[2][1], d[2][0]] for d in pts])
        refs = [d[2] for d in pts]
        stats = {"scale": self.scale}
        length, _ = sweep(cube, basis.shape[2], z, wrows, refs, self.degs,
                          min(1e-13, self.thr), False, stats)
        self.scale = stats["scale"]
        out = cube[:, :, :length].copy()
        normalize_columns(out)
        return out


def extract(basis, degs, n):
    """ref:tanint.py:470-491."""
    zero = np.flatnonzero(degs == 0)
    if zero.size != 1:
        raise OracleSingular(f"expected one degree-zero column, found {zero.size}")
    j = int(zero[0])
    const = basis[-1, j, 0]
    if abs(const) < 1e-12 * np.abs(basis[:, j, :]).max():
        raise OracleSingular("constant slot vanished; no unique solution")
    col = basis[0, j, :]
    x = np.zeros(n, dtype=np.complex128)
    take = min(n, col.size)
    x[:take] = col[:take]
    return x / const


# ------------------------------------------------------ normal operator

def normal_apply(problem, x):
    """(T^H T + L^H L) x, matrix free (ref:solver.py:104-167)."""
    x = np.asarray(x, dtype=np.complex128)
    v = problem.variant
    n = x.size

    def emb(gen, rows, cols, q):
        c = np.zeros(q, dtype=np.complex128)
        c[:rows] = gen[cols - 1:]
        if cols > 1:
            c[q - (cols - 1):] = gen[:cols - 1]
        return np.fft.fft(c)

    if v == "general":
        need = max(problem.T.rows + n, problem.L.rows + n) - 1
    elif v == "l2":
        need = problem.T.rows + n - 1
    else:
        need = max(2 * n, problem.L.rows + n) - 1
    q = fast_len(need)
    fx = np.fft.fft(x, q)

    def gram(spec):
        g = _gen(spec)
        fwd = emb(g, spec.rows, spec.cols, q)
        adj = emb(adjoint_gen(g), spec.cols, spec.rows, q)
        mid = np.fft.ifft(fwd * fx)
        mid[spec.rows:] = 0.0
        return np.fft.ifft(adj * np.fft.fft(mid, q))[:n]

    if v == "general":
        return gram(problem.T) + gram(problem.L)
    if v == "l2":
        return gram(problem.T) + beta_sq(problem) * x
    gfull = hermitian_full_gen(problem.G.gen)
    gx = np.fft.ifft(emb(gfull, n, n, q) * fx)[:n]
    return gx + gram(problem.L)


# ----------------------------------------------------------------- solve

def solve(problem, n_lim=256, pivot_threshold=1e-8, fill="auto", paired=True,
          force_even=True, trace=None):
    """Full path (ref:solver.py:58-78).  Returns a dict with the same fields
    as the reference SolveReport plus a diagnostics dict."""
    t0 = time.perf_counter()
    asm = assemble(problem, n_lim, fill, paired, force_even)
    degs = -asm.tau.copy()
    run = _Run(asm, degs, n_lim, pivot_threshold, paired, trace)
    basis = run.node((0,), 1, 1)
    basis = run.cleanup(basis)
    x = extract(basis, degs, asm.n)
    wall = time.perf_counter() - t0
    rhs = normal_rhs(problem)
    den = float(np.linalg.norm(rhs))
    rel = float(np.linalg.norm(normal_apply(problem, x) - rhs)) / (den if den > 0.0 else 1.0)
    return {
        "x_hat": x,
        "variant": problem.variant,
        "wall_time": wall,
        "relative_residual": rel,
        "final_col_degrees": degs.copy(),
        "diagnostics": {
            "conditions_total": asm.rows * asm.order,
            "difficult_points": len(run.deferred),
            "recursion_depth": run.depth,
            "max_column_scale": run.scale,
        },
        "order": asm.order,
        "retried_leaves": run.retried,
    }


def dense_solution(problem):
    """Dense normal-equation solve (ref:solver.py:81-101), for exact-ish
    references at small n."""
    v = problem.variant
    n = problem.G.order if v == "gramian" else problem.T.cols

    def mat(gen, rows, cols):
        i = np.arange(rows)[:, None]
        j = np.arange(cols)[None, :]
        return np.asarray(gen)[i - j + cols - 1]

    if v == "general":
        t = mat(problem.T.gen, problem.T.rows, problem.T.cols)
        l = mat(problem.L.gen, problem.L.rows, problem.L.cols)
        a = t.conj().T @ t + l.conj().T @ l
    elif v == "l2":
        t = mat(problem.T.gen, problem.T.rows, problem.T.cols)
        a = t.conj().T @ t + beta_sq(problem) * np.eye(n)
    else:
        l = mat(problem.L.gen, problem.L.rows, problem.L.cols)
        a = mat(hermitian_full_gen(problem.G.gen), n, n) + l.conj().T @ l
    return np.linalg.solve(a, normal_rhs(problem))


def cg_exact(problem, tol=1e-15, max_iter=None):
    """Conjugate gradients on normal_apply to a tight tolerance: the
    'exact' reference of SURVEY Appendix B for sizes too big for dense."""
    rhs = normal_rhs(problem)
    n = rhs.size
    x = np.zeros(n, dtype=np.complex128)
    r = rhs.copy()
    d = r.copy()
    rho = float(np.vdot(r, r).real)
    nrm = float(np.linalg.norm(rhs))
    for _ in range(max_iter or 20 * n):
        ad = normal_apply(problem, d)
        alpha = rho / float(np.vdot(d, ad).real)
        x += alpha * d
        r -= alpha * ad
        rho2 = float(np.vdot(r, r).real)
        if math.sqrt(rho2) <= tol * nrm:
            break
        d = r + (rho2 / rho) * d
        rho = rho2
    return x


def cg_solve(problem, max_iterations=None, tolerance=1e-12):
    """Plain conjugate gradients from a zero start, restating the reference's
    cg_solve (ref:solver.py:184-215) on normal_apply; the time budget is not
    restated.  Returns (x, iterations)."""
    rhs = normal_rhs(problem)
    n = rhs.size
    x = np.zeros(n, dtype=np.complex128)
    rhs_norm = float(np.linalg.norm(rhs))
    if rhs_norm == 0.0:
        return x, 0
    limit = max_iterations if max_iterations is not None else max(10 * n, 100)
    r = rhs.copy()
    d = r.copy()
    rho = float(np.vdot(r, r).real)
    iterations = 0
    for _ in range(limit):
        ad = normal_apply(problem, d)
        alpha = rho / float(np.vdot(d, ad).real)
        x += alpha * d
        r -= alpha * ad
        rho_next = float(np.vdot(r, r).real)
        iterations += 1
        if math.sqrt(rho_next) <= tolerance * rhs_norm:
            break
        d = r + (rho_next / rho) * d
        rho = rho_next
    return x, iterations


def nufft_gramian_col(freqs, weights, n):
    """First column of A^H W A (ref:nufft.py:60-72), dense as the reference."""
    lags = np.arange(n)
    return np.einsum("k,kd->d", np.asarray(weights, dtype=np.float64) + 0j,
                     np.exp(2j * np.pi * np.outer(np.asarray(freqs, dtype=np.float64), lags)))


def nufft_samples_and_rhs(freqs, weights, x):
    """Samples A x and rhs A^H (w * samples), dense (ref:nufft.py:106-114)."""
    a = np.exp(-2j * np.pi * np.outer(freqs, np.arange(x.size)))
    samples = a @ x
    return samples, a.conj().T @ (weights * samples)
