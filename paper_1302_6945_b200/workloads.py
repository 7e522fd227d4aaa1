"""Seeded synthetic inputs for the five BASELINE configurations.

BASELINE.json names no public dataset: its configs *are* synthetic inputs,
so these generators are the workloads.  Draws follow the reference's
``SeedSequence`` tuple pattern (ref: pkg/src/toepreg/experiments.py:83-85):
config ``c``, item ``i`` under master seed ``S`` use
``default_rng(SeedSequence((S, c, i)))``.  "N(0, s)" is read as variance s.

Each generator returns plain numpy arrays in a dict (``variant`` plus the
generator-form operands); ``to_problem`` turns one into any ProblemSpec class
with the reference's constructor conventions (ours or the reference's own).
Real configs are complex128 with zero imaginary parts, as the reference
promotes them (ref: toeplitz.py:48).
"""

from __future__ import annotations

import numpy as np

__all__ = ["rng_for", "c1_blur", "c2_rect", "c3_firstdiff", "c4_nufft",
           "c5_random", "random_problem", "to_problem", "CONFIG_SHAPES"]

# config -> (variant, m, n) of the full-size BASELINE instance
CONFIG_SHAPES = {
    "c1": ("l2", 256, 256),
    "c2": ("l2", 8192, 4096),
    "c3": ("general", 65536, 65536),
    "c4": ("gramian", 8192, 16384),
    "c5": ("l2", 16384, 16384),
    "c5b": ("l2", 1 << 22, 1 << 22),
}


def rng_for(seed: int, config: int, item: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence((seed, config, item)))


def _cplx(a):
    return np.asarray(a, dtype=np.complex128)


def _toeplitz_matvec(gen, rows, cols, x):
    """Dense-free T @ x for input synthesis (circulant embedding, pow2 FFT)."""
    q = 1
    while q < rows + cols - 1:
        q *= 2
    col = np.zeros(q, dtype=np.complex128)
    col[:rows] = gen[cols - 1:]
    if cols > 1:
        col[q - (cols - 1):] = gen[:cols - 1]
    return np.fft.ifft(np.fft.fft(col) * np.fft.fft(x, q))[:rows]


def c1_blur(n: int = 256, seed: int = 0, item: int = 0, width: float = 4.0,
            lam: float = 1e-2):
    """Config 1: symmetric Gaussian blur a_k = exp(-k^2 / (2 w^2)), |k| < n,
    x ~ N(0,1), b = T x + N(0, 1e-6), L = I, lambda = 1e-2 (l2, beta = lambda)."""
    rng = rng_for(seed, 1, item)
    k = np.arange(-(n - 1), n)
    gen = _cplx(np.exp(-(k.astype(np.float64) ** 2) / (2.0 * width * width)))
    x = rng.standard_normal(n)
    b = _toeplitz_matvec(gen, n, n, _cplx(x)).real + 1e-3 * rng.standard_normal(n)
    return {"variant": "l2", "m": n, "n": n, "T_gen": gen, "beta": lam,
            "b": _cplx(b), "x_true": _cplx(x)}


def c2_rect(m: int = 8192, n: int = 4096, nrhs: int = 64, seed: int = 0,
            item: int = 0, lam: float = 1e-1):
    """Config 2: rectangular T (first column and row i.i.d. N(0,1)/sqrt(n)),
    shared by ``nrhs`` right-hand sides b_j = T x_j + N(0, 1e-4)."""
    rng = rng_for(seed, 2, item)
    gen = _cplx(rng.standard_normal(m + n - 1) / np.sqrt(n))
    bs, xs = [], []
    for _ in range(nrhs):
        x = rng.standard_normal(n)
        b = _toeplitz_matvec(gen, m, n, _cplx(x)).real + 1e-2 * rng.standard_normal(m)
        bs.append(_cplx(b))
        xs.append(_cplx(x))
    return {"variant": "l2", "m": m, "n": n, "T_gen": gen, "beta": lam,
            "b": np.stack(bs), "x_true": np.stack(xs)}


def c3_firstdiff(n: int = 65536, lam: float = 1e-2, seed: int = 0, item: int = 0):
    """Config 3: square T with gen_k = 0.9^|k| N(0,1), L = lambda * D with D the
    first difference (1 on the diagonal, -1 on the subdiagonal),
    b = T x + N(0, 1e-4)."""
    rng = rng_for(seed, 3, item)
    k = np.arange(-(n - 1), n)
    gen = _cplx(0.9 ** np.abs(k) * rng.standard_normal(2 * n - 1))
    lgen = np.zeros(2 * n - 1, dtype=np.complex128)
    lgen[n - 1] = lam
    lgen[n] = -lam
    x = rng.standard_normal(n)
    b = _toeplitz_matvec(gen, n, n, _cplx(x)).real + 1e-2 * rng.standard_normal(n)
    return {"variant": "general", "m": n, "n": n, "T_gen": gen, "L_rows": n,
            "L_gen": lgen, "b": _cplx(b), "x_true": _cplx(x)}


def c4_nufft(m: int = 8192, n: int = 16384, lam: float = 1e-2, seed: int = 0,
             item: int = 0, chunk: int = 256):
    """Config 4: nonuniform Fourier sampling T_kj = exp(-2 pi i f_k j),
    f_k ~ U[0,1); G = T^H T by its first column g_r = sum_k exp(2 pi i f_k r);
    x complex N(0,1); b = T x + complex N(0,1e-4); rhs = T^H b; L = lam * I.
    (Setup only; O(mn) exponential sums, done in row chunks.)"""
    rng = rng_for(seed, 4, item)
    f = rng.uniform(0.0, 1.0, m)
    x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2.0)
    noise = 1e-2 * (rng.standard_normal(m) + 1j * rng.standard_normal(m)) / np.sqrt(2.0)
    j = np.arange(n, dtype=np.float64)
    g = np.zeros(n, dtype=np.complex128)
    b = np.empty(m, dtype=np.complex128)
    rows = []
    for s in range(0, m, chunk):
        ph = np.exp(-2j * np.pi * np.outer(f[s:s + chunk], j))
        b[s:s + chunk] = ph @ x + noise[s:s + chunk]
        g += np.conj(ph).sum(axis=0)
        rows.append(s)
    rhs = np.zeros(n, dtype=np.complex128)
    for s in rows:
        ph = np.exp(-2j * np.pi * np.outer(f[s:s + chunk], j))
        rhs += np.conj(ph).T @ b[s:s + chunk]
    g[0] = g[0].real
    lgen = np.zeros(2 * n - 1, dtype=np.complex128)
    lgen[n - 1] = lam
    return {"variant": "gramian", "m": n, "n": n, "G_col": g, "L_rows": n,
            "L_gen": lgen, "normal_rhs": rhs, "x_true": x}


def c5_random(n: int = 16384, count: int = 1, seed: int = 0, first: int = 0,
              lam: float = 1e-1):
    """Config 5: independent square systems, kernel and rhs i.i.d.
    N(0,1)/sqrt(n), L = I, lambda = 0.1.  Item i uses stream (seed, 5, i)."""
    gens, bs = [], []
    for i in range(first, first + count):
        rng = rng_for(seed, 5, i)
        gens.append(_cplx(rng.standard_normal(2 * n - 1) / np.sqrt(n)))
        bs.append(_cplx(rng.standard_normal(n) / np.sqrt(n)))
    return {"variant": "l2", "m": n, "n": n, "T_gen": np.stack(gens),
            "beta": lam, "b": np.stack(bs)}


def random_problem(variant: str, n: int, rng: np.random.Generator):
    """Square random instance with the reference's random_problem
    distribution (ref: experiments.py:88-106), as a raw dict."""
    def cn(size):
        return (rng.standard_normal(size) + 1j * rng.standard_normal(size)) / np.sqrt(2.0)

    if variant == "general":
        tg = cn(2 * n - 1)
        lg = cn(2 * n - 1)
        return {"variant": "general", "m": n, "n": n, "T_gen": tg, "L_rows": n,
                "L_gen": lg, "b": cn(n)}
    if variant == "l2":
        tg = cn(2 * n - 1)
        return {"variant": "l2", "m": n, "n": n, "T_gen": tg, "beta": n ** 0.25,
                "b": cn(n)}
    if variant == "gramian":
        col = np.empty(n, dtype=np.complex128)
        col[0] = 10.0 * np.sqrt(n)
        col[1:] = cn(n - 1)
        lg = cn(2 * n - 1)
        return {"variant": "gramian", "m": n, "n": n, "G_col": col, "L_rows": n,
                "L_gen": lg, "normal_rhs": cn(n)}
    raise ValueError(variant)


def to_problem(d, mod, index=None):
    """Build ``mod.ProblemSpec`` (ours or the reference's) from a raw dict.
    ``index`` picks one item from batched arrays (leading axis)."""
    def pick(key):
        v = d.get(key)
        if v is None:
            return None
        v = np.asarray(v)
        if index is not None and v.ndim == 2:
            return v[index]
        return v

    variant = d["variant"]
    if variant == "l2":
        T = mod.ToeplitzSpec(d["m"], d["n"], pick("T_gen"))
        if d.get("normal_rhs") is not None:
            return mod.ProblemSpec(variant="l2", T=T, beta=complex(d["beta"]),
                                   b=None, normal_rhs=pick("normal_rhs"))
        return mod.ProblemSpec.l2(T, d["beta"], pick("b"))
    if variant == "general":
        T = mod.ToeplitzSpec(d["m"], d["n"], pick("T_gen"))
        L = mod.ToeplitzSpec(d["L_rows"], d["n"], pick("L_gen"))
        if d.get("normal_rhs") is not None:
            return mod.ProblemSpec(variant="general", T=T, L=L, b=None,
                                   normal_rhs=pick("normal_rhs"))
        return mod.ProblemSpec.general(T, L, pick("b"))
    if variant == "gramian":
        G = mod.HermitianToeplitzSpec(d["n"], pick("G_col"))
        L = mod.ToeplitzSpec(d["L_rows"], d["n"], pick("L_gen"))
        return mod.ProblemSpec.gramian(G, L, pick("normal_rhs"))
    raise ValueError(variant)
