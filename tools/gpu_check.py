"""Quick GPU diagnostics (run under gpurun): stage and end-to-end parity
against numpy, the golden fixtures and the oracle, plus rough timings."""

import ctypes as C
import glob
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_1302_6945_b200 as tb  # noqa: E402
from paper_1302_6945_b200 import _lib, workloads as wl  # noqa: E402

lib = _lib.load()
GOLD = os.path.join(ROOT, "tests", "golden")


def dev(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return torch.from_numpy(a.view(np.float64).copy()).cuda()


def host(t):
    return t.cpu().numpy().view(np.complex128)


def p(t):
    return C.c_void_p(t.data_ptr())


def rel(a, b):
    d = np.linalg.norm(np.ravel(a) - np.ravel(b))
    nb = np.linalg.norm(np.ravel(b))
    return d / (nb if nb > 0 else 1.0)


def check_fft():
    rng = np.random.default_rng(0)
    for n in (1, 2, 3, 8, 48, 64, 96, 1024, 4096, 6144, 12288, 32768, 65536, 98304, 1 << 20,
              3 << 18, 1 << 21):
        lines = max(1, min(8, (1 << 22) // n))
        x = rng.standard_normal((lines, n)) + 1j * rng.standard_normal((lines, n))
        dx = dev(x)
        out = torch.empty_like(dx)
        for sign in (-1, 1):
            rc = lib.tr_fft(p(dx), p(out), n, lines, sign, None)
            assert rc == 0, _lib.last_error()
            ref = np.fft.fft(x, axis=-1) if sign < 0 else n * np.fft.ifft(x, axis=-1)
            print(f"fft n={n:8d} sign={sign:+d} rel={rel(host(out).reshape(lines, n), ref):.2e}")


def check_stages():
    g = np.load(os.path.join(GOLD, "stages", "grid_eval.npz"))
    cube = g["cube"]
    for key in g.files:
        if not key.startswith("N"):
            continue
        N, off, st = [int(s[1:]) for s in key.split("_")]
        cnt = N // st
        lines = cube.shape[0] * cube.shape[1]
        out = torch.empty((lines, cnt, 2), dtype=torch.float64, device="cuda")
        rc = lib.tr_grid_eval(p(dev(cube.reshape(lines, -1))), lines, cube.shape[2], N, off, st,
                              p(out), None)
        assert rc == 0, _lib.last_error()
        print(f"grid_eval {key}: rel={rel(host(out).reshape(g[key].shape), g[key]):.2e}")
    m = np.load(os.path.join(GOLD, "stages", "matpoly.npz"))
    a, b = m["a"], m["b"]
    L = a.shape[2] + b.shape[2] - 1
    out = torch.empty((25, L, 2), dtype=torch.float64, device="cuda")
    rc = lib.tr_matpoly_mul(p(dev(a)), a.shape[2], p(dev(b)), b.shape[2], 5, p(out), None)
    assert rc == 0, _lib.last_error()
    got = host(out).reshape(5, 5, L)
    print(f"matpoly vs LD: rel={rel(got, m['ld']):.2e}  maxabs/max={np.abs(got - m['ld']).max() / np.abs(m['ld']).max():.2e}"
          f"  (ref f64 vs LD: {np.abs(m['f64'] - m['ld']).max() / np.abs(m['ld']).max():.2e})")
    for name in ("assemble_l2_n64", "assemble_general_n32", "assemble_gramian_n32"):
        a = dict(np.load(os.path.join(GOLD, "stages", name + ".npz")))
        W = a["weights"]
        rows, N, P = W.shape
        if "general" in name:
            var, n, m, pl = "general", 32, 32, int(a["L_rows"])
        elif "gramian" in name:
            var, n, m, pl = "gramian", 32, 32, int(a["L_rows"])
        else:
            var, n, m, pl = "l2", 64, 64, 64
        d = tb.solver.make_desc(var, m, n, pl, tb.SolverConfig())
        out = torch.zeros((N, rows, P, 2), dtype=torch.float64, device="cuda")
        tg = dev(a["T_gen"]) if "T_gen" in a else None
        lg = dev(a["L_gen"]) if "L_gen" in a else None
        gc = dev(a["G_col"]) if "G_col" in a else None
        bsq = torch.tensor([abs(float(a["beta"])) ** 2], dtype=torch.float64, device="cuda") if "beta" in a else None
        rhs = dev(a["normal_rhs"]) if "normal_rhs" in a else dev(a["b"])
        rc = lib.tr_assemble(C.byref(d), p(tg) if tg is not None else None, p(lg) if lg is not None else None,
                             p(gc) if gc is not None else None, p(bsq) if bsq is not None else None,
                             p(rhs), int("normal_rhs" in a), p(out), None)
        assert rc == 0, _lib.last_error()
        got = np.transpose(host(out).reshape(N, rows, P), (1, 0, 2))
        print(f"{name}: rel={rel(got, W):.2e} maxabs={np.abs(got - W).max():.2e}")


def load_case(f):
    d = dict(np.load(f))
    raw = {k: (v.item() if v.ndim == 0 else v) for k, v in d.items()}
    raw["variant"] = str(d["variant"])
    if "recipe" in d:
        r = str(d["recipe"])
        if r.startswith("c2_rect"):
            raw.update({k: v for k, v in wl.c2_rect(nrhs=1, seed=0).items()})
            raw["b"] = raw["b"][0]
        elif r.startswith("c5_random"):
            src = wl.c5_random(n=16384, count=1, seed=0)
            raw["T_gen"], raw["b"] = src["T_gen"][0], src["b"][0]
            raw["beta"] = src["beta"]
    return raw, d


def check_solves(refine):
    cfg = tb.SolverConfig(refine=refine)
    print(f"---- end-to-end, refine={refine}")
    worst = 0.0
    for f in sorted(glob.glob(os.path.join(GOLD, "cases", "*.npz"))):
        name = os.path.basename(f)[:-4]
        raw, d = load_case(f)
        prob = wl.to_problem(raw, tb)
        t0 = time.perf_counter()
        try:
            rep = tb.solve_tikhonov(prob, cfg)
        except Exception as e:  # noqa: BLE001
            print(f"{name:28s} FAILED {type(e).__name__}: {e}")
            continue
        dt = time.perf_counter() - t0
        x = rep.x_hat
        e_ref = rel(x, d["x_hat"])
        e_ex = rel(x, d["x_exact"])
        r_ex = rel(d["x_hat"], d["x_exact"])
        worst = max(worst, e_ref)
        dg = rep.diagnostics
        print(f"{name:28s} gpu<->ref={e_ref:.2e} gpu<->exact={e_ex:.2e} ref<->exact={r_ex:.2e} "
              f"degs={'ok' if np.array_equal(np.sort(rep.final_col_degrees), np.sort(d['final_col_degrees'])) else rep.final_col_degrees} "
              f"dp={dg.difficult_points}/{int(d['difficult_points'])} retried={dg.retried_leaves} "
              f"res={rep.relative_residual:.1e}/{float(d['relative_residual']):.1e} "
              f"scale={dg.max_column_scale:.3g}/{float(d['max_column_scale']):.3g} tro={dg.trim_overflow} {dt*1e3:.1f}ms")
    return worst


def check_determinism():
    raw = wl.c5_random(n=2048, count=4, seed=3)
    probs = [wl.to_problem(raw, tb, i) for i in range(4)]
    a = tb.solve_tikhonov_batch(probs)
    b = tb.solve_tikhonov_batch(probs)
    same = all(np.array_equal(x.x_hat, y.x_hat) for x, y in zip(a, b))
    single = tb.solve_tikhonov(probs[2])
    print(f"determinism batch-vs-batch bitwise={same}; batch-vs-single bitwise="
          f"{np.array_equal(single.x_hat, a[2].x_hat)}")


def timing():
    for label, raw, count in (("c2 full 64 rhs", wl.c2_rect(nrhs=64, seed=0), 64),
                              ("c5 n=16384 x 64", wl.c5_random(n=16384, count=64, seed=0), 64)):
        probs = [wl.to_problem(raw, tb, i) for i in range(count)]
        db = tb.DeviceBatch(probs).stage()
        db.run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            db.run(with_diag=False)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"timing {label}: {t*1e3:.1f} ms per batch -> {count / t:.1f} solves/s")


if __name__ == "__main__":
    which = sys.argv[1:] or ["fft", "stages", "solves", "det", "time"]
    if "fft" in which:
        check_fft()
    if "stages" in which:
        check_stages()
    if "solves" in which:
        check_solves(0)
        check_solves(1)
    if "det" in which:
        check_determinism()
    if "time" in which:
        timing()
