"""Compare the GPU leaf sweep (tr_leaf) with the oracle's leaf on the first
leaves of a few problems (weights from the GPU assembly)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import toepreg_oracle as O  # noqa: E402
import paper_1302_6945_b200 as tb  # noqa: E402
from paper_1302_6945_b200 import _lib, workloads as wl  # noqa: E402

lib = _lib.load()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128).view(np.float64).copy()).cuda()


def run(label, raw, index=None):
    prob = wl.to_problem(raw, tb, index)
    asm = O.assemble(wl.to_problem(raw, tb, index))
    v, m, n, pl = tb.solver._shape(prob)
    d = tb.solver.make_desc(v, m, n, pl, tb.SolverConfig())
    W = asm.weights                        # (rows, N, P)
    Wd = dev(np.ascontiguousarray(np.transpose(W, (1, 0, 2))))
    rows, N, P = W.shape
    # first leaf per the reference tree walk
    offsets, stride = (0,), 1
    while rows * len(offsets) * (N // stride) > 256:
        cut = O.split_rule(N, offsets, stride, True)
        offsets, _, stride = cut
    idx = O.coset_indices(N, offsets, stride)
    K = rows * idx.size
    cap = K + 1
    degs = -asm.tau.copy()
    coeffs, d_ref, deferred, factor, res, attempts = O.leaf_basis(W, asm.nodes, idx, degs.copy(), 1e-8)
    cd = (C.c_int64 * 8)(*([int(x) for x in degs] + [0] * (8 - P)))
    out = torch.zeros((P * P * cap * 2,), dtype=torch.float64, device="cuda")
    nd, att = C.c_int32(), C.c_int32()
    rr = C.c_double()
    rc = lib.tr_leaf(C.byref(d), C.c_void_p(Wd.data_ptr()), 0, cd, C.c_void_p(out.data_ptr()), cap,
                     C.byref(nd), C.byref(rr), C.byref(att), None)
    if rc:
        print(label, "rc", rc, _lib.last_error())
        return
    torch.cuda.synchronize()
    g = out.cpu().numpy().view(np.complex128).reshape(P, P, cap)
    L = coeffs.shape[2]
    diff = np.abs(g[:, :, :L] - coeffs).max() / np.abs(coeffs).max()
    print(f"{label}: K={K} degs gpu={list(cd)[:P]} ref={list(d_ref)} ndef gpu={nd.value} ref={len(deferred)} "
          f"res gpu={rr.value:.2e} ref={res:.2e} attempts ref={attempts} basis maxdiff/max={diff:.2e} "
          f"tail={np.abs(g[:, :, L:]).max() if cap > L else 0:.1e}")


if __name__ == "__main__":
    print("legacy" if os.environ.get("TR_LEAF_LEGACY") else "leaf2")
    run("c1", wl.c1_blur(256))
    run("c2mini", wl.c2_rect(m=1024, n=512, nrhs=1), 0)
    run("c5mini", wl.c5_random(n=2048, count=1), 0)
    run("c3mini", wl.c3_firstdiff(n=512, lam=1e-2))
    run("rand64_general", wl.random_problem("general", 64, np.random.default_rng(5)))
