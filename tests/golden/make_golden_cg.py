"""Golden fixtures for the normal operator and conjugate gradients, made by
running the REFERENCE (read-only at /root/reference) in the build container:

    python tests/golden/make_golden_cg.py

For one small problem per variant it stores the inputs, NormalOperator.apply
of a seeded vector (ref: pkg/src/toepreg/solver.py:104-167) and cg_solve at
the default tolerance and at a 5-iteration cap (ref: solver.py:184-215).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import toepreg  # noqa: E402  (the reference, read-only)
from paper_1302_6945_b200 import workloads as wl  # noqa: E402

STAGE = os.path.join(HERE, "stages")


def main():
    os.makedirs(STAGE, exist_ok=True)
    for code, variant in enumerate(("general", "l2", "gramian")):
        rng = np.random.default_rng(np.random.SeedSequence((4242, code, 96)))
        raw = wl.random_problem(variant, 96, rng)
        prob = wl.to_problem(raw, toepreg)
        x = rng.standard_normal(96) + 1j * rng.standard_normal(96)
        op = toepreg.NormalOperator(prob)
        ax = op.apply(x)
        xc, it = toepreg.cg_solve(prob)
        x5, it5 = toepreg.cg_solve(prob, toepreg.CGConfig(max_iterations=5))
        extra = {k: np.asarray(raw[k]) for k in ("T_gen", "L_gen", "G_col", "b", "normal_rhs")
                 if raw.get(k) is not None}
        for k in ("beta", "L_rows"):
            if raw.get(k) is not None:
                extra[k] = np.array(raw[k])
        np.savez_compressed(os.path.join(STAGE, f"cg_{variant}_n96.npz"), variant=np.array(variant),
                            m=np.array(raw["m"]), n=np.array(raw["n"]), x=x, ax=ax,
                            transforms=np.array(op.transforms), x_cg=xc, it_cg=np.array(it),
                            x_cg5=x5, it_cg5=np.array(it5), **extra)
        print(variant, "cg iterations", it, "transforms/apply", op.transforms)


if __name__ == "__main__":
    main()
