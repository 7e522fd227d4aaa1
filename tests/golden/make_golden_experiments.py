"""Golden fixtures for the experiment drivers, made by running the REFERENCE
(read-only at /root/reference) in the build container:

    python tests/golden/make_golden_experiments.py

Stores the reference's random_problem draws (generator checksums) for the
accuracy / cg streams, run_accuracy rows for small sizes and a
fit_complexity result on fixed data (ref: pkg/src/toepreg/experiments.py).
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from toepreg import experiments as rx  # noqa: E402  (the reference, read-only)

STAGE = os.path.join(HERE, "stages")


def main():
    cfg = rx.ExperimentConfig(sizes=(16, 32), trials=2, seed=2024)
    out = {"accuracy": rx.run_accuracy(cfg)}
    draws = {}
    for variant in rx.VARIANTS:
        rng = rx._trial_rng(2024, "accuracy", variant, 16, 1)
        p = rx.random_problem(variant, 16, rng)
        x = rx.complex_normal(rng, 16)
        parts = [p.T.gen if p.T is not None else np.zeros(0), p.L.gen if p.L is not None else np.zeros(0),
                 p.G.gen if p.G is not None else np.zeros(0), p.b if p.b is not None else np.zeros(0), x]
        draws[variant] = [float(np.abs(np.concatenate([np.ravel(q) for q in parts])).sum()),
                          float(abs(p.beta)) if p.beta is not None else 0.0]
    out["draws"] = draws
    fit = rx.fit_complexity([256, 512, 1024, 2048], [0.011, 0.026, 0.060, 0.135])
    out["fit"] = [fit.c1, fit.c2, fit.r_squared]
    out["free_parameters"] = {v: rx.free_parameters(v, 100) for v in rx.VARIANTS}
    with open(os.path.join(STAGE, "experiments.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out)[:400])


if __name__ == "__main__":
    main()
