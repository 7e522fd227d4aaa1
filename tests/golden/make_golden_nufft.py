"""Golden fixtures for the NUFFT setup and driver, made by running the
REFERENCE (read-only at /root/reference) in the build container:

    python tests/golden/make_golden_nufft.py

Stores weighted_fourier_gramian (ref: pkg/src/toepreg/nufft.py:60-72), the
dense samples A x and rhs A^H (w * samples) (ref :106-114) for a seeded
triangular frequency draw, and run_nufft(NufftConfig(n=256, samples=320)).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from toepreg import nufft as rn  # noqa: E402  (the reference, read-only)

STAGE = os.path.join(HERE, "stages")


def main():
    os.makedirs(STAGE, exist_ok=True)
    rng = np.random.default_rng(np.random.SeedSequence((7, 93)))
    freqs = rng.triangular(-0.5, 0.0, 0.5, size=300)
    w = rn.voronoi_weights(freqs)
    x = rn.make_signal(256, 3, 0.02, rng)
    a = rn.sample_matrix(freqs, 256)
    samples = a @ x
    rhs = a.conj().T @ (w * samples)
    gram = rn.weighted_fourier_gramian(freqs, w, 256)
    # large lags: phases up to 2 pi f d with d ~ 2e4 (accuracy of the phase reduction)
    gram_big = rn.weighted_fourier_gramian(freqs[:64], w[:64], 20000)
    out = rn.run_nufft(rn.NufftConfig(n=256, samples=320))
    np.savez_compressed(os.path.join(STAGE, "nufft.npz"), freqs=freqs, weights=w, x=x, samples=samples,
                        rhs=rhs, gram=np.asarray(gram.gen), gram_big=np.asarray(gram_big.gen),
                        run_x=np.array(out["x_direct_re"]) + 1j * np.array(out["x_direct_im"]),
                        run_err=np.array(out["rel_err_direct"]), run_dp=np.array(out["difficult_points"]),
                        run_wsum=np.array(out["weights_sum"]))
    print("rel_err_direct", out["rel_err_direct"], "dp", out["difficult_points"])


if __name__ == "__main__":
    main()
