"""Generates tests/golden/fmnm_v2_small.bin with the oracle's independent
restatement of the FMNM v2 container (oracle/fmnm.py, io.cpp:49-82), from a
seeded model shaped like test_io.cpp:17-38 (layout {2, 3}, two per-block
models over 4 bins x 6 frames, 2 sources, 3 bases).  Run from the repo root:

  python tests/golden/make_fmnm_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import fmnm  # noqa: E402


def instance(seed=1):
    rng = np.random.default_rng(seed)
    F, J, N, K, sizes = 4, 6, 2, 3, [2, 3]
    models = [(1e-6 + rng.random((N, F, K)), 1e-6 + rng.random((N, K, J))) for _ in range(2)]
    lam = rng.random((F, N, sum(sizes)))
    w = [rng.standard_normal((F, mb, mb)) + 1j * rng.standard_normal((F, mb, mb)) for mb in sizes]
    cfg = dict(n_sources=N, k_bases=K, iterations=17, floor=1e-6, seed=seed, sample_rate=8000.0, window_len=256,
               hop_len=64)
    return cfg, sizes, False, models, lam, w


if __name__ == "__main__":
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fmnm_v2_small.bin")
    fmnm.write(out, *instance())
    print(out, os.path.getsize(out), "bytes")
