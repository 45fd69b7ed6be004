"""Seeded synthetic data for the golden cases whose base vectors are not stored.

``mix_data`` is a Gaussian mixture drawn with NumPy's default_rng (PCG64), whose
stream is fixed for a given NumPy version; the generator (gen_golden.py) and the
tests (conftest.load_case) call the same function, so the stored fixtures only
carry what the reference computed from it.
"""

from __future__ import annotations

import numpy as np


def mix_data(n: int, nq: int, dims: int, seed: int):
    rng = np.random.default_rng(4000 + seed)
    centres = rng.standard_normal((12, dims)) * 2.0
    x = (centres[rng.integers(0, 12, n)] + rng.standard_normal((n, dims))).astype(np.float32)
    q = centres[rng.integers(0, 12, nq)] + rng.standard_normal((nq, dims))
    return x, q
