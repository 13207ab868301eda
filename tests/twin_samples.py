"""Seeded sample indices and projection weights of the config-5 n=24 twins
(SURVEY.md §8(c) c.4 (iv)).  Input generation only: no arithmetic of the
method.  Shared by tools/make_golden.py (oracle side) and
tests/test_gpu_fullsize.py (CUDA side)."""
from __future__ import annotations

import numpy as np

TWIN_N = 24
TWIN_NS = (24, 26)          # reduced twins of config 5 with golden oracle files
TWIN_SAMPLES = 4096
_SEED = 251223183 + 50


def twin_indices(n: int, m: int) -> np.ndarray:
    rng = np.random.default_rng(_SEED + m)
    return np.sort(rng.choice(1 << n, size=TWIN_SAMPLES, replace=False)).astype(np.int64)


def twin_weights(n: int, count: int = 3):
    """``count`` vectors of +-1.0 over all 2^n indices."""
    rng = np.random.default_rng(_SEED)
    return [rng.integers(0, 2, size=1 << n).astype(np.float64) * 2.0 - 1.0 for _ in range(count)]
