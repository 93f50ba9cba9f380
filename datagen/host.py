"""numpy stand-in generator for CPU-only tests (harness; no method arithmetic).

It draws from the same distributions as gen.cu, but not the same bits. GPU parity tests
always use the device generator and copy its bytes to the oracle.
"""
from __future__ import annotations

import numpy as np


def walks(N: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.cumsum(rng.standard_normal((N, n)), axis=1).astype(np.float32)


def sines(N: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    c = rng.uniform(1, 20, (N, 3, 1))
    ph = rng.uniform(0, 2 * np.pi, (N, 3, 1))
    a = rng.standard_normal((N, 3, 1))
    t = np.arange(n)[None, None, :]
    x = (a * np.sin(2 * np.pi * c * t / n + ph)).sum(1) + 0.3 * rng.standard_normal((N, n))
    return x.astype(np.float32)
