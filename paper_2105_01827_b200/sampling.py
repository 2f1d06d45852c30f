"""Host-supplied randomness for keys and encryptions.

The north_star contract is "the same ciphertext words given the same
host-supplied randomness": every random polynomial is drawn here, on the
host, from a NumPy ``Generator`` and handed to the CUDA library (and, in the
tests, to the CPU oracle) as plain integer arrays.  The samplers are pinned:

* secret      ternary, ``rng.integers(-1, 2, N)``
* uniform     ``rng.integers(0, q_j, N, dtype=uint64)`` per prime, coefficient domain
* error       rounded Gaussian, sigma = HEParams.sigma (3.2), tail-cut at 6 sigma
* mask r      ``default_rng(seed).integers(0, p, n, dtype=int64)`` exactly as the
              reference draws it (``pkg/src/gala/sharing.py:42-44``)
"""
from __future__ import annotations

import numpy as np


def secret(rng: np.random.Generator, N: int) -> np.ndarray:
    return rng.integers(-1, 2, N).astype(np.int8)


def uniform(rng: np.random.Generator, moduli, N: int) -> np.ndarray:
    out = np.empty((len(moduli), N), dtype=np.uint64)
    for j, q in enumerate(moduli):
        out[j] = rng.integers(0, q, N, dtype=np.uint64)
    return out


def gaussian(rng: np.random.Generator, N: int, sigma: float = 3.2, rows: int | None = None) -> np.ndarray:
    shape = (N,) if rows is None else (rows, N)
    bound = int(np.ceil(6 * sigma))
    e = np.rint(rng.normal(0.0, sigma, shape))
    return np.clip(e, -bound, bound).astype(np.int64)


def encryption_randomness(rng, bfv, sigma: float = 3.2):
    """(a [L][N] uniform, e [N]) for one symmetric-key encryption."""
    return uniform(rng, bfv.primes, bfv.N), gaussian(rng, bfv.N, sigma)


def rotation_key_randomness(rng, bfv, sigma: float = 3.2):
    """(a [L][L+1][N] uniform, e [L][N]) for one rotation key."""
    a = np.stack([uniform(rng, bfv.all_primes, bfv.N) for _ in range(bfv.L)])
    return a, gaussian(rng, bfv.N, sigma, rows=bfv.L)
