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

Where the secret, keys and encryption randomness come from is the caller's
choice: ``SystemRng`` (the default of a context, ``HEParams.seed=None``) draws
from the operating system's CSPRNG; a seeded NumPy PCG64 generator is the
explicit, INSECURE opt-in that word-parity tests and benchmarks use to hand the
CPU oracle the same randomness.
"""
from __future__ import annotations

import math
import os

import numpy as np


class SystemRng:
    """The ``integers`` / ``normal`` subset of ``numpy.random.Generator`` used by the samplers,
    backed by ``os.urandom`` (uniform integers by rejection on masked 64-bit words; normals by
    Box-Muller on 53-bit uniforms)."""

    @staticmethod
    def _words(count: int) -> np.ndarray:
        return np.frombuffer(os.urandom(8 * count), dtype=np.uint64)

    def integers(self, low, high, size, dtype=np.int64):
        low, high = int(low), int(high)
        span = high - low
        if span <= 0:
            raise ValueError("empty range")
        shape = (size,) if isinstance(size, (int, np.integer)) else tuple(size)
        count = int(np.prod(shape))
        mask = np.uint64((1 << max(1, (span - 1).bit_length())) - 1) if span > 1 else np.uint64(0)
        out = np.empty(0, dtype=np.uint64)
        while out.size < count:
            w = self._words(max(64, 2 * (count - out.size))) & mask
            out = np.concatenate([out, w[w < np.uint64(span)]])
        vals = out[:count]
        if low >= 0:
            res = (vals + np.uint64(low)).astype(dtype)
        else:
            res = (vals.astype(np.int64) + low).astype(dtype)
        return res.reshape(shape)

    def normal(self, loc, scale, size):
        shape = (size,) if isinstance(size, (int, np.integer)) else tuple(size)
        count = int(np.prod(shape))
        half = (count + 1) // 2
        u = (self._words(2 * half) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
        u1, u2 = 1.0 - u[:half], u[half:]                 # u1 in (0, 1]
        r = np.sqrt(-2.0 * np.log(u1))
        z = np.concatenate([r * np.cos(2 * math.pi * u2), r * np.sin(2 * math.pi * u2)])[:count]
        return (loc + scale * z).reshape(shape)


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
