"""Plaintext truth for the side benchmarks in tools/ (exact int64 numpy; verification only)."""
import numpy as np


def dot_mod_p(w, x, p):
    w = np.asarray(w, dtype=np.int64) % p
    x = np.asarray(x, dtype=np.int64) % p
    return (w * x).sum(axis=1) % p if w.shape[1] <= 4096 else None


def conv2d_mod_p(x, w, p, stride=1):
    x = np.asarray(x, dtype=np.int64) % p
    w = np.asarray(w, dtype=np.int64) % p
    c_i, s, _ = x.shape
    k, h = w.shape[2], w.shape[2] // 2
    xp = np.zeros((c_i, s + 2 * h, s + 2 * h), dtype=np.int64)
    xp[:, h:h + s, h:h + s] = x
    out = np.zeros((w.shape[0], s, s), dtype=np.int64)
    for dy in range(k):
        for dx in range(k):
            win = xp[:, dy:dy + s, dx:dx + s].reshape(c_i, -1)
            out += (w[:, :, dy, dx] @ win % p).reshape(-1, s, s)
            out %= p
    return out[:, ::stride, ::stride]
