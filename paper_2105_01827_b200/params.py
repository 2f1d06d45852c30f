"""BFV parameter derivation for the GPU backend (host side, pure Python ints).

The reference's ``HEParams`` (``pkg/src/gala/backend.py:80-114``) only names a
slot count ``n`` and a plaintext prime ``p``; its backend is a mock.  A real
RNS-BFV backend needs a ring degree, ciphertext primes, a key-switching
special prime and primitive roots.  This module derives them
deterministically from ``(n, p, rns_limbs)`` so that the CUDA library and the
CPU oracle (``oracle/``) are always built on the same numbers:

* ring degree ``N = 2 n`` -- one logical slot vector per hypercube row
  (slot mapping option A); the two rows rotate
  independently under the Galois element ``3^k mod 2N``.
* ``p`` must satisfy ``p = 1 (mod 2N)`` (batching).  The reference default
  1048573 does not; 1032193 = 2^14 * 63 + 1 does for every N <= 8192.
* every ciphertext and special prime has the *special form* ``q = a 2^32 + 1``
  (so ``q = 1 (mod 2N)`` for every N <= 8192): the CUDA NTT's Shoup reduction
  then needs one 32-bit multiply for ``hi * q`` instead of a 64x64 product.
* ``rns_limbs == 1`` (BASELINE configs 1 and 3 select it explicitly): one
  ciphertext prime ``q < 2^62`` with ``q = 1 (mod 2^32 p)`` so the BFV
  plaintext-product rounding term ``(q mod p) * k`` collapses to ``k``
  (SURVEY.md A.3).  Delta / 2 = 2^41 holds one convolution or dot product of
  the configs' sizes, not more.
* ``rns_limbs`` 2..4: the largest special-form primes below 2^60.  The default
  is 2 for N <= 4096 -- the smallest modulus under which every circuit the
  reference's own test suite runs (Table VII row 4: 51 200 rotate-then-multiply
  terms, measured at 0.49 Delta with one prime) decrypts with room to spare --
  and 3 for N = 8192.
* one special prime ``P`` (hybrid key switching, one digit per ciphertext
  prime): the largest special-form prime below 2^62 (L = 1) or the next one
  below the ciphertext primes (L = 3).

Roots: for every modulus m the primitive 2N-th root is ``g^((m-1)/2N)`` with
``g`` the smallest quadratic non-residue mod m.  The plaintext root pins the
slot encoding (slot (r, c) <-> evaluation at zeta^(+-3^c)).
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

MAX_N = 8192
_SMALL = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(x: int) -> bool:
    """Deterministic Miller-Rabin for x < 3.3e24 (same bases as backend.py:38-61)."""
    if x < 2:
        return False
    for q in _SMALL:
        if x % q == 0:
            return x == q
    d, r = x - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in _SMALL:
        y = pow(a, d, x)
        if y in (1, x - 1):
            continue
        for _ in range(r - 1):
            y = y * y % x
            if y == x - 1:
                break
        else:
            return False
    return True


def _primes_below(bound_bits: int, modulus: int, count: int, exclude=()) -> list[int]:
    out = []
    k = ((1 << bound_bits) - 1) // modulus
    while len(out) < count:
        c = k * modulus + 1
        if c > 1 and is_prime(c) and c not in exclude:
            out.append(c)
        k -= 1
        if k <= 0:
            raise ValueError("prime search exhausted")
    return out


def primitive_root_2n(m: int, two_n: int) -> int:
    """psi of order exactly 2N mod prime m: g^((m-1)/2N), g least non-residue."""
    if (m - 1) % two_n:
        raise ValueError(f"{m} is not 1 mod {two_n}")
    g = 2
    while pow(g, (m - 1) // 2, m) == 1:
        g += 1
    psi = pow(g, (m - 1) // two_n, m)
    assert pow(psi, two_n // 2, m) == m - 1
    return psi


@dataclass(frozen=True)
class BFVParams:
    """Concrete RNS-BFV instance: ring degree, primes, roots."""

    N: int
    p: int
    primes: tuple[int, ...]      # L ciphertext primes q_0..q_{L-1}
    special: int                 # key-switching prime P (K = 1)
    psis: tuple[int, ...]        # primitive 2N-th roots for primes + (special,)
    psi_p: int                   # primitive 2N-th root mod p (slot encoding)

    @property
    def L(self) -> int:
        return len(self.primes)

    @property
    def n(self) -> int:
        return self.N // 2

    @property
    def all_primes(self) -> tuple[int, ...]:
        return self.primes + (self.special,)

    @property
    def Q(self) -> int:
        out = 1
        for q in self.primes:
            out *= q
        return out

    @property
    def delta(self) -> int:
        return self.Q // self.p

    def log2_budget(self) -> float:
        import math
        return math.log2(self.delta / 2)


def default_limbs(N: int) -> int:
    return 2 if N <= 4096 else 3


@lru_cache(maxsize=None)
def derive(n: int, p: int, rns_limbs: int | None = None) -> BFVParams:
    """BFV parameters for logical slot count n (ring degree N = 2n)."""
    N = 2 * n
    if N < 8 or N > MAX_N or N & (N - 1):
        raise ValueError(f"ring degree N = 2n = {N} must be a power of two in [8, {MAX_N}]")
    if (p - 1) % (2 * N):
        raise ValueError(f"p = {p} is not 1 mod 2N = {2 * N}: slot batching impossible")
    L = rns_limbs or default_limbs(N)
    SF = 1 << 32      # special form q = a 2^32 + 1 (also 1 mod 2N since 2N <= 2^14)
    if L == 1:
        primes = tuple(_primes_below(62, SF * p, 1))
        special = _primes_below(62, SF, 1, exclude=primes)[0]
    elif L in (2, 3, 4):
        primes = tuple(_primes_below(60, SF, L))
        special = _primes_below(60, SF, 1, exclude=primes)[0]
    else:
        raise ValueError("rns_limbs must be 1..4")
    psis = tuple(primitive_root_2n(m, 2 * N) for m in primes + (special,))
    return BFVParams(N, p, primes, special, psis, primitive_root_2n(p, 2 * N))


def galois_element(step: int, N: int) -> int:
    """Galois element 3^step mod 2N: left rotation of both rows by `step`."""
    n = N // 2
    return pow(3, step % n, 2 * N)
