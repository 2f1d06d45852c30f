"""Shared setup for parity tests: one GPU context and one CPU oracle built on
the same BFV parameters, secret and key randomness (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle.bfv import Oracle
from paper_2105_01827_b200 import sampling
from paper_2105_01827_b200.backend import Context, HEParams

P = 1032193


class Twin:
    def __init__(self, n: int, rns_limbs: int | None = None, seed: int = 11):
        self.params = HEParams(n=n, p=P, rns_limbs=rns_limbs, seed=seed)
        self.bfv = self.params.bfv()
        self.N, self.L = self.bfv.N, self.bfv.L
        self.rng = np.random.default_rng(seed)
        s = sampling.secret(self.rng, self.N)
        self.gpu = Context(self.params, secret=s)
        self.cpu = Oracle(self.bfv)
        self.cpu.set_secret(s)
        self.keys = set()

    def keys_for(self, steps):
        for st in steps:
            st = st % self.bfv.n
            if st == 0 or st in self.keys:
                continue
            a, e = sampling.rotation_key_randomness(self.rng, self.bfv)
            self.gpu.gen_rotation_key(st, a, e)
            self.cpu.gen_rotkey(st, a, e)
            self.keys.add(st)

    def slots(self, count=None):
        shape = (self.N,) if count is None else (count, self.N)
        return self.rng.integers(0, P, shape).astype(np.uint32)

    def encrypt(self, phys):
        a, e = sampling.encryption_randomness(self.rng, self.bfv)
        return self.gpu.encrypt_physical(phys, a, e), self.cpu.encrypt(phys, a, e)


class Mirror:
    """The product's own (cached, seeded) context and a CPU oracle holding the same secret and the
    same rotation keys: the seeded context derives them from PCG64 streams keyed by (seed, tag)
    (backend.Context._rng), which the mirror replays.  Lets the tests drive the product's layer
    objects (GalaFC, KernelGroupingConv, ConvLayer) end to end and compare their words."""

    def __init__(self, params):
        from paper_2105_01827_b200.backend import context

        assert params.seed is not None, "word parity needs a seeded (reproducible) context"
        self.params = params
        self.bfv = params.bfv()
        self.N, self.L = self.bfv.N, self.bfv.L
        self.gpu = context(params)
        self.cpu = Oracle(self.bfv)
        self.cpu.set_secret(sampling.secret(np.random.default_rng([params.seed, 0]), self.N))
        self.mirrored = set()
        self.rng = np.random.default_rng([params.seed, 99])

    def sync_keys(self):
        for st in sorted(self.gpu.own_key_steps - self.mirrored):
            a, e = sampling.rotation_key_randomness(np.random.default_rng([self.params.seed, 1, st]), self.bfv,
                                                    self.params.sigma)
            self.cpu.gen_rotkey(st, a, e)
            self.mirrored.add(st)

    def encrypt(self, phys):
        a, e = sampling.encryption_randomness(self.rng, self.bfv)
        return self.gpu.encrypt_physical(phys, a, e), self.cpu.encrypt(phys, a, e)
