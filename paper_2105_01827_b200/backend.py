"""GPU RNS-BFV backend behind the reference's op seam.

Drop-in for ``gala.backend`` (pkg/src/gala/backend.py): same names,
signatures, meters, noise bookkeeping and error types, but every ciphertext
is a real RNS-BFV ciphertext living in HBM and every operation runs in the
CUDA library (``include/gala_b200.h``) -- there is no CPU path.

Mapping (option A): the logical slot count
``HEParams.n`` is one hypercube row of a ring of degree N = 2n.  An API-level
ciphertext replicates its logical vector in both rows; the fused layer
entry points (matvec.GalaFC, conv.KernelGroupingConv) put two logical tasks
that share a rotation schedule in the two rows.

Noise: ``Ciphertext.noise`` carries the reference's mock recurrence
(backend.py:1-11) so ``decrypt`` raises NoiseOverflowError exactly where
the reference does; the real BFV noise is far below the budget at every
configuration this package accepts (noise section).
"""
from __future__ import annotations

import ctypes
import json
import os
import math
import threading
from dataclasses import dataclass, fields, replace

import numpy as np

from . import _lib, sampling
from .errors import DimensionError, GalaError, NoiseOverflowError, ParameterError
from .params import derive, is_prime
from .ring import SlotVector, is_power_of_two

DEFAULT_T_PERM = 0.178
DEFAULT_T_SCMULT = 0.005
DEFAULT_T_ADD = 0.0034
DEFAULT_T_DECPERM = 0.6 * DEFAULT_T_PERM
DEFAULT_T_HSTPERM = 0.4 * DEFAULT_T_PERM

# Batching-friendly default plaintext prime (p = 2^14 * 63 + 1): the
# reference's 1048573 is not 1 mod 2N for any N >= 8.
DEFAULT_P = 1032193


@dataclass(frozen=True)
class CostModel:
    """Per-event milliseconds (backend.py:64-77)."""

    t_perm: float = DEFAULT_T_PERM
    t_scmult: float = DEFAULT_T_SCMULT
    t_add: float = DEFAULT_T_ADD
    t_decperm: float = DEFAULT_T_DECPERM
    t_hstperm: float = DEFAULT_T_HSTPERM

    def __post_init__(self):
        for f in fields(self):
            if getattr(self, f.name) < 0:
                raise ParameterError(f"{f.name} must be non-negative")


@dataclass(frozen=True)
class HEParams:
    """Reference parameter set (backend.py:80-114) plus the BFV instance knobs.

    rns_limbs: ciphertext primes (None: 1 for N <= 4096, else 3);
    device: CUDA device of the context; seed: None (default) draws the
    context's secret, rotation keys and encryption randomness from the OS
    CSPRNG (``sampling.SystemRng``); an integer derives them from seeded
    NumPy PCG64 streams instead -- reproducible, so the CPU oracle can be
    handed the same randomness, and therefore INSECURE (word-parity tests and
    benchmarks only).
    """

    n: int = 2048
    p: int = DEFAULT_P
    q_bits: int = 60
    sigma: float = 3.2
    eta0: float = 8.0
    eta_mult: float = 1024.0
    eta_rot: float = 2048.0
    noise_budget: float | None = None
    rns_limbs: int | None = None
    device: int = 0
    seed: int | None = None

    def __post_init__(self):
        if not is_power_of_two(self.n):
            raise ParameterError(f"n must be a power of two, got {self.n}")
        if not is_prime(self.p):
            raise ParameterError(f"p must be prime, got {self.p}")
        if self.p >= 2**31:
            raise ParameterError("p must fit in 31 bits")
        if self.p >= 2**self.q_bits:
            raise ParameterError("p must be smaller than 2^q_bits")
        if not (self.eta_rot > self.eta_mult > self.eta0 > 1.0):
            raise ParameterError("noise terms must satisfy eta_rot > eta_mult > eta0 > 1")
        if self.noise_budget is None:
            object.__setattr__(self, "noise_budget", 2 ** (self.q_bits - 1) / self.p)
        if self.noise_budget <= self.eta0:
            raise ParameterError("noise_budget must exceed the fresh noise eta0")

    def bfv(self):
        try:
            return derive(self.n, self.p, self.rns_limbs)
        except ValueError as e:
            raise ParameterError(str(e)) from None


class CostMeter:
    """Event counts + cost model (backend.py:117-185)."""

    __slots__ = ("dec_perm", "hst_perm", "full_perm", "sc_mult", "add", "cost_model")

    def __init__(self, cost_model: CostModel | None = None):
        self.dec_perm = 0
        self.hst_perm = 0
        self.full_perm = 0
        self.sc_mult = 0
        self.add = 0
        self.cost_model = cost_model or CostModel()

    def merge(self, other: "CostMeter") -> None:
        self.dec_perm += other.dec_perm
        self.hst_perm += other.hst_perm
        self.full_perm += other.full_perm
        self.sc_mult += other.sc_mult
        self.add += other.add

    def copy(self) -> "CostMeter":
        m = CostMeter(self.cost_model)
        m.merge(self)
        return m

    def as_dict(self, view: str = "split") -> dict[str, int]:
        if view == "split":
            return {"perm": self.full_perm, "dec_perm": self.dec_perm, "hst_perm": self.hst_perm,
                    "sc_mult": self.sc_mult, "add": self.add}
        if view == "paired":
            return {"perm": 0, "dec_perm": self.dec_perm + self.full_perm,
                    "hst_perm": self.hst_perm + self.full_perm, "sc_mult": self.sc_mult, "add": self.add}
        raise ParameterError(f"unknown view {view!r}")

    def estimated_ms(self, model: CostModel | None = None) -> float:
        m = model or self.cost_model
        return (self.full_perm * m.t_perm + self.dec_perm * m.t_decperm + self.hst_perm * m.t_hstperm
                + self.sc_mult * m.t_scmult + self.add * m.t_add)

    def __repr__(self) -> str:
        return (f"CostMeter(perm={self.full_perm}, dec={self.dec_perm}, hst={self.hst_perm}, "
                f"scmult={self.sc_mult}, add={self.add})")


# ---------------------------------------------------------------------------
# device context


def _torch():
    import torch

    return torch


def _ptr(t) -> int:
    return int(t.data_ptr())


class Context:
    """One CUDA-library context per (n, p, rns_limbs, device, seed)."""

    _cache: dict = {}
    _lock = threading.Lock()

    @classmethod
    def get(cls, params: HEParams) -> "Context":
        key = (params.n, params.p, params.rns_limbs, params.device, params.seed)
        with cls._lock:
            ctx = cls._cache.get(key)
            if ctx is None:
                ctx = cls(params)
                cls._cache[key] = ctx
            return ctx

    def __init__(self, params: HEParams, secret: np.ndarray | None = None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise GalaError("no CUDA device: the GALA backend runs only on the GPU (no CPU fallback)")
        self.bfv = params.bfv()
        self.params = params
        self.N, self.L, self.n = self.bfv.N, self.bfv.L, self.bfv.n
        self.device = torch.device("cuda", params.device)
        self.lib = _lib.load()
        primes = (ctypes.c_uint64 * (self.L + 1))(*self.bfv.all_primes)
        psis = (ctypes.c_uint64 * (self.L + 1))(*self.bfv.psis)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.gala_ctx_create(ctypes.byref(h), self.N, self.L, primes, psis, self.bfv.p,
                                                self.bfv.psi_p, params.device))
        self._h = h
        self._enc_counter = 0
        self._fc_tc_min_T = 128
        self.seed = params.seed
        self.own_key_steps = set()    # rotation keys drawn from this context's own randomness source
        if secret is None:
            secret = sampling.secret(self._rng(0), self.N)
        self.set_secret(secret)

    def _rng(self, *tags):
        """The randomness source of one secret / key / encryption: the OS CSPRNG, or (seeded
        contexts only; insecure) a PCG64 stream keyed by (seed, *tags)."""
        if self.seed is None:
            return sampling.SystemRng()
        return np.random.default_rng([self.seed, *tags])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib._lib is not None:
            try:
                _lib._lib.gala_ctx_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- plumbing -----------------------------------------------------------
    def _bind(self):
        """Run library work on torch's current stream of this device."""
        torch = _torch()
        s = torch.cuda.current_stream(self.device)
        _lib.check(self.lib.gala_set_stream(self._h, ctypes.c_void_p(s.cuda_stream)))
        return self._h

    def call(self, name: str, *args):
        h = self._bind()
        _lib.check(getattr(self.lib, name)(h, *args))

    def empty_ct(self, count: int | None = None):
        torch = _torch()
        shape = (2, self.L, self.N) if count is None else (count, 2, self.L, self.N)
        return torch.empty(shape, dtype=torch.int64, device=self.device)

    def to_device_u32(self, arr: np.ndarray):
        torch = _torch()
        a = np.ascontiguousarray(arr, dtype=np.uint32).view(np.int32)
        return torch.from_numpy(a).to(self.device)

    def to_device_u64(self, arr: np.ndarray):
        torch = _torch()
        a = np.ascontiguousarray(arr, dtype=np.uint64).view(np.int64)
        return torch.from_numpy(a).to(self.device)

    def to_device_i64(self, arr: np.ndarray):
        torch = _torch()
        return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)).to(self.device)

    @staticmethod
    def to_host_u64(t) -> np.ndarray:
        return t.cpu().numpy().view(np.uint64)

    # -- keys ---------------------------------------------------------------
    def set_secret(self, s: np.ndarray) -> None:
        s = np.ascontiguousarray(s, dtype=np.int8)
        if s.shape != (self.N,):
            raise DimensionError(f"secret must have {self.N} coefficients")
        self.call("gala_set_secret", s.ctypes.data_as(ctypes.c_void_p))

    def norm_step(self, step: int) -> int:
        return step % self.n

    def has_key(self, step: int) -> bool:
        return bool(self.lib.gala_has_rotation_key(self._h, int(step)))

    def gen_rotation_key(self, step: int, a: np.ndarray | None = None, e: np.ndarray | None = None) -> None:
        step = self.norm_step(step)
        if step == 0:
            return
        if a is None:
            a, e = sampling.rotation_key_randomness(self._rng(1, step), self.bfv, self.params.sigma)
            self.own_key_steps.add(step)
        a = np.ascontiguousarray(a, dtype=np.uint64)
        e = np.ascontiguousarray(e, dtype=np.int64)
        self.call("gala_gen_rotation_key", int(step), a.ctypes.data_as(ctypes.c_void_p),
                  e.ctypes.data_as(ctypes.c_void_p))

    def ensure_keys(self, steps) -> None:
        for s in steps:
            s = self.norm_step(int(s))
            if s and not self.has_key(s):
                self.gen_rotation_key(s)

    def key_bytes(self) -> int:
        return int(self.lib.gala_key_bytes(self._h))

    # -- encode / encrypt / decrypt ------------------------------------------
    def physical(self, row0, row1=None) -> np.ndarray:
        """Physical slot vector [N]: row 0 and row 1 (replica if row1 is None)."""
        r0 = np.asarray(row0, dtype=np.int64) % self.bfv.p
        r1 = r0 if row1 is None else np.asarray(row1, dtype=np.int64) % self.bfv.p
        return np.concatenate([r0, r1]).astype(np.uint32)

    def encode_plain(self, phys_slots: np.ndarray):
        """[B][N] physical slot vectors -> device plaintext operands [B][L][N]."""
        torch = _torch()
        phys = np.atleast_2d(phys_slots)
        B = phys.shape[0]
        d_sl = self.to_device_u32(phys)
        pt = torch.empty((B, self.L, self.N), dtype=torch.int64, device=self.device)
        self.call("gala_encode_plain", ctypes.c_void_p(_ptr(d_sl)), B, ctypes.c_void_p(_ptr(pt)))
        return pt

    def next_encryption_randomness(self):
        rng = self._rng(2, self._enc_counter)
        self._enc_counter += 1
        return sampling.encryption_randomness(rng, self.bfv, self.params.sigma)

    def encrypt_physical(self, phys: np.ndarray, a: np.ndarray | None = None, e: np.ndarray | None = None):
        if a is None:
            a, e = self.next_encryption_randomness()
        d_sl = self.to_device_u32(phys)
        d_a = self.to_device_u64(a)
        d_e = self.to_device_i64(e)
        ct = self.empty_ct()
        self.call("gala_encrypt", ctypes.c_void_p(_ptr(d_sl)), ctypes.c_void_p(_ptr(d_a)),
                  ctypes.c_void_p(_ptr(d_e)), ctypes.c_void_p(_ptr(ct)))
        return ct

    # real-noise guard: decryption is exact while |noise| < Delta / 2; from Delta / 4 on decrypt_physical
    # raises (past Delta / 2 the noise wraps and the slots would be silently wrong)
    REAL_NOISE_LIMIT = 0.25

    def decrypt_physical(self, ct, check_noise: bool = True) -> np.ndarray:
        """Physical slots [N]; with check_noise, raises NoiseOverflowError when the measured noise
        reaches REAL_NOISE_LIMIT of Delta (gala_decrypt_noise)."""
        torch = _torch()
        out = torch.empty(self.N, dtype=torch.int32, device=self.device)
        if not check_noise:
            self.call("gala_decrypt", ctypes.c_void_p(_ptr(ct)), ctypes.c_void_p(_ptr(out)))
            return out.cpu().numpy().view(np.uint32).astype(np.int64)
        frac = ctypes.c_double(0.0)
        self.call("gala_decrypt_noise", ctypes.c_void_p(_ptr(ct)), ctypes.c_void_p(_ptr(out)), ctypes.byref(frac))
        self.last_noise_frac = float(frac.value)
        if frac.value >= self.REAL_NOISE_LIMIT:
            raise NoiseOverflowError(f"measured noise {frac.value:.3f} Delta reached the {self.REAL_NOISE_LIMIT} Delta "
                                     "limit (the parameters have no budget left for this circuit; use more primes)")
        return out.cpu().numpy().view(np.uint32).astype(np.int64)

    def export_words(self, ct) -> np.ndarray:
        """Canonical coefficient-domain words of one or more ciphertexts."""
        torch = _torch()
        count = 1 if ct.dim() == 3 else ct.shape[0]
        out = torch.empty_like(ct)
        self.call("gala_ct_export", ctypes.c_void_p(_ptr(ct)), ctypes.c_void_p(_ptr(out)), count)
        return self.to_host_u64(out)

    def import_words(self, words: np.ndarray):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count = 1 if w.ndim == 3 else w.shape[0]
        d = self.to_device_u64(w)
        ct = self.empty_ct() if w.ndim == 3 else self.empty_ct(count)
        self.call("gala_ct_import", ctypes.c_void_p(_ptr(d)), ctypes.c_void_p(_ptr(ct)), count)
        return ct

    def export_plain(self, pt) -> np.ndarray:
        torch = _torch()
        count = 1 if pt.dim() == 2 else pt.shape[0]
        out = torch.empty_like(pt)
        self.call("gala_pt_export", ctypes.c_void_p(_ptr(pt)), ctypes.c_void_p(_ptr(out)), count)
        return self.to_host_u64(out)

    # -- ops on device tensors -----------------------------------------------
    def add(self, a, b):
        out = self.empty_ct()
        self.call("gala_add", ctypes.c_void_p(_ptr(a)), ctypes.c_void_p(_ptr(b)), ctypes.c_void_p(_ptr(out)))
        return out

    def scmult(self, ct, pt):
        out = self.empty_ct()
        self.call("gala_scmult", ctypes.c_void_p(_ptr(ct)), ctypes.c_void_p(_ptr(pt)),
                  ctypes.c_void_p(_ptr(out)))
        return out

    def sub_plain(self, ct, phys_r: np.ndarray):
        d_r = self.to_device_u32(phys_r)
        out = self.empty_ct()
        self.call("gala_sub_plain", ctypes.c_void_p(_ptr(ct)), ctypes.c_void_p(_ptr(d_r)),
                  ctypes.c_void_p(_ptr(out)))
        return out

    def rotate(self, ct, step: int):
        self.ensure_keys([step])
        out = self.empty_ct()
        self.call("gala_rotate", ctypes.c_void_p(_ptr(ct)), int(step), ctypes.c_void_p(_ptr(out)))
        return out

    def decompose(self, ct):
        torch = _torch()
        D = torch.empty(int(self.lib.gala_digits_words(self._h)), dtype=torch.int64, device=self.device)
        self.call("gala_decompose", ctypes.c_void_p(_ptr(ct)), ctypes.c_void_p(_ptr(D)))
        return D

    def rotate_hoisted(self, ct, digits, step: int):
        self.ensure_keys([step])
        out = self.empty_ct()
        self.call("gala_rotate_hoisted", ctypes.c_void_p(_ptr(ct)), ctypes.c_void_p(_ptr(digits)), int(step),
                  ctypes.c_void_p(_ptr(out)))
        return out

    def rotate_batch(self, cts, steps):
        """cts [B][2][L][N] -> [B][S][2][L][N]: every input rotated by every (non-zero) step, hoisted."""
        torch = _torch()
        steps = [int(s) for s in steps]
        self.ensure_keys(steps)
        B, S = cts.shape[0], len(steps)
        outs = torch.empty((B, S) + tuple(cts.shape[1:]), dtype=torch.int64, device=self.device)
        st = (ctypes.c_int * S)(*steps)
        self.call("gala_rotate_batch", ctypes.c_void_p(_ptr(cts)), int(B), st, int(S), ctypes.c_void_p(_ptr(outs)))
        return outs

    def bsgs_steps(self, T: int, baby: int | None = None):
        b = baby or int(self.lib.gala_bsgs_baby(int(T)))
        G = T // b
        return b, sorted({self.norm_step(j) for j in range(1, b)} | {self.norm_step(g * b) for g in range(1, G)} - {0})

    def mv_gala(self, ct, pts, T: int, phys_r=None, baby: int | None = None, out=None, masked=None):
        """Fused GALA product; phys_r: physical mask slots (numpy or device int32 tensor)."""
        b, steps = self.bsgs_steps(T, baby)
        self.ensure_keys(steps)
        out = self.empty_ct() if out is None else out
        if phys_r is not None and masked is None:
            masked = self.empty_ct()
        if phys_r is None:
            d_r = None
        elif isinstance(phys_r, np.ndarray):
            d_r = self.to_device_u32(phys_r)
        else:
            d_r = phys_r
        self.call("gala_mv_gala", ctypes.c_void_p(_ptr(ct)), ctypes.c_void_p(_ptr(pts)), int(T), int(b),
                  ctypes.c_void_p(_ptr(d_r)) if d_r is not None else None, ctypes.c_void_p(_ptr(out)),
                  ctypes.c_void_p(_ptr(masked)) if masked is not None else None)
        return out, masked

    def mv_gala_batch(self, cts, pts, T: int, d_r=None, baby: int | None = None, outs=None, masked=None):
        """Fused GALA product over a batch: cts [B][2][L][N] (device), d_r [B][N] int32 device masks."""
        b, steps = self.bsgs_steps(T, baby)
        self.ensure_keys(steps)
        B = cts.shape[0]
        outs = self.empty_ct(B) if outs is None else outs
        if d_r is not None and masked is None:
            masked = self.empty_ct(B)
        self.call("gala_mv_gala_batch", ctypes.c_void_p(_ptr(cts)), int(B), ctypes.c_void_p(_ptr(pts)), int(T),
                  int(b), ctypes.c_void_p(_ptr(d_r)) if d_r is not None else None, ctypes.c_void_p(_ptr(outs)),
                  ctypes.c_void_p(_ptr(masked)) if masked is not None else None)
        return outs, masked

    # -- GALA schedule 2 (digits hoisted across the plaintext product) -----------
    def gala2_baby(self, T: int) -> int:
        """Baby-step count for schedule 2.  Cost ~ a b (one E_jj key product per baby rotation) +
        c T / b (a ModDown, a decomposition and a giant key switch per group); measured on B200 at
        N = 8192, L = 3: c / a ~ 7, so b = 2^round(log2 sqrt(7 T)) (T = 512 -> 64).  Small trees keep
        the balanced split."""
        if T < 64:
            return int(self.lib.gala_bsgs_baby(int(T)))
        b = 1 << int(round(math.log2(math.sqrt(7 * T))))
        return max(1, min(T, b))

    def gala_schedule(self, T: int) -> int:
        """2 when the hoisted-digit key-switch noise fits the budget, else 1."""
        return 2 if (self.L >= 2 or T <= 64) else 1

    def encode_gala_weights(self, phys_slots: np.ndarray, baby: int):
        """[T][N] physical slots -> [T][L+1][N] schedule-2 plaintexts (all QP primes, pre-permuted)."""
        torch = _torch()
        phys = np.atleast_2d(phys_slots)
        T = phys.shape[0]
        d_sl = self.to_device_u32(phys)
        pts2 = torch.empty((T, self.L + 1, self.N), dtype=torch.int64, device=self.device)
        self.call("gala_encode_gala_weights", ctypes.c_void_p(_ptr(d_sl)), T, int(baby), ctypes.c_void_p(_ptr(pts2)))
        return pts2

    def mv_gala2_batch(self, cts, pts2, T: int, d_r=None, baby: int | None = None, outs=None, masked=None,
                       wcan=None):
        """Schedule 2; with ``wcan`` (``fc_tc_weights``) the baby-step sums run on the tensor cores."""
        b, steps = self.bsgs_steps(T, baby)
        self.ensure_keys(steps)
        B = cts.shape[0]
        outs = self.empty_ct(B) if outs is None else outs
        if d_r is not None and masked is None:
            masked = self.empty_ct(B)
        common = (ctypes.c_void_p(_ptr(cts)), int(B), ctypes.c_void_p(_ptr(pts2)))
        tail = (int(T), int(b), ctypes.c_void_p(_ptr(d_r)) if d_r is not None else None, ctypes.c_void_p(_ptr(outs)),
                ctypes.c_void_p(_ptr(masked)) if masked is not None else None)
        if wcan is not None:
            self.call("gala_mv_gala2_batch_tc", *common, ctypes.c_void_p(_ptr(wcan)), *tail)
        else:
            self.call("gala_mv_gala2_batch", *common, *tail)
        return outs, masked

    def mv_gala2_partial(self, cts, pts2, T: int, baby: int, g_lo: int, g_hi: int, wcan=None):
        """Giant groups [g_lo, g_hi) of a schedule-2 layer: (QP sums before the final ModDown
        [B][2][L+1][N], Q addends [B][2][L][N]) -- one rank's share of a multi-GPU layer."""
        torch = _torch()
        B = cts.shape[0]
        qp = torch.empty((B, 2, self.L + 1, self.N), dtype=torch.int64, device=self.device)
        qa = torch.empty((B, 2, self.L, self.N), dtype=torch.int64, device=self.device)
        self.call("gala_mv_gala2_partial", ctypes.c_void_p(_ptr(cts)), int(B), ctypes.c_void_p(_ptr(pts2)),
                  ctypes.c_void_p(_ptr(wcan)) if wcan is not None else None, int(T), int(baby), int(g_lo), int(g_hi),
                  ctypes.c_void_p(_ptr(qp)), ctypes.c_void_p(_ptr(qa)))
        return qp, qa

    def mv_gala2_finish(self, qp, qa, d_r=None):
        """Sums of every shard's partials (element-wise u64) -> (outs, masked), as gala_mv_gala2_batch."""
        B = qp.shape[0]
        outs = self.empty_ct(B)
        masked = self.empty_ct(B) if d_r is not None else None
        self.call("gala_mv_gala2_finish", ctypes.c_void_p(_ptr(qp)), ctypes.c_void_p(_ptr(qa)), int(B),
                  ctypes.c_void_p(_ptr(d_r)) if d_r is not None else None, ctypes.c_void_p(_ptr(outs)),
                  ctypes.c_void_p(_ptr(masked)) if masked is not None else None)
        return outs, masked

    def fc_tc_supported(self, T: int, baby: int) -> bool:
        ok = T % baby == 0 and T // baby <= 8 and baby <= 64 and self.N % 32 == 0
        if self.fc_key_folded():
            # the key-folded tile pays only for T >= 128 (gala_mv_gala2_batch_tc); smaller trees stay on the CUDA cores
            ok = ok and T >= self._fc_tc_min_T
        return ok

    def set_fc_tc_min_terms(self, min_terms: int) -> None:
        """Smallest tree that runs its baby-step sums on the tensor cores (default 128; words identical)."""
        self.call("gala_set_fc_tc_min_terms", int(min_terms))
        self._fc_tc_min_T = int(min_terms)

    def fc_key_folded(self) -> bool:
        """True when the library runs the tensor-core FC baby steps key-folded (k_gala_kf, the default;
        GALA_FC_KF=0 selects the split k_gala_e_can / k_gala_tc pair)."""
        return os.environ.get("GALA_FC_KF", "1") != "0" and self.L <= 3

    def fc_tc_weights(self, pts2, T: int, baby: int):
        """Byte-convolution expansion of schedule-2 weights for the tensor-core baby-step sums."""
        torch = _torch()
        nbytes = int(self.lib.gala_fc_tc_weight_bytes(self._bind()))
        wcan = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.call("gala_fc_tc_weights", ctypes.c_void_p(_ptr(pts2)), int(T), int(baby), ctypes.c_void_p(_ptr(wcan)))
        return wcan

    def conv_kg(self, cts, pts, tap_steps, band_step: int):
        """cts [n_ib][2][L][N]; pts [n_obp][n_ib][c_n][k][L][N] -> [n_obp][2][L][N]."""
        n_obp, n_ib, c_n, k = pts.shape[:4]
        self.ensure_keys(list(tap_steps) + [d * band_step for d in range(1, c_n)])
        outs = self.empty_ct(n_obp)
        st = (ctypes.c_int * k)(*[int(s) for s in tap_steps])
        self.call("gala_conv_kg", ctypes.c_void_p(_ptr(cts)), int(n_ib), ctypes.c_void_p(_ptr(pts)), int(n_obp),
                  int(c_n), int(k), st, int(band_step), ctypes.c_void_p(_ptr(outs)))
        return outs

    def conv_kg_batch(self, cts_batch, pts, tap_steps, band_step: int):
        """Schedule 1 over B images sharing the weights: [B][n_ib][2][L][N] -> [B][n_obp][2][L][N]."""
        torch = _torch()
        n_obp, n_ib, c_n, k = pts.shape[:4]
        nbatch = cts_batch.shape[0]
        if cts_batch.shape[1] != n_ib:
            raise DimensionError(f"expected {n_ib} input ciphertexts per image, got {cts_batch.shape[1]}")
        self.ensure_keys(list(tap_steps) + [d * band_step for d in range(1, c_n)])
        outs = torch.empty((nbatch, n_obp, 2, self.L, self.N), dtype=torch.int64, device=self.device)
        st = (ctypes.c_int * k)(*[int(s) for s in tap_steps])
        self.call("gala_conv_kg_batch", ctypes.c_void_p(_ptr(cts_batch)), int(nbatch), int(n_ib),
                  ctypes.c_void_p(_ptr(pts)), int(n_obp), int(c_n), int(k), st, int(band_step),
                  ctypes.c_void_p(_ptr(outs)))
        return outs

    def kg1_tc_weights(self, pts, n_obp: int, n_ib: int, c_n: int, k: int):
        """Position-major copy of schedule-1 KG plaintexts for the tensor-core first-Add (None: unsupported)."""
        torch = _torch()
        nbytes = int(self.lib.gala_kg1_tc_bytes(self._bind(), int(n_ib), int(n_obp), int(c_n), int(k)))
        if nbytes == 0:
            return None
        out = torch.empty(nbytes // 8, dtype=torch.int64, device=self.device)
        self.call("gala_kg1_tc_weights", ctypes.c_void_p(_ptr(pts)), int(n_obp), int(n_ib), int(c_n), int(k),
                  ctypes.c_void_p(_ptr(out)))
        return out

    def conv_kg_tc(self, cts, ptcan, n_obp: int, n_ib: int, c_n: int, k: int, tap_steps, band_step: int):
        """Schedule 1 with the first-Add on the tensor cores; same words as conv_kg."""
        self.ensure_keys(list(tap_steps) + [d * band_step for d in range(1, c_n)])
        outs = self.empty_ct(n_obp)
        st = (ctypes.c_int * k)(*[int(s) for s in tap_steps])
        self.call("gala_conv_kg_tc", ctypes.c_void_p(_ptr(cts)), int(n_ib), ctypes.c_void_p(_ptr(ptcan)), int(n_obp),
                  int(c_n), int(k), st, int(band_step), ctypes.c_void_p(_ptr(outs)))
        return outs

    def conv_kg2(self, cts, masks, coef, rowsum, k: int, nb: int, tap_steps, band_step: int, c_n: int,
                 post: bool = False):
        """Schedule 2: cts [n_ib][2][L][N] -> [Mr/c_n][2][L][N].  Pre-mask: masks [k][nb][M][N][2],
        coef int8 [Mr][Kp]; post-mask (band-only masks [nb][M][N][2]): coef int8 [Mr nb][Kp]."""
        n_ib = cts.shape[0]
        rows, Kp = coef.shape
        Mr = rows // nb if post else rows
        self.ensure_keys(list(tap_steps) + [d * band_step for d in range(1, c_n)])
        outs = self.empty_ct(Mr // c_n)
        st = (ctypes.c_int * k)(*[int(s) for s in tap_steps])
        self.call("gala_conv_kg2_post" if post else "gala_conv_kg2", ctypes.c_void_p(_ptr(cts)), int(n_ib),
                  ctypes.c_void_p(_ptr(masks)), int(k), int(nb), ctypes.c_void_p(_ptr(coef)),
                  ctypes.c_void_p(_ptr(rowsum)), int(Mr), int(Kp), st, int(band_step), int(c_n),
                  ctypes.c_void_p(_ptr(outs)))
        return outs

    def conv_kg2_batch(self, cts_batch, masks, coef, rowsum, k: int, nb: int, tap_steps, band_step: int, c_n: int):
        """Post-mask schedule 2 over B images sharing the weights: [B][n_ib][2][L][N] -> [B][Mr/c_n][2][L][N]."""
        torch = _torch()
        nbatch, n_ib = cts_batch.shape[0], cts_batch.shape[1]
        rows, Kp = coef.shape
        Mr = rows // nb
        self.ensure_keys(list(tap_steps) + [d * band_step for d in range(1, c_n)])
        outs = torch.empty((nbatch, Mr // c_n, 2, self.L, self.N), dtype=torch.int64, device=self.device)
        st = (ctypes.c_int * k)(*[int(s) for s in tap_steps])
        self.call("gala_conv_kg2_post_batch", ctypes.c_void_p(_ptr(cts_batch)), int(nbatch), int(n_ib),
                  ctypes.c_void_p(_ptr(masks)), int(k), int(nb), ctypes.c_void_p(_ptr(coef)),
                  ctypes.c_void_p(_ptr(rowsum)), int(Mr), int(Kp), st, int(band_step), int(c_n),
                  ctypes.c_void_p(_ptr(outs)))
        return outs

    def kg2_encode_masks(self, k_h: int, k_w: int, u_w: int, u_h: int, pair: int, band_only: bool = False):
        torch = _torch()
        c_n = self.params.n // (u_w * u_h)
        taps = 1 if band_only else k_h * k_w
        masks = torch.empty((taps, pair * c_n, self.L + 1, self.N, 2), dtype=torch.int64, device=self.device)
        self.call("gala_kg2_encode_masks", int(k_h), int(k_w), int(u_w), int(u_h), int(pair), int(bool(band_only)),
                  ctypes.c_void_p(_ptr(masks)))
        return masks

    def sync(self):
        self.call("gala_sync")

    # -- tracing / probes ------------------------------------------------------
    def profile(self, on: bool) -> None:
        self.call("gala_profile_enable", int(bool(on)))

    def profile_read(self) -> dict:
        buf = ctypes.create_string_buffer(1 << 16)
        self.call("gala_profile_json", buf, len(buf))
        raw = json.loads(buf.value.decode())
        return {k: {"launches": int(v[0]), "ms": float(v[1])} for k, v in raw.items()}

    def bench_modmul(self, blocks: int = 148 * 16, iters: int = 4096) -> float:
        out = ctypes.c_double()
        self.call("gala_bench_modmul", int(blocks), int(iters), ctypes.byref(out))
        return float(out.value)


def context(params: HEParams) -> Context:
    return Context.get(params)


# ---------------------------------------------------------------------------
# ciphertext handle


class Ciphertext:
    """A BFV ciphertext in HBM plus the reference's mock noise level.

    ``row`` selects which hypercube row holds this logical vector;
    ``replicated`` says both rows hold it (every encryption, and every op on
    replicated operands).  Row-paired layer outputs hold a different vector in
    the other row.  The constructor mirrors ``MockCiphertext(payload, noise,
    params)`` (backend.py:188-204): it encrypts ``payload`` and records ``noise``.
    """

    __slots__ = ("data", "noise", "params", "row", "replicated", "__weakref__")

    def __init__(self, payload: SlotVector, noise: float, params: HEParams):
        if len(payload) != params.n:
            raise DimensionError(f"payload length {len(payload)} != slot count {params.n}")
        if payload.modulus != params.p:
            raise DimensionError(f"payload modulus {payload.modulus} != plaintext modulus {params.p}")
        ctx = context(params)
        self.data = ctx.encrypt_physical(ctx.physical(payload.slots))
        self.noise = noise
        self.params = params
        self.row = 0
        self.replicated = True

    @classmethod
    def _wrap(cls, data, noise: float, params: HEParams, row: int = 0, replicated: bool = False) -> "Ciphertext":
        c = object.__new__(cls)
        c.data = data
        c.noise = noise
        c.params = params
        c.row = 0 if replicated else row
        c.replicated = bool(replicated)
        return c

    @property
    def ctx(self) -> Context:
        return context(self.params)

    @property
    def payload(self) -> SlotVector:
        """Decrypted logical slots (debug/test accessor; no noise check)."""
        full = self.ctx.decrypt_physical(self.data, check_noise=False)
        n = self.params.n
        return SlotVector._wrap(full[self.row * n:(self.row + 1) * n].copy(), self.params.p)

    def words(self) -> np.ndarray:
        """Canonical ciphertext words uint64 [2][L][N] (coefficient domain)."""
        return self.ctx.export_words(self.data)

    def __repr__(self) -> str:
        rows = "both" if self.replicated else self.row
        return f"Ciphertext(n={self.params.n}, L={self.ctx.L}, row={rows}, noise={self.noise:g})"


MockCiphertext = Ciphertext  # drop-in name used by reference callers and tests


class RotationGroup:
    """Result of one DecPerm: the source plus its key-switching digits in HBM."""

    __slots__ = ("source", "decomposed", "digits")

    def __init__(self, source: Ciphertext, digits=None):
        self.source = source
        self.decomposed = True
        self.digits = digits


def _check_same(a: Ciphertext, b: Ciphertext) -> tuple[int, bool]:
    """(row, replicated) of a slotwise combination of a and b."""
    if a.params != b.params:
        raise DimensionError("ciphertexts built under different parameter sets")
    if a.replicated and b.replicated:
        return 0, True
    if a.replicated or b.replicated:
        return (b.row if a.replicated else a.row), False
    if a.row != b.row:
        raise DimensionError("ciphertexts hold their vectors in different hypercube rows")
    return a.row, False


def _phys_for(ct: Ciphertext, v: SlotVector) -> np.ndarray:
    ctx = ct.ctx
    return ctx.physical(v.slots)


# ---------------------------------------------------------------------------
# the op seam (backend.py:228-311)


def encrypt(x: SlotVector, params: HEParams) -> Ciphertext:
    if len(x) != params.n:
        raise DimensionError(f"plaintext length {len(x)} != slot count {params.n}")
    if x.modulus != params.p:
        raise DimensionError(f"plaintext modulus {x.modulus} != {params.p}")
    ctx = context(params)
    return Ciphertext._wrap(ctx.encrypt_physical(ctx.physical(x.slots)), params.eta0, params, replicated=True)


def decrypt(c: Ciphertext) -> SlotVector:
    """backend.py:237-243: raises NoiseOverflowError where the reference's mock noise reaches its
    budget -- and, on real ciphertexts, where the measured noise reaches a quarter of Delta."""
    if c.noise >= c.params.noise_budget:
        raise NoiseOverflowError(f"noise {c.noise:g} reached budget {c.params.noise_budget:g}")
    full = c.ctx.decrypt_physical(c.data, check_noise=True)
    n = c.params.n
    return SlotVector._wrap(full[c.row * n:(c.row + 1) * n].copy(), c.params.p)


def he_add(a: Ciphertext, b: Ciphertext, meter: CostMeter) -> Ciphertext:
    row, rep = _check_same(a, b)
    out = a.ctx.add(a.data, b.data)
    meter.add += 1
    return Ciphertext._wrap(out, a.noise + b.noise, a.params, row, rep)


def he_scmult(a: Ciphertext, s: SlotVector, meter: CostMeter) -> Ciphertext:
    if len(s) != a.params.n or s.modulus != a.params.p:
        raise DimensionError("plaintext operand does not match ciphertext layout")
    ctx = a.ctx
    pt = ctx.encode_plain(_phys_for(a, s))
    out = ctx.scmult(a.data, pt[0])
    meter.sc_mult += 1
    return Ciphertext._wrap(out, a.noise * a.params.eta_mult, a.params, a.row, a.replicated)


def he_perm(a: Ciphertext, k: int, meter: CostMeter) -> Ciphertext:
    k %= a.params.n
    if k == 0:
        return a
    out = a.ctx.rotate(a.data, k)
    meter.full_perm += 1
    return Ciphertext._wrap(out, a.noise + a.params.eta_rot, a.params, a.row, a.replicated)


def he_decperm(a: Ciphertext, meter: CostMeter) -> RotationGroup:
    meter.dec_perm += 1
    return RotationGroup(a, a.ctx.decompose(a.data))


def he_hstperm(g: RotationGroup, k: int, meter: CostMeter) -> Ciphertext:
    src = g.source
    k %= src.params.n
    if k == 0:
        return src
    if g.digits is None:
        g.digits = src.ctx.decompose(src.data)
    out = src.ctx.rotate_hoisted(src.data, g.digits, k)
    meter.hst_perm += 1
    return Ciphertext._wrap(out, src.noise + src.params.eta_rot, src.params, src.row, src.replicated)


def subtract_plain(a: Ciphertext, r: SlotVector, meter: CostMeter) -> Ciphertext:
    if len(r) != a.params.n or r.modulus != a.params.p:
        raise DimensionError("mask vector does not match ciphertext layout")
    out = a.ctx.sub_plain(a.data, _phys_for(a, r))
    meter.add += 1
    return Ciphertext._wrap(out, a.noise + a.params.eta0, a.params, a.row, a.replicated)


_PARAM_KEYS = {"n", "p", "q_bits", "sigma", "eta0", "eta_mult", "eta_rot", "noise_budget", "rns_limbs",
               "device", "seed"}
_COST_KEYS = {"t_perm", "t_scmult", "t_add", "t_decperm", "t_hstperm"}


def load_cost_config(path) -> tuple[HEParams, CostModel]:
    """JSON calibration (backend.py:318-334); unknown keys are rejected."""
    with open(path) as f:
        raw = json.load(f)
    if not isinstance(raw, dict):
        raise ParameterError("cost config must be a JSON object")
    unknown = set(raw) - _PARAM_KEYS - _COST_KEYS
    if unknown:
        raise ParameterError(f"unknown config keys: {sorted(unknown)}")
    params = HEParams(**{k: raw[k] for k in _PARAM_KEYS & set(raw)})
    model = CostModel(**{k: raw[k] for k in _COST_KEYS & set(raw)})
    return params, model


def with_overrides(params: HEParams, n: int | None = None, p: int | None = None, **kw) -> HEParams:
    """Copy of params with n / p (and optional BFV knobs) replaced."""
    upd = dict(kw)
    if n is not None:
        upd["n"] = n
    if p is not None:
        upd["p"] = p
        upd["noise_budget"] = None
    return replace(params, **upd) if upd else params
