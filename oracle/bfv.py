"""ctypes wrapper for the CPU BFV oracle (oracle/bfv_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never
imports this module.

All arrays are canonical words: ciphertexts ``uint64[2][L][N]`` in the
coefficient domain, slot vectors ``uint32[N]`` (row 0 = slots [0, N/2),
row 1 = slots [N/2, N)).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

u64p = ctypes.POINTER(ctypes.c_uint64)
u32p = ctypes.POINTER(ctypes.c_uint32)
i64p = ctypes.POINTER(ctypes.c_int64)
i8p = ctypes.POINTER(ctypes.c_int8)
ip = ctypes.POINTER(ctypes.c_int)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.o_create.restype = ctypes.c_void_p
        L.o_create.argtypes = [ctypes.c_int, ctypes.c_int, u64p, u64p, ctypes.c_uint64, ctypes.c_uint64]
        L.o_destroy.argtypes = [ctypes.c_void_p]
        L.o_set_secret.argtypes = [ctypes.c_void_p, i8p]
        L.o_gen_rotkey.argtypes = [ctypes.c_void_p, ctypes.c_int, u64p, i64p]
        L.o_encode_p.argtypes = [ctypes.c_void_p, u32p, u64p]
        L.o_decode_p.argtypes = [ctypes.c_void_p, u64p, u32p]
        L.o_encode.argtypes = [ctypes.c_void_p, u32p, u64p]
        L.o_encrypt.argtypes = [ctypes.c_void_p, u32p, u64p, i64p, u64p]
        L.o_decrypt.argtypes = [ctypes.c_void_p, u64p, u32p]
        L.o_add.argtypes = [ctypes.c_void_p, u64p, u64p, u64p]
        L.o_sub_plain.argtypes = [ctypes.c_void_p, u64p, u32p, u64p]
        L.o_scmult.argtypes = [ctypes.c_void_p, u64p, u32p, u64p]
        L.o_rotate_hoisted.argtypes = [ctypes.c_void_p, u64p, ip, ctypes.c_int, u64p]
        L.o_mv_gala.argtypes = [ctypes.c_void_p, u64p, u32p, ctypes.c_int, ctypes.c_int, u32p, u64p, u64p]
        L.o_mv_gala2.argtypes = [ctypes.c_void_p, u64p, u32p, ctypes.c_int, ctypes.c_int, u32p, u64p, u64p]
        L.o_conv_kg.argtypes = [ctypes.c_void_p, u64p, ctypes.c_int, u32p, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, ip, ctypes.c_int, u64p]
        L.o_conv_kg2.argtypes = [ctypes.c_void_p, u64p, ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, u64p]
        L.o_ntt.argtypes = [ctypes.c_void_p, ctypes.c_int, u64p, ctypes.c_int]
        L.o_bsgs_baby.argtypes = [ctypes.c_int]
        L.o_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class OracleError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise OracleError(f"oracle call failed with status {rc}")


class Oracle:
    """One BFV context on the CPU; mirrors the GPU library entry points."""

    def __init__(self, bfv):
        self.bfv = bfv
        self.N, self.L = bfv.N, bfv.L
        primes = np.array(bfv.all_primes, dtype=np.uint64)
        psis = np.array(bfv.psis, dtype=np.uint64)
        self._h = lib().o_create(bfv.N, bfv.L, _p(primes, u64p), _p(psis, u64p), bfv.p, bfv.psi_p)
        if not self._h:
            raise OracleError("o_create failed")

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.o_destroy(h)

    @property
    def ct_shape(self):
        return (2, self.L, self.N)

    def set_secret(self, s):
        s = _c(s, np.int8)
        _check(lib().o_set_secret(self._h, _p(s, i8p)))

    def gen_rotkey(self, step, a, e):
        a, e = _c(a, np.uint64), _c(e, np.int64)
        assert a.shape == (self.L, self.L + 1, self.N) and e.shape == (self.L, self.N)
        _check(lib().o_gen_rotkey(self._h, int(step), _p(a, u64p), _p(e, i64p)))

    def encode_p(self, slots):
        s = _c(slots, np.uint32)
        m = np.zeros(self.N, np.uint64)
        lib().o_encode_p(self._h, _p(s, u32p), _p(m, u64p))
        return m

    def decode_p(self, m):
        m = _c(m, np.uint64)
        s = np.zeros(self.N, np.uint32)
        lib().o_decode_p(self._h, _p(m, u64p), _p(s, u32p))
        return s

    def encode(self, slots):
        s = _c(slots, np.uint32)
        pt = np.zeros((self.L, self.N), np.uint64)
        lib().o_encode(self._h, _p(s, u32p), _p(pt, u64p))
        return pt

    def encrypt(self, slots, a, e):
        s, a, e = _c(slots, np.uint32), _c(a, np.uint64), _c(e, np.int64)
        ct = np.zeros(self.ct_shape, np.uint64)
        lib().o_encrypt(self._h, _p(s, u32p), _p(a, u64p), _p(e, i64p), _p(ct, u64p))
        return ct

    def decrypt(self, ct):
        ct = _c(ct, np.uint64)
        s = np.zeros(self.N, np.uint32)
        lib().o_decrypt(self._h, _p(ct, u64p), _p(s, u32p))
        return s

    def add(self, a, b):
        a, b = _c(a, np.uint64), _c(b, np.uint64)
        out = np.zeros(self.ct_shape, np.uint64)
        lib().o_add(self._h, _p(a, u64p), _p(b, u64p), _p(out, u64p))
        return out

    def sub_plain(self, ct, r):
        ct, r = _c(ct, np.uint64), _c(r, np.uint32)
        out = np.zeros(self.ct_shape, np.uint64)
        lib().o_sub_plain(self._h, _p(ct, u64p), _p(r, u32p), _p(out, u64p))
        return out

    def scmult(self, ct, slots):
        ct, s = _c(ct, np.uint64), _c(slots, np.uint32)
        out = np.zeros(self.ct_shape, np.uint64)
        lib().o_scmult(self._h, _p(ct, u64p), _p(s, u32p), _p(out, u64p))
        return out

    def rotate_hoisted(self, ct, steps):
        ct = _c(ct, np.uint64)
        st = np.array(list(steps), dtype=np.intc)
        outs = np.zeros((len(st),) + self.ct_shape, np.uint64)
        _check(lib().o_rotate_hoisted(self._h, _p(ct, u64p), _p(st, ip), len(st), _p(outs, u64p)))
        return outs

    def rotate(self, ct, step):
        return self.rotate_hoisted(ct, [step])[0]

    def mv_gala(self, ct, pts, r=None, baby=0, schedule=1):
        """schedule 1: per-term decomposition; schedule 2: digits hoisted across the plaintext product."""
        ct, pts = _c(ct, np.uint64), _c(pts, np.uint32)
        T = pts.shape[0]
        out = np.zeros(self.ct_shape, np.uint64)
        masked = np.zeros(self.ct_shape, np.uint64)
        rp = None
        if r is not None:
            r = _c(r, np.uint32)
            rp = _p(r, u32p)
        fn = lib().o_mv_gala2 if schedule == 2 else lib().o_mv_gala
        _check(fn(self._h, _p(ct, u64p), _p(pts, u32p), T, baby, rp, _p(out, u64p), _p(masked, u64p)))
        return out, (masked if r is not None else None)

    def conv_kg(self, cts, pts, tap_steps, band_step):
        cts, pts = _c(cts, np.uint64), _c(pts, np.uint32)
        n_obp, n_ib, c_n, k = pts.shape[:4]
        assert cts.shape[0] == n_ib
        st = np.array(list(tap_steps), dtype=np.intc)
        outs = np.zeros((n_obp,) + self.ct_shape, np.uint64)
        _check(lib().o_conv_kg(self._h, _p(cts, u64p), n_ib, _p(pts, u32p), n_obp, c_n, k,
                               _p(st, ip), int(band_step), _p(outs, u64p)))
        return outs

    def conv_kg2(self, cts, kern_centred, u_w, u_h, pair=2, band_only=False):
        """Schedule 2 (factored plaintexts, integer first-Add); kern_centred int [c_o][c_i][k_h][k_w].
        band_only: masks without the tap-validity factor (frame-embedded inputs)."""
        cts = _c(cts, np.uint64)
        kern = _c(kern_centred, np.int32)
        c_o, c_i, k_h, k_w = kern.shape
        n = self.N // 2
        c_n = n // (u_w * u_h)
        n_obp = (c_o // c_n + pair - 1) // pair
        outs = np.zeros((n_obp,) + self.ct_shape, np.uint64)
        _check(lib().o_conv_kg2(self._h, _p(cts, u64p), cts.shape[0], kern.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                c_o, c_i, k_h, k_w, u_w, u_h, pair, int(bool(band_only)), _p(outs, u64p)))
        return outs

    def ntt(self, a, idx, inverse=False):
        a = _c(a, np.uint64).copy()
        lib().o_ntt(self._h, int(idx), _p(a, u64p), int(inverse))
        return a


def bsgs_baby(T: int) -> int:
    return lib().o_bsgs_baby(int(T))


def num_threads() -> int:
    return lib().o_num_threads()
