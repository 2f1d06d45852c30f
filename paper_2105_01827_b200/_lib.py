"""ctypes binding of the CUDA library (include/gala_b200.h).

The shared object is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2105_01827_b200.build``) into ``paper_2105_01827_b200/_lib/``.
There is no CPU fallback: if the library or a GPU is missing, every backend
call raises :class:`GalaError`.
"""
from __future__ import annotations

import ctypes
import os

from .errors import DimensionError, GalaError, ParameterError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GALA_LIB_PATH") or os.path.join(_HERE, "_lib", "libgala_b200.so")   # override: experiments

GALA_OK = 0
GALA_ERR_PARAM = -1
GALA_ERR_DIM = -2
GALA_ERR_NOKEY = -3
GALA_ERR_CUDA = -4
GALA_ERR_STATE = -5

vp = ctypes.c_void_p
i32 = ctypes.c_int
u64 = ctypes.c_uint64
szt = ctypes.c_size_t

# (name, restype, argtypes) -- every symbol declared in include/gala_b200.h
SIGNATURES = [
    ("gala_last_error", ctypes.c_char_p, []),
    ("gala_version", i32, []),
    ("gala_ctx_create", i32, [ctypes.POINTER(vp), i32, i32, vp, vp, u64, u64, i32]),
    ("gala_ctx_destroy", None, [vp]),
    ("gala_set_stream", i32, [vp, vp]),
    ("gala_sync", i32, [vp]),
    ("gala_set_secret", i32, [vp, vp]),
    ("gala_gen_rotation_key", i32, [vp, i32, vp, vp]),
    ("gala_has_rotation_key", i32, [vp, i32]),
    ("gala_key_bytes", szt, [vp]),
    ("gala_encrypt", i32, [vp, vp, vp, vp, vp]),
    ("gala_decrypt", i32, [vp, vp, vp]),
    ("gala_decrypt_noise", i32, [vp, vp, vp, vp]),
    ("gala_encode_plain", i32, [vp, vp, i32, vp]),
    ("gala_add", i32, [vp, vp, vp, vp]),
    ("gala_scmult", i32, [vp, vp, vp, vp]),
    ("gala_sub_plain", i32, [vp, vp, vp, vp]),
    ("gala_rotate", i32, [vp, vp, i32, vp]),
    ("gala_decompose", i32, [vp, vp, vp]),
    ("gala_digits_words", szt, [vp]),
    ("gala_rotate_hoisted", i32, [vp, vp, vp, i32, vp]),
    ("gala_mv_gala", i32, [vp, vp, vp, i32, i32, vp, vp, vp]),
    ("gala_bsgs_baby", i32, [i32]),
    ("gala_mv_gala_batch", i32, [vp, vp, i32, vp, i32, i32, vp, vp, vp]),
    ("gala_encode_gala_weights", i32, [vp, vp, i32, i32, vp]),
    ("gala_mv_gala2_batch", i32, [vp, vp, i32, vp, i32, i32, vp, vp, vp]),
    ("gala_mv_gala2_partial", i32, [vp, vp, i32, vp, vp, i32, i32, i32, i32, vp, vp]),
    ("gala_mv_gala2_finish", i32, [vp, vp, vp, i32, vp, vp, vp]),
    ("gala_mv_gala2_batch_host", i32, [vp, vp, i32, vp, i32, i32, vp, vp]),
    ("gala_mv_gala_host", i32, [vp, vp, vp, i32, i32, vp, vp]),
    ("gala_mv_gala_batch_host", i32, [vp, vp, i32, vp, i32, i32, vp, vp]),
    ("gala_conv_kg", i32, [vp, vp, i32, vp, i32, i32, i32, vp, i32, vp]),
    ("gala_kg_encode_weights", i32, [vp, vp, i32, i32, i32, i32, i32, i32, i32, vp]),
    ("gala_rotate_batch", i32, [vp, vp, i32, vp, i32, vp]),
    ("gala_fc_tc_weight_bytes", ctypes.c_size_t, [vp]),
    ("gala_fc_tc_weights", i32, [vp, vp, i32, i32, vp]),
    ("gala_mv_gala2_batch_tc", i32, [vp, vp, i32, vp, vp, i32, i32, vp, vp, vp]),
    ("gala_mv_gala2_batch_tc_host", i32, [vp, vp, i32, vp, vp, i32, i32, vp, vp]),
    ("gala_mv_gala2_stream_host", i32, [vp, vp, i32, i32, vp, vp, i32, i32, vp, vp]),
    ("gala_kg1_tc_bytes", ctypes.c_size_t, [vp, i32, i32, i32, i32]),
    ("gala_kg1_tc_weights", i32, [vp, vp, i32, i32, i32, i32, vp]),
    ("gala_conv_kg_tc", i32, [vp, vp, i32, vp, i32, i32, i32, vp, i32, vp]),
    ("gala_conv_kg_batch", i32, [vp, vp, i32, i32, vp, i32, i32, i32, vp, i32, vp]),
    ("gala_kg2_encode_masks", i32, [vp, i32, i32, i32, i32, i32, i32, vp]),
    ("gala_conv_kg2", i32, [vp, vp, i32, vp, i32, i32, vp, vp, i32, i32, vp, i32, i32, vp]),
    ("gala_conv_kg2_post", i32, [vp, vp, i32, vp, i32, i32, vp, vp, i32, i32, vp, i32, i32, vp]),
    ("gala_conv_kg2_post_batch", i32, [vp, vp, i32, i32, vp, i32, i32, vp, vp, i32, i32, vp, i32, i32, vp]),
    ("gala_ct_export", i32, [vp, vp, vp, i32]),
    ("gala_ct_import", i32, [vp, vp, vp, i32]),
    ("gala_pt_export", i32, [vp, vp, vp, i32]),
    ("gala_set_fc_tc_min_terms", i32, [vp, i32]),
    ("gala_launch_count", ctypes.c_uint64, []),
    ("gala_profile_enable", i32, [vp, i32]),
    ("gala_profile_json", i32, [vp, ctypes.c_char_p, szt]),
    ("gala_bench_modmul", i32, [vp, i32, i32, ctypes.POINTER(ctypes.c_double)]),
]

_lib = None


def load():
    """Load the shared library (raises GalaError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise GalaError(
            f"CUDA library {LIB_PATH} is missing; run __graft_entry__.build() "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == GALA_OK:
        return
    msg = load().gala_last_error().decode(errors="replace")
    if rc in (GALA_ERR_PARAM, GALA_ERR_NOKEY):
        raise ParameterError(msg)
    if rc == GALA_ERR_DIM:
        raise DimensionError(msg)
    raise GalaError(msg)


def launch_count() -> int:
    return int(load().gala_launch_count())
