"""The C-ABI library loads (no GPU needed) and exports every symbol declared
in include/gala_b200.h; the ctypes binding covers all of them."""
import ctypes
import os
import re

from paper_2105_01827_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gala_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gala_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ("gala_ctx_create", "gala_encrypt", "gala_decrypt", "gala_rotate", "gala_decompose",
                 "gala_rotate_hoisted", "gala_mv_gala", "gala_mv_gala_batch", "gala_conv_kg", "gala_scmult",
                 "gala_add", "gala_sub_plain"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_symbols()) <= bound
    lib = _lib.load()
    assert lib.gala_version() == 1
    assert lib.gala_bsgs_baby(512) == 32 and lib.gala_bsgs_baby(8) == 4 and lib.gala_bsgs_baby(1) == 1


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_path_without_gpu():
    import pytest

    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2105_01827_b200 import HEParams, SlotVector, encrypt
    from paper_2105_01827_b200.errors import GalaError

    with pytest.raises(GalaError):
        encrypt(SlotVector.zeros(2048, HEParams().p), HEParams())
