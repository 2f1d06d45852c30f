"""`gala.oracle` -> oracle.plain, the CPU plaintext truth (test shim; checker only)."""
import sys

from oracle import plain as _m

sys.modules[__name__] = _m
