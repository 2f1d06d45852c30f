"""`gala.errors` -> paper_2105_01827_b200.errors (test shim)."""
import sys

from paper_2105_01827_b200 import errors as _m

sys.modules[__name__] = _m
