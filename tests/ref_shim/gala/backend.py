"""`gala.backend` -> paper_2105_01827_b200.backend (test shim)."""
import sys

from paper_2105_01827_b200 import backend as _m

sys.modules[__name__] = _m
