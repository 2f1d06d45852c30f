"""`gala.matvec` -> paper_2105_01827_b200.matvec (test shim)."""
import sys

from paper_2105_01827_b200 import matvec as _m

sys.modules[__name__] = _m
