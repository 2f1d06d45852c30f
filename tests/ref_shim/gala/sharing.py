"""`gala.sharing` -> paper_2105_01827_b200.sharing (test shim)."""
import sys

from paper_2105_01827_b200 import sharing as _m

sys.modules[__name__] = _m
