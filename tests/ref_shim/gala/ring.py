"""`gala.ring` -> paper_2105_01827_b200.ring (test shim)."""
import sys

from paper_2105_01827_b200 import ring as _m

sys.modules[__name__] = _m
