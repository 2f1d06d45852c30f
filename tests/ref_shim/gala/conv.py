"""`gala.conv` -> paper_2105_01827_b200.conv (test shim)."""
import sys

from paper_2105_01827_b200 import conv as _m

sys.modules[__name__] = _m
