"""`gala.analytics` -> paper_2105_01827_b200.analytics (test shim)."""
import sys

from paper_2105_01827_b200 import analytics as _m

sys.modules[__name__] = _m
