"""`gala` import shim (TEST INFRASTRUCTURE): maps the reference package's module paths
(pkg/src/gala/__init__.py:78-97) onto the GPU drop-in so the reference's own
test files run unmodified against it (tools/ref_suite.sh).  Only `gala.oracle` points at the
CPU plaintext oracle (oracle/plain.py), which the reference tests use as their checker."""
from paper_2105_01827_b200 import *  # noqa: F401,F403
from paper_2105_01827_b200 import __all__, __version__  # noqa: F401
