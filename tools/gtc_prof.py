"""Role timing of k_gala_tc (library built with GALA_NVCC_EXTRA=-DGTC_PROF): cycles per position."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import runpy  # noqa: E402

runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "time_fc.py"))
from paper_2105_01827_b200 import _lib  # noqa: E402

lib = ctypes.CDLL(_lib.LIB_PATH if hasattr(_lib, "LIB_PATH") else os.path.join(os.path.dirname(_lib.__file__), "_lib", "libgala_b200.so"))
buf = np.zeros((1024, 16), np.uint64)
rc = lib.gala_debug_gtc_prof(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), 1024)
rows = buf[buf[:, 11] > 0]
npos = rows[:, 11].astype(float)
names = ["prod.wait_empty", "mma.wait_tempty", "mma.wait_full", "mma.wait_bfull", "epi.head", "exp.wait_full",
         "exp.wait_bempty", "exp.work", "epi.wait_tfull", "epi.work", "total", "positions", "epi.tld", "epi.iter", "epi.loop"]
print("rc", rc, "ctas", len(rows), "positions/cta", npos.mean())
for i, nm in enumerate(names):
    if nm == "-":
        continue
    v = rows[:, i].astype(float) / (npos if i != 11 else 1)
    print(f"{nm:18s} {v.mean():10.1f} cycles/position")
