"""Timeline of k_gala_kf's CTA 0 (library built with -DKF_TRACE): where the pair's MMA issuer waits.
Usage: GALA_LIB_PATH=probe_libs/lib_trace.so B=256 python tools/kf_trace.py"""
import ctypes
import os
import runpy
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("B", "256")
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "time_fc.py"))
from paper_2105_01827_b200 import _lib  # noqa: E402

lib = ctypes.CDLL(_lib.LIB_PATH)
buf = np.zeros((32, 1024), np.uint64)
print("rc", lib.gala_debug_kf_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong))))
t = buf.astype(np.int64)
NST = int(os.environ.get("NST", "16"))     # stages per position
ST = int(os.environ.get("ST", "6"))        # ring depth
lo, hi = 2 * NST, min(1000, 40 * NST)
gs = np.arange(lo, hi)
period = np.diff(t[9, lo:hi + 1])
print(f"stages {lo}..{hi}: period mean {period.mean():.0f} median {np.median(period):.0f} clk")
print("period percentiles 10/50/90/99:", [int(np.percentile(period, x)) for x in (10, 50, 90, 99)])
big = np.where(period > 4000)[0]
print("stages with period > 4000 clk (index within position, position):", [(int((lo + i) % NST), int((lo + i) // NST)) for i in big[:20]])
print("mean period by stage within position:", [int(period[(gs % NST) == s_].mean()) if np.any((gs % NST) == s_) else 0 for s_ in range(NST)])
iss = t[1, gs] - t[0, gs]
print("issue+commit by stage within position:", [int(iss[(gs % NST) == s_].mean()) for s_ in range(NST)])
fw = t[0, gs] - t[9, gs]
print("full wait by stage within position:", [int(fw[(gs % NST) == s_].mean()) for s_ in range(NST)])
print(f"issuer full wait: mean {np.mean(t[0, gs] - t[9, gs]):.0f} median {np.median(t[0, gs] - t[9, gs]):.0f}")
print(f"issuer issue+commit: mean {np.mean(t[1, gs] - t[0, gs]):.0f}")
pos = np.arange(2, hi // NST - 1)
tw = t[6, pos] - t[1, pos * NST - 1]
print(f"per position tempty wait after the previous position's last commit: mean {tw.mean():.0f} median {np.median(tw):.0f}")
print(f"producer: empty ok -> copies issued mean {np.mean(t[3, gs] - t[2, gs]):.0f}")
g2 = gs[:-ST]
print(f"issuer commit(s) -> producer sees empty for s+ST: median {np.median(t[2, g2 + ST] - t[1, g2]):.0f}")
print(f"producer issued A(s) -> issuer full ok(s): median {np.median(t[0, gs] - t[3, gs]):.0f} mean {np.mean(t[0, gs] - t[3, gs]):.0f}")
print(f"producer issued A(s) -> issuer starts waiting: median {np.median(t[9, gs] - t[3, gs]):.0f}")
if os.environ.get("RANK1"):
    print(f"rank 1: producer issued A(s) -> relay sees full(s): median {np.median(t[4, gs] - t[3, gs]):.0f}")
    print(f"rank 1: producer empty ok -> issued: median {np.median(t[3, gs] - t[2, gs]):.0f}")
    print(f"rank 1: relay period median {np.median(np.diff(t[4, lo:hi + 1])):.0f}")
exp_last = np.max(t[12:16, gs], axis=0)
print(f"expanders' last arrive(s) - producer issued A(s): median {np.median(exp_last - t[3, gs]):.0f}")
print(f"issuer full ok(s) - expanders' last arrive(s): median {np.median(t[0, gs] - exp_last):.0f}")
print(f"expander: wfull ok -> empty ok median {np.median(t[16, gs] - t[20, gs]):.0f}; empty ok -> arrive median {np.median(t[12, gs] - t[16, gs]):.0f}")
print(f"expander: arrive(s-1) -> wfull ok(s) median {np.median(t[20, gs[1:]] - t[12, gs[1:] - 1]):.0f}")
