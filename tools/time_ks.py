"""Kernel breakdown of the raw key-switch probe (bench.py ks_probe): 96 config-2 inputs, each rotated by
8 steps with one decomposition per input (gala_rotate_batch)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_01827_b200.backend import HEParams, context  # noqa: E402

B = int(os.environ.get("B", "96"))
ctx = context(HEParams(n=4096, p=1032193, rns_limbs=3, seed=7))
rng = np.random.default_rng(0)
cts = torch.stack([ctx.encrypt_physical(rng.integers(0, 1032193, ctx.N).astype(np.uint32)) for _ in range(B)])
steps = [1, 2, 3, 5, 8, 13, 21, 34]
for _ in range(3):
    ctx.rotate_batch(cts, steps)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.rotate_batch(cts, steps)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ctx.profile(True)
ctx.rotate_batch(cts, steps)
prof = ctx.profile_read()
ctx.profile(False)
ms = float(np.median(ts))
print(json.dumps({"ms": round(ms, 4), "rotations_per_s": round(B * len(steps) / ms * 1e3, 1),
                  "gmodmul_s": round(B * len(steps) * 1310720 / ms / 1e6, 1),
                  "breakdown_ms": {k: round(v["ms"], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}}))
