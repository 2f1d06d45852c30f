"""Kernel breakdown of the config-2 FC layer (no correctness gate; for A/B experiments via env flags)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_01827_b200.backend import HEParams  # noqa: E402
from paper_2105_01827_b200.matvec import GalaFC  # noqa: E402

B = int(os.environ.get("B", "32"))
P = 1032193
rng = np.random.default_rng(0)
w = rng.integers(-128, 128, (1024, 4096)) % P
layer = GalaFC(w, HEParams(n=4096, p=P, rns_limbs=3, seed=7), tensor_cores=os.environ.get("TC", "1") == "1")
ctx = layer.ctx
cts = torch.stack([layer.encrypt_input(rng.integers(0, P, 4096))[0] for _ in range(B)])
d_r = ctx.to_device_u32(rng.integers(0, P, (B, ctx.N)).astype(np.uint32))
pts = layer.blocks[0][1]
for _ in range(3):
    layer.run_batch(cts, pts, d_r)
torch.cuda.synchronize()
ctx.profile(True)
for _ in range(5):
    layer.run_batch(cts, pts, d_r)
torch.cuda.synchronize()
prof = ctx.profile_read()
ctx.profile(False)
print(json.dumps({k: round(v["ms"] / 5, 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}))
