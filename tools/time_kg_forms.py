"""Config 4 (56x56x64 -> 64 in 64x64 frames, N = 8192, L = 3) through every schedule-2 form:
post-mask (production, row-paired), pre-mask row-paired, and the drop-in pre-mask one-block-per-
ciphertext layer.  Prints one JSON line per form: ms per layer (CUDA events, median of 5) and the
per-kernel breakdown (library tracer)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2105_01827_b200.backend import HEParams  # noqa: E402
from paper_2105_01827_b200.conv import ConvTask, KernelGroupingConv, encrypt_inputs  # noqa: E402

P = 1032193
params = HEParams(n=4096, rns_limbs=3, seed=32)
rng = np.random.default_rng(2)
kern = rng.integers(-128, 128, (64, 64, 3, 3)) % P
img = np.zeros((64, 64, 64), dtype=np.int64)
img[:, :56, :56] = rng.integers(0, P, (64, 56, 56))
task = ConvTask(64, 64, 64, 3, 3, 64, kern, params)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for name, kw in (("post_paired", dict(band_only=True)), ("pre_paired", dict(band_only=False)),
                 ("pre_single_dropin", dict(pair_rows=False))):
    layer = KernelGroupingConv(task, **kw)
    ctx = layer.ctx
    x = torch.stack([c.data for c in encrypt_inputs(task, img)])
    layer.forward_device(x)
    ts = []
    for _ in range(5):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        layer.forward_device(x)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ctx.profile(True)
    layer.forward_device(x)
    prof = ctx.profile_read()
    ctx.profile(False)
    print(json.dumps({"form": name, "schedule": layer.schedule, "post": layer.post, "pair": layer.pair,
                      "ms": round(float(np.median(ts)), 4),
                      "breakdown_ms": {k: round(v["ms"], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}}))
    del layer
