"""Probe of the streamed e2e path: host enqueue time of one device step, streamed call with and
without the copies (GALA_STREAM_NOCOPY), plain H2D / D2H copy rates."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2105_01827_b200 import _lib  # noqa: E402
from paper_2105_01827_b200.backend import HEParams  # noqa: E402
from paper_2105_01827_b200.matvec import GalaFC  # noqa: E402

params = HEParams(n=bench.SLOTS, p=bench.P, rns_limbs=3, seed=7)
layer = GalaFC(bench.weights(), params)
ctx = layer.ctx
N, L, T, baby, B = ctx.N, ctx.L, layer.T, layer.baby, 32
rng = np.random.default_rng(1)
cts = torch.stack([layer.encrypt_input(rng.integers(0, bench.P, bench.N_IN))[0] for _ in range(B)])
masks = [layer.draw_masks(5 + b) for b in range(B)]
phys_r = np.stack([ctx.physical(m[0][0].slots, m[0][1].slots) for m in masks])
d_r = ctx.to_device_u32(phys_r)
pts = layer.blocks[0][1]
outs, masked = ctx.empty_ct(B), ctx.empty_ct(B)
step = lambda: layer.run_batch(cts, pts, d_r, outs=outs, masked=masked)  # noqa: E731
for _ in range(3):
    step()
torch.cuda.synchronize()
hs = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    hs.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize()
print("host enqueue ms per device step", [round(v, 3) for v in hs])
K = 20
h = ctx._bind()
host_ct = torch.from_numpy(np.broadcast_to(ctx.export_words(cts).view(np.int64)[None], (K, B, 2, L, N)).copy()).pin_memory()
host_r = torch.from_numpy(np.broadcast_to(phys_r.view(np.int32)[None], (K, B, N)).copy()).pin_memory()
host_out = torch.empty((K, B, 2, L, N), dtype=torch.int64).pin_memory()
wc = layer.wcan[0]


def stream(k):
    _lib.check(ctx.lib.gala_mv_gala2_stream_host(h, ctypes.c_void_p(host_ct.data_ptr()), k, B,
                                                 ctypes.c_void_p(pts.data_ptr()), ctypes.c_void_p(wc.data_ptr()), T,
                                                 baby, ctypes.c_void_p(host_r.data_ptr()),
                                                 ctypes.c_void_p(host_out.data_ptr())))


for flag in (None, "both", "in", "out"):
    if flag:
        os.environ["GALA_STREAM_NOCOPY"] = flag
    stream(3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    stream(K)
    dt = (time.perf_counter() - t0) * 1e3
    print("stream, skipped copies:", flag, round(dt / K, 3), "ms/step")
os.environ.pop("GALA_STREAM_NOCOPY")
d = torch.empty(host_ct[0].shape, dtype=torch.int64, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(host_ct[0], non_blocking=True)),
                 ("d2h", lambda: host_out[0].copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(name, round(d.numel() * 8 / dt / 1e9, 1), "GB/s")
