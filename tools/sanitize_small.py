"""Smoke-sized calls of the warp-specialised tcgen05 / mbarrier kernels for compute-sanitizer
(memcheck, racecheck, synccheck): k_gala_e_can + k_gala_tc (FC schedule 2 on the tensor cores),
k_kg_zy + k_kg_tc (conv schedule 2, post-mask and pre-mask), k_kg1_tc (conv schedule 1 first-Add on
the tensor cores).  Each result is checked word for word against the CUDA-core path so a run under
the sanitizer also exercises correctness.

    compute-sanitizer --tool memcheck --target-processes all python tools/sanitize_small.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from twins import P, Twin  # noqa: E402

from paper_2105_01827_b200.conv import ConvTask, kg2_coefficients, kg2_post_coefficients  # noqa: E402

tw = Twin(256, 3, seed=5)
g = tw.gpu
# FC schedule 2, tensor-core baby-step sums (T = 16, 16 inputs)
T = 16
baby, steps = g.bsgs_steps(T)
tw.keys_for(steps)
pts = tw.slots(T)
pts2 = g.encode_gala_weights(pts, baby)
wcan = g.fc_tc_weights(pts2, T, baby)
B = 16
cts = torch.stack([tw.encrypt(tw.slots())[0] for _ in range(B)])
r = g.to_device_u32(tw.slots(B))
_, m_tc = g.mv_gala2_batch(cts, pts2, T, r, baby, wcan=wcan)
_, m_cc = g.mv_gala2_batch(cts, pts2, T, r, baby)
assert np.array_equal(g.export_words(m_tc), g.export_words(m_cc)), "k_gala_tc words"
print("k_gala_e_can + k_gala_tc ok")

# conv schedule 2 on k_kg_tc: post-mask and pre-mask
u, c_n = 8, 4
c_i, c_o = 2 * c_n, 3 * c_n
kern = tw.rng.integers(-128, 128, (c_o, c_i, 3, 3))
task = ConvTask(u, u, c_i, 3, 3, c_o, kern, tw.params)
taps = [rot for _, _, rot in task.offsets()]
tw.keys_for(taps + [d * u * u for d in range(1, c_n)])
xs = torch.stack([tw.encrypt(np.concatenate([b, b]).astype(np.uint32))[0]
                  for b in tw.rng.integers(0, P, (c_i // c_n, c_n * u * u))])
dev = g.device
for post in (True, False):
    A, rowsum, K = kg2_coefficients(task, c_n, 2)
    if post:
        A, rowsum = kg2_post_coefficients(A, K, 2 * c_n)
    masks = g.kg2_encode_masks(3, 3, u, u, 2, band_only=post)
    out = g.conv_kg2(xs, masks, torch.from_numpy(A).to(dev), torch.from_numpy(rowsum).to(dev), 9, 2 * c_n, taps,
                     u * u, c_n, post=post)
    torch.cuda.synchronize()
    print("k_kg_zy + k_kg_tc ok (post=%s)" % post, out.shape)

# conv schedule 1 first-Add on the tensor cores vs the CUDA cores
n = tw.bfv.n
band, c_n, k, n_ib, n_obp = n // 4, 4, 3, 2, 2
tap_steps = [0, 1, n - 1]
tw.keys_for(tap_steps + [d * band for d in range(1, c_n)])
g_in = torch.stack([tw.encrypt(tw.slots())[0] for _ in range(n_ib)])
spts = tw.slots(n_obp * n_ib * c_n * k).reshape(n_obp, n_ib, c_n, k, tw.N)
d_pts = g.encode_plain(spts.reshape(-1, tw.N)).view(n_obp, n_ib, c_n, k, tw.L, tw.N)
ptcan = g.kg1_tc_weights(d_pts, n_obp, n_ib, c_n, k)
assert ptcan is not None
a = g.conv_kg_tc(g_in, ptcan, n_obp, n_ib, c_n, k, tap_steps, band)
b = g.conv_kg(g_in, d_pts, tap_steps, band)
assert np.array_equal(g.export_words(a), g.export_words(b)), "k_kg1_tc words"
print("k_kg1_tc ok")
