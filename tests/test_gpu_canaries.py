"""Out-of-bounds write checks for the warp-specialised tcgen05 / mbarrier kernels.

compute-sanitizer is closed on this GPU pool (profiles/r2_sanitizer.md), so this is the substitute
for its memcheck of the kernels' output writes: every C-ABI entry point that runs k_gala_tc,
k_kg_tc or k_kg1_tc writes into a buffer flanked by 1 MiB guard regions of a fixed pattern, at
ragged sizes (partial 32-input tiles, odd block counts); the guards must be untouched and the words
must equal the CUDA-core path's.  (Reads past the operands would change the words, which the parity
tests pin.)"""
import ctypes

import numpy as np
import pytest

from twins import P, Twin

pytestmark = pytest.mark.gpu

GUARD = 1 << 17          # words (1 MiB) on each side
PATTERN = -0x5A5A5A5A5A5A5A5B


def _guarded(torch, shape, device):
    n = int(np.prod(shape))
    buf = torch.full((2 * GUARD + n,), PATTERN, dtype=torch.int64, device=device)
    return buf, buf[GUARD:GUARD + n].view(shape)


def _guards_intact(buf, n):
    b = buf.cpu().numpy()
    return bool((b[:GUARD] == PATTERN).all() and (b[GUARD + n:] == PATTERN).all())


@pytest.mark.parametrize("B", [17, 31])
def test_fc_tensor_core_writes_stay_in_bounds(B):
    import torch

    tw = Twin(256, 3, seed=9)
    g = tw.gpu
    g.set_fc_tc_min_terms(1)          # the key-folded tile at this small T (production: T >= 128)
    T = 16
    baby, steps = g.bsgs_steps(T)
    tw.keys_for(steps)
    pts2 = g.encode_gala_weights(tw.slots(T), baby)
    wcan = g.fc_tc_weights(pts2, T, baby)
    cts = torch.stack([tw.encrypt(tw.slots())[0] for _ in range(B)])
    d_r = g.to_device_u32(tw.slots(B))
    shape = (B, 2, g.L, g.N)
    ob, outs = _guarded(torch, shape, g.device)
    mb, masked = _guarded(torch, shape, g.device)
    g.call("gala_mv_gala2_batch_tc", ctypes.c_void_p(cts.data_ptr()), B, ctypes.c_void_p(pts2.data_ptr()),
           ctypes.c_void_p(wcan.data_ptr()), T, baby, ctypes.c_void_p(d_r.data_ptr()),
           ctypes.c_void_p(outs.data_ptr()), ctypes.c_void_p(masked.data_ptr()))
    n = int(np.prod(shape))
    assert _guards_intact(ob, n) and _guards_intact(mb, n)
    _, ref = g.mv_gala2_batch(cts, pts2, T, d_r, baby)          # CUDA-core baby-step sums
    assert np.array_equal(g.export_words(masked), g.export_words(ref))


@pytest.mark.parametrize("post,nimg", [(True, 1), (True, 3), (False, 1)])
def test_conv_tensor_core_writes_stay_in_bounds(post, nimg):
    import torch

    from paper_2105_01827_b200.conv import ConvTask, kg2_coefficients, kg2_post_coefficients

    tw = Twin(256, 3, seed=10)
    g = tw.gpu
    u, c_n = 8, 4
    c_i, c_o = 2 * c_n, 3 * c_n                     # 3 output blocks: an odd count of row pairs
    kern = tw.rng.integers(-128, 128, (c_o, c_i, 3, 3))
    task = ConvTask(u, u, c_i, 3, 3, c_o, kern, tw.params)
    taps = [rot for _, _, rot in task.offsets()]
    tw.keys_for(taps + [d * u * u for d in range(1, c_n)])
    imgs = [torch.stack([tw.encrypt(np.concatenate([b, b]).astype(np.uint32))[0]
                         for b in tw.rng.integers(0, P, (c_i // c_n, c_n * u * u))]) for _ in range(nimg)]
    A, rowsum, K = kg2_coefficients(task, c_n, 2)
    if post:
        A, rowsum = kg2_post_coefficients(A, K, 2 * c_n)
    masks = g.kg2_encode_masks(3, 3, u, u, 2, band_only=post)
    dev = g.device
    coef, rs = torch.from_numpy(A).to(dev), torch.from_numpy(rowsum).to(dev)
    Mr = coef.shape[0] // (2 * c_n) if post else coef.shape[0]
    st = (ctypes.c_int * 9)(*taps)
    if nimg == 1:
        shape = (Mr // c_n, 2, g.L, g.N)
        buf, outs = _guarded(torch, shape, dev)
        g.call("gala_conv_kg2_post" if post else "gala_conv_kg2", ctypes.c_void_p(imgs[0].data_ptr()), c_i // c_n,
               ctypes.c_void_p(masks.data_ptr()), 9, 2 * c_n, ctypes.c_void_p(coef.data_ptr()),
               ctypes.c_void_p(rs.data_ptr()), Mr, coef.shape[1], st, u * u, c_n, ctypes.c_void_p(outs.data_ptr()))
        ref = g.conv_kg2(imgs[0], masks, coef, rs, 9, 2 * c_n, taps, u * u, c_n, post=post)
    else:
        batch = torch.stack(imgs)
        shape = (nimg, Mr // c_n, 2, g.L, g.N)
        buf, outs = _guarded(torch, shape, dev)
        g.call("gala_conv_kg2_post_batch", ctypes.c_void_p(batch.data_ptr()), nimg, c_i // c_n,
               ctypes.c_void_p(masks.data_ptr()), 9, 2 * c_n, ctypes.c_void_p(coef.data_ptr()),
               ctypes.c_void_p(rs.data_ptr()), Mr, coef.shape[1], st, u * u, c_n, ctypes.c_void_p(outs.data_ptr()))
        ref = torch.stack([g.conv_kg2(im, masks, coef, rs, 9, 2 * c_n, taps, u * u, c_n, post=True) for im in imgs])
    assert _guards_intact(buf, int(np.prod(shape)))
    assert np.array_equal(g.export_words(outs), g.export_words(ref))


def test_conv_schedule1_tensor_core_writes_stay_in_bounds():
    import torch

    tw = Twin(256, 3, seed=11)
    g = tw.gpu
    n = tw.bfv.n
    band, c_n, k, n_ib, n_obp = n // 4, 4, 3, 3, 3
    tap_steps = [0, 1, n - 1]
    tw.keys_for(tap_steps + [d * band for d in range(1, c_n)])
    g_in = torch.stack([tw.encrypt(tw.slots())[0] for _ in range(n_ib)])
    spts = tw.slots(n_obp * n_ib * c_n * k).reshape(n_obp, n_ib, c_n, k, tw.N)
    d_pts = g.encode_plain(spts.reshape(-1, tw.N)).view(n_obp, n_ib, c_n, k, tw.L, tw.N)
    ptcan = g.kg1_tc_weights(d_pts, n_obp, n_ib, c_n, k)
    assert ptcan is not None
    shape = (n_obp, 2, g.L, g.N)
    buf, outs = _guarded(torch, shape, g.device)
    st = (ctypes.c_int * k)(*tap_steps)
    g.call("gala_conv_kg_tc", ctypes.c_void_p(g_in.data_ptr()), n_ib, ctypes.c_void_p(ptcan.data_ptr()), n_obp, c_n, k,
           st, band, ctypes.c_void_p(outs.data_ptr()))
    assert _guards_intact(buf, int(np.prod(shape)))
    assert np.array_equal(g.export_words(outs), g.export_words(g.conv_kg(g_in, d_pts, tap_steps, band)))
