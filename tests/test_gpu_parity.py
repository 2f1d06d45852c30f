"""Word-level parity: CUDA library vs the CPU BFV oracle (same randomness)."""
import numpy as np
import pytest

from twins import P, Twin

pytestmark = pytest.mark.gpu

SHAPES = [(4, 1), (32, 1), (32, 3), (256, 2), (2048, 1), (4096, 3)]


@pytest.fixture(scope="module", params=SHAPES, ids=lambda s: f"n{s[0]}L{s[1]}")
def tw(request):
    n, L = request.param
    return Twin(n, L)


def test_encrypt_words_and_decrypt(tw):
    x = tw.slots()
    g, c = tw.encrypt(x)
    assert np.array_equal(tw.gpu.export_words(g), c)
    assert np.array_equal(tw.gpu.decrypt_physical(g), x.astype(np.int64))


def test_encode_plain_words(tw):
    s = tw.slots(3)
    pts = tw.gpu.encode_plain(s)
    got = tw.gpu.export_plain(pts)
    for i in range(3):
        assert np.array_equal(got[i], tw.cpu.encode(s[i]))


def test_add_scmult_subplain_words(tw):
    x, y, r = tw.slots(), tw.slots(), tw.slots()
    g1, c1 = tw.encrypt(x)
    g2, c2 = tw.encrypt(y)
    assert np.array_equal(tw.gpu.export_words(tw.gpu.add(g1, g2)), tw.cpu.add(c1, c2))
    pt = tw.gpu.encode_plain(y)[0]
    gs = tw.gpu.scmult(g1, pt)
    assert np.array_equal(tw.gpu.export_words(gs), tw.cpu.scmult(c1, y))
    assert np.array_equal(tw.gpu.decrypt_physical(gs), (x.astype(np.int64) * y) % P)
    gsub = tw.gpu.sub_plain(g1, r)
    assert np.array_equal(tw.gpu.export_words(gsub), tw.cpu.sub_plain(c1, r))


def test_rotations_words(tw):
    n = tw.bfv.n
    steps = sorted({1, 3 % n, n - 1, n // 2})
    tw.keys_for(steps)
    x = tw.slots()
    g, c = tw.encrypt(x)
    want = tw.cpu.rotate_hoisted(c, steps)
    D = tw.gpu.decompose(g)
    for s, w in zip(steps, want):
        gr = tw.gpu.rotate(g, s)
        assert np.array_equal(tw.gpu.export_words(gr), w), s
        gh = tw.gpu.rotate_hoisted(g, D, s)
        assert np.array_equal(tw.gpu.export_words(gh), w), s
        dec = tw.gpu.decrypt_physical(gr)
        xs = x.astype(np.int64)
        assert np.array_equal(dec, np.concatenate([np.roll(xs[:n], -s), np.roll(xs[n:], -s)]))


@pytest.mark.parametrize("T", [1, 2, 4, 8, 16])
def test_mv_gala_words(tw, T):
    n = tw.bfv.n
    if T > n:
        pytest.skip("T > n")
    b, steps = tw.gpu.bsgs_steps(T)
    tw.keys_for(steps)
    x = tw.slots()
    pts = tw.slots(T)
    r = tw.slots()
    g, c = tw.encrypt(x)
    out, masked = tw.gpu.mv_gala(g, tw.gpu.encode_plain(pts), T, r)
    c_out, c_masked = tw.cpu.mv_gala(c, pts, r, baby=b)
    assert np.array_equal(tw.gpu.export_words(out), c_out)
    assert np.array_equal(tw.gpu.export_words(masked), c_masked)


def test_conv_kg_words(tw):
    """Schedule 1 (CUDA-core and tensor-core first-Add) == oracle o_conv_kg."""
    n = tw.bfv.n
    if n < 16:
        pytest.skip("tiny")
    band = n // 4
    c_n, k, n_ib, n_obp = 4, 3, 2, 2
    tap_steps = [0, 1, n - 1]
    tw.keys_for(tap_steps + [d * band for d in range(1, c_n)])
    xs = [tw.encrypt(tw.slots()) for _ in range(n_ib)]
    pts = tw.slots(n_obp * n_ib * c_n * k).reshape(n_obp, n_ib, c_n, k, tw.N)
    import torch

    g_in = torch.stack([g for g, _ in xs])
    c_in = np.stack([c for _, c in xs])
    d_pts = tw.gpu.encode_plain(pts.reshape(-1, tw.N)).view(n_obp, n_ib, c_n, k, tw.L, tw.N)
    g_out = tw.gpu.conv_kg(g_in, d_pts, tap_steps, band)
    c_out = tw.cpu.conv_kg(c_in, pts, tap_steps, band)
    assert np.array_equal(tw.gpu.export_words(g_out), c_out)
    # the same first-Add on the tensor cores (byte-convolution int8 MMA per position)
    ptcan = tw.gpu.kg1_tc_weights(d_pts, n_obp, n_ib, c_n, k)
    if ptcan is not None:
        t_out = tw.gpu.conv_kg_tc(g_in, ptcan, n_obp, n_ib, c_n, k, tap_steps, band)
        assert np.array_equal(tw.gpu.export_words(t_out), c_out)


@pytest.mark.parametrize("nimg", [1, 3, 6])
def test_conv_kg_batch_words(tw, nimg):
    """Schedule 1 over a batch of images sharing the weights (2 and 4 images per thread, ragged
    tails) == one oracle o_conv_kg per image."""
    n = tw.bfv.n
    if n < 16:
        pytest.skip("tiny")
    band = n // 4
    c_n, k, n_ib, n_obp = 4, 3, 3, 2
    tap_steps = [0, 1, n - 1]
    tw.keys_for(tap_steps + [d * band for d in range(1, c_n)])
    imgs = [[tw.encrypt(tw.slots()) for _ in range(n_ib)] for _ in range(nimg)]
    pts = tw.slots(n_obp * n_ib * c_n * k).reshape(n_obp, n_ib, c_n, k, tw.N)
    import torch

    d_pts = tw.gpu.encode_plain(pts.reshape(-1, tw.N)).view(n_obp, n_ib, c_n, k, tw.L, tw.N)
    g_batch = torch.stack([torch.stack([g for g, _ in im]) for im in imgs])
    outs = tw.gpu.conv_kg_batch(g_batch, d_pts, tap_steps, band)
    for b, im in enumerate(imgs):
        c_out = tw.cpu.conv_kg(np.stack([c for _, c in im]), pts, tap_steps, band)
        assert np.array_equal(tw.gpu.export_words(outs[b]), c_out), f"image {b}"


def test_conv_kg_long_second_perm_words(tw):
    """A second-Perm of 39 rotations: the engine splits the group's key MACs into chunks (k_ks_mac
    slices + k_fold_groups); words == oracle."""
    n = tw.bfv.n
    if n < 256:
        pytest.skip("needs 40 distinct band steps")
    band = n // 64
    c_n, k, n_ib, n_obp = 40, 2, 1, 1
    tap_steps = [0, 1]
    tw.keys_for(tap_steps + [d * band for d in range(1, c_n)])
    xs = [tw.encrypt(tw.slots()) for _ in range(n_ib)]
    pts = tw.slots(n_obp * n_ib * c_n * k).reshape(n_obp, n_ib, c_n, k, tw.N)
    import torch

    g_in = torch.stack([g for g, _ in xs])
    c_in = np.stack([c for _, c in xs])
    d_pts = tw.gpu.encode_plain(pts.reshape(-1, tw.N)).view(n_obp, n_ib, c_n, k, tw.L, tw.N)
    g_out = tw.gpu.conv_kg(g_in, d_pts, tap_steps, band)
    c_out = tw.cpu.conv_kg(c_in, pts, tap_steps, band)
    assert np.array_equal(tw.gpu.export_words(g_out), c_out)


def test_mv_gala_batch_words(tw):
    """Batched entry point == per-input fused calls == oracle."""
    import torch

    n = tw.bfv.n
    T = min(8, n)
    b, steps = tw.gpu.bsgs_steps(T)
    tw.keys_for(steps)
    pts = tw.slots(T)
    d_pts = tw.gpu.encode_plain(pts)
    xs = [tw.encrypt(tw.slots()) for _ in range(3)]
    rs = tw.slots(3)
    outs, masked = tw.gpu.mv_gala_batch(torch.stack([g for g, _ in xs]), d_pts, T, tw.gpu.to_device_u32(rs))
    for i, (g, c) in enumerate(xs):
        c_out, c_masked = tw.cpu.mv_gala(c, pts, rs[i], baby=b)
        assert np.array_equal(tw.gpu.export_words(outs[i]), c_out)
        assert np.array_equal(tw.gpu.export_words(masked[i]), c_masked)


@pytest.mark.parametrize("T", [1, 2, 4, 8, 16])
def test_mv_gala2_words(tw, T):
    """Schedule 2 (digits hoisted across the plaintext product) == oracle o_mv_gala2, batched."""
    import torch

    n = tw.bfv.n
    if T > n:
        pytest.skip("T > n")
    b, steps = tw.gpu.bsgs_steps(T)
    tw.keys_for(steps)
    pts = tw.slots(T)
    pts2 = tw.gpu.encode_gala_weights(pts, b)
    xs = [tw.encrypt(tw.slots()) for _ in range(2)]
    rs = tw.slots(2)
    outs, masked = tw.gpu.mv_gala2_batch(torch.stack([g for g, _ in xs]), pts2, T, tw.gpu.to_device_u32(rs), b)
    for i, (g, c) in enumerate(xs):
        c_out, c_masked = tw.cpu.mv_gala(c, pts, rs[i], baby=b, schedule=2)
        assert np.array_equal(tw.gpu.export_words(outs[i]), c_out)
        assert np.array_equal(tw.gpu.export_words(masked[i]), c_masked)


KG2_GEOM = {32: (4, 4), 256: (8, 8), 2048: (16, 16), 4096: (16, 16)}


@pytest.mark.parametrize("pair", [1, 2])
def test_conv_kg2_words(tw, pair):
    """Schedule 2 (band masks x int8 coefficients on the tensor cores) == oracle o_conv_kg2, word for word,
    and decrypts to the plaintext convolution when the noise budget allows (L >= 2)."""
    import torch

    from oracle.plain import conv2d_mod_p
    from paper_2105_01827_b200.conv import ConvTask, kg2_coefficients

    n = tw.bfv.n
    if n not in KG2_GEOM:
        pytest.skip("no geometry for this ring")
    u_w, u_h = KG2_GEOM[n]
    c_n = n // (u_w * u_h)
    c_i, c_o = 2 * c_n, 3 * c_n
    kern = tw.rng.integers(-128, 128, (c_o, c_i, 3, 3))
    task = ConvTask(u_w, u_h, c_i, 3, 3, c_o, kern, tw.params)
    taps = [rot for _, _, rot in task.offsets()]
    tw.keys_for(taps + [d * u_w * u_h for d in range(1, c_n)])
    x = tw.rng.integers(0, P, (c_i, u_h, u_w))
    blocks = x.reshape(c_i // c_n, c_n * u_w * u_h)
    xs = [tw.encrypt(np.concatenate([b, b]).astype(np.uint32)) for b in blocks]
    A, rowsum, _ = kg2_coefficients(task, c_n, pair)
    masks = tw.gpu.kg2_encode_masks(3, 3, u_w, u_h, pair)
    g_out = tw.gpu.conv_kg2(torch.stack([g for g, _ in xs]), masks, torch.from_numpy(A).to(tw.gpu.device),
                            torch.from_numpy(rowsum).to(tw.gpu.device), 9, pair * c_n, taps, u_w * u_h, c_n)
    c_out = tw.cpu.conv_kg2(np.stack([c for _, c in xs]), kern, u_w, u_h, pair)
    assert np.array_equal(tw.gpu.export_words(g_out), c_out)
    if tw.L >= 2:
        want = conv2d_mod_p(x, kern, P).reshape(c_o // c_n, c_n * u_w * u_h)
        for ob in range(c_o // c_n):
            got = tw.gpu.decrypt_physical(g_out[ob // pair]).reshape(2, -1)[ob % pair if pair == 2 else 0]
            assert np.array_equal(got, want[ob])


def test_conv_kg2_post_words(tw):
    """Post-mask form (band-only masks applied after the GEMM) == oracle o_conv_kg2(band_only=1), word
    for word; on a zero-margin frame it decrypts to the plaintext convolution inside the image."""
    import torch

    from oracle.plain import conv2d_mod_p
    from paper_2105_01827_b200.conv import ConvTask, kg2_coefficients, kg2_post_coefficients

    n = tw.bfv.n
    if n not in KG2_GEOM:
        pytest.skip("no geometry for this ring")
    u_w, u_h = KG2_GEOM[n]
    c_n = n // (u_w * u_h)
    c_i, c_o, pair = 2 * c_n, 3 * c_n, 2
    kern = tw.rng.integers(-128, 128, (c_o, c_i, 3, 3))
    task = ConvTask(u_w, u_h, c_i, 3, 3, c_o, kern, tw.params)
    taps = [rot for _, _, rot in task.offsets()]
    tw.keys_for(taps + [d * u_w * u_h for d in range(1, c_n)])
    x = np.zeros((c_i, u_h, u_w), dtype=np.int64)
    x[:, :u_h - 1, :u_w - 1] = tw.rng.integers(0, P, (c_i, u_h - 1, u_w - 1))   # zero margin of 1
    blocks = x.reshape(c_i // c_n, c_n * u_w * u_h)
    xs = [tw.encrypt(np.concatenate([b, b]).astype(np.uint32)) for b in blocks]
    A, _, K = kg2_coefficients(task, c_n, pair)
    B, rowsum = kg2_post_coefficients(A, K, pair * c_n)
    masks = tw.gpu.kg2_encode_masks(3, 3, u_w, u_h, pair, band_only=True)
    dev = tw.gpu.device
    g_out = tw.gpu.conv_kg2(torch.stack([g for g, _ in xs]), masks, torch.from_numpy(B).to(dev),
                            torch.from_numpy(rowsum).to(dev), 9, pair * c_n, taps, u_w * u_h, c_n, post=True)
    c_out = tw.cpu.conv_kg2(np.stack([c for _, c in xs]), kern, u_w, u_h, pair, band_only=True)
    assert np.array_equal(tw.gpu.export_words(g_out), c_out)
    if tw.L >= 2:
        want = conv2d_mod_p(x, kern, P)[:, :u_h - 1, :u_w - 1]
        for ob in range(c_o // c_n):
            got = tw.gpu.decrypt_physical(g_out[ob // pair]).reshape(2, -1)[ob % pair]
            got = got.reshape(c_n, u_h, u_w)[:, :u_h - 1, :u_w - 1]
            assert np.array_equal(got, want[ob * c_n:(ob + 1) * c_n])


@pytest.mark.parametrize("ksz,post", [(1, False), (1, True), (5, False), (5, True)])
def test_conv_kg2_kernel_sizes(tw, ksz, post):
    """Schedule 2 with 1x1 kernels (no rotated tap: the decomposition is skipped) and 5x5 kernels."""
    import torch

    from paper_2105_01827_b200.conv import ConvTask, kg2_coefficients, kg2_post_coefficients

    n = tw.bfv.n
    if n not in KG2_GEOM or n < 256:
        pytest.skip("no geometry for this ring")
    u_w, u_h = KG2_GEOM[n]
    c_n = n // (u_w * u_h)
    c_i, c_o, pair = 2 * c_n, 2 * c_n, 2
    kern = tw.rng.integers(-128, 128, (c_o, c_i, ksz, ksz))
    task = ConvTask(u_w, u_h, c_i, ksz, ksz, c_o, kern, tw.params)
    taps = [rot for _, _, rot in task.offsets()]
    tw.keys_for(taps + [d * u_w * u_h for d in range(1, c_n)])
    x = tw.rng.integers(0, P, (c_i, u_h, u_w))
    xs = [tw.encrypt(np.concatenate([b, b]).astype(np.uint32)) for b in x.reshape(c_i // c_n, -1)]
    A, rowsum, K = kg2_coefficients(task, c_n, pair)
    if post:
        A, rowsum = kg2_post_coefficients(A, K, pair * c_n)
    masks = tw.gpu.kg2_encode_masks(ksz, ksz, u_w, u_h, pair, band_only=post)
    dev = tw.gpu.device
    g_out = tw.gpu.conv_kg2(torch.stack([g for g, _ in xs]), masks, torch.from_numpy(A).to(dev),
                            torch.from_numpy(rowsum).to(dev), ksz * ksz, pair * c_n, taps, u_w * u_h, c_n, post=post)
    c_out = tw.cpu.conv_kg2(np.stack([c for _, c in xs]), kern, u_w, u_h, pair, band_only=post)
    assert np.array_equal(tw.gpu.export_words(g_out), c_out)


@pytest.mark.parametrize("T,nb", [(2, 17), (4, 17), (8, 17), (16, 17), (8, 48), (16, 64), (16, 130), (128, 17),
                                  (256, 40), (128, 259)])
def test_mv_gala2_tensor_core_words(tw, T, nb):
    """Tensor-core baby-step sums (byte-convolution int8 MMA) == CUDA-core schedule 2 == oracle o_mv_gala2."""
    import torch

    n = tw.bfv.n
    if T > n or tw.N % 32 or (nb > 256 and tw.N > 4096):
        pytest.skip("shape")               # (two key-folded tiles: checked on the smaller rings)
    b, steps = tw.gpu.bsgs_steps(T)
    if T >= 64:                            # the production split for schedule 2 (Context.gala2_baby)
        b, steps = tw.gpu.bsgs_steps(T, tw.gpu.gala2_baby(T))
    tw.gpu.set_fc_tc_min_terms(1)          # tiles at every T (production: T >= 128)
    try:
        _tensor_core_words(tw, T, nb, b, steps)
    finally:
        tw.gpu.set_fc_tc_min_terms(128)


def _tensor_core_words(tw, T, nb, b, steps):
    import torch

    if not tw.gpu.fc_tc_supported(T, b):
        pytest.skip("tensor-core path not applicable")
    tw.keys_for(steps)
    pts = tw.slots(T)
    pts2 = tw.gpu.encode_gala_weights(pts, b)
    wcan = tw.gpu.fc_tc_weights(pts2, T, b)
    # key-folded tiles of 256 inputs: 17 .. 130 = one partial tile, 259 = 256 + 3 (two tiles)
    xs = [tw.encrypt(tw.slots()) for _ in range(nb)]
    rs = tw.slots(nb)
    cts = torch.stack([g for g, _ in xs])
    d_r = tw.gpu.to_device_u32(rs)
    outs, masked = tw.gpu.mv_gala2_batch(cts, pts2, T, d_r, b, wcan=wcan)
    outs1, masked1 = tw.gpu.mv_gala2_batch(cts, pts2, T, d_r, b)
    assert np.array_equal(tw.gpu.export_words(outs), tw.gpu.export_words(outs1))
    assert np.array_equal(tw.gpu.export_words(masked), tw.gpu.export_words(masked1))
    for i in (0, nb - 1):
        g, c = xs[i]
        c_out, c_masked = tw.cpu.mv_gala(c, pts, rs[i], baby=b, schedule=2)
        assert np.array_equal(tw.gpu.export_words(outs[i]), c_out)
        assert np.array_equal(tw.gpu.export_words(masked[i]), c_masked)


def test_rotate_batch_words(tw):
    """Batched hoisted rotations == per-input rotations == oracle."""
    import torch

    n = tw.bfv.n
    steps = sorted({1 % n, 3 % n, (n - 1) % n} - {0})
    if not steps:
        pytest.skip("tiny")
    tw.keys_for(steps)
    xs = [tw.encrypt(tw.slots()) for _ in range(3)]
    outs = tw.gpu.rotate_batch(torch.stack([g for g, _ in xs]), steps)
    for b, (g, c) in enumerate(xs):
        want = tw.cpu.rotate_hoisted(c, steps)
        for i in range(len(steps)):
            assert np.array_equal(tw.gpu.export_words(outs[b, i]), want[i])


@pytest.mark.parametrize("form", ["hoist", "generic"])
def test_rotate_batch_forms_words(tw, form, monkeypatch):
    """Hoisted rotations of a batch through k_ks_hoist (step keys shared by up to 8 inputs per thread) and
    through the generic k_ks_mac (GALA_KS_HOIST) == oracle, word for word."""
    import torch

    n = tw.bfv.n
    steps = sorted({1 % n, 2 % n, 5 % n, (n - 1) % n} - {0})
    if len(steps) < 2:
        pytest.skip("tiny")
    if form == "generic":
        monkeypatch.setenv("GALA_KS_HOIST", "off")
    tw.keys_for(steps)
    xs = [tw.encrypt(tw.slots()) for _ in range(11)]
    outs = tw.gpu.rotate_batch(torch.stack([g for g, _ in xs]), steps)
    for b in (0, 5, 10):
        want = tw.cpu.rotate_hoisted(xs[b][1], steps)
        for i in range(len(steps)):
            assert np.array_equal(tw.gpu.export_words(outs[b, i]), want[i])


@pytest.mark.parametrize("form", ["force", "off"])
def test_mv_gala2_giant_forms_words(tw, form, monkeypatch):
    """FC giant-step key switches through k_ks_giant (forced on this small ring; production enables it when
    its grid fills the GPU) and through the generic k_ks_mac == oracle o_mv_gala2, word for word."""
    import torch

    n = tw.bfv.n
    T = min(16, n)
    b, steps = tw.gpu.bsgs_steps(T, 4 if T >= 16 else None)
    if T // b < 2:
        pytest.skip("one giant group")
    monkeypatch.setenv("GALA_KS_GIANT", form)
    tw.keys_for(steps)
    pts = tw.slots(T)
    pts2 = tw.gpu.encode_gala_weights(pts, b)
    nb = 5
    xs = [tw.encrypt(tw.slots()) for _ in range(nb)]
    rs = tw.slots(nb)
    _, masked = tw.gpu.mv_gala2_batch(torch.stack([g for g, _ in xs]), pts2, T, tw.gpu.to_device_u32(rs), b)
    for i in (0, nb - 1):
        _, c_masked = tw.cpu.mv_gala(xs[i][1], pts, rs[i], baby=b, schedule=2)
        assert np.array_equal(tw.gpu.export_words(masked[i]), c_masked)


def test_conv_kg2_post_batch_words(tw):
    """Batched post-mask convolution (several images in one pass) == per-image calls == oracle."""
    import torch

    from paper_2105_01827_b200.conv import ConvTask, kg2_coefficients, kg2_post_coefficients

    n = tw.bfv.n
    if n not in KG2_GEOM:
        pytest.skip("no geometry for this ring")
    u_w, u_h = KG2_GEOM[n]
    c_n = n // (u_w * u_h)
    c_i, c_o, pair, nimg = 2 * c_n, 2 * c_n, 2, 3
    kern = tw.rng.integers(-128, 128, (c_o, c_i, 3, 3))
    task = ConvTask(u_w, u_h, c_i, 3, 3, c_o, kern, tw.params)
    taps = [rot for _, _, rot in task.offsets()]
    tw.keys_for(taps + [d * u_w * u_h for d in range(1, c_n)])
    A, _, K = kg2_coefficients(task, c_n, pair)
    B, rowsum = kg2_post_coefficients(A, K, pair * c_n)
    masks = tw.gpu.kg2_encode_masks(3, 3, u_w, u_h, pair, band_only=True)
    dev = tw.gpu.device
    dB, drs = torch.from_numpy(B).to(dev), torch.from_numpy(rowsum).to(dev)
    imgs = []
    for _ in range(nimg):
        x = tw.rng.integers(0, P, (c_i, u_h, u_w))
        imgs.append([tw.encrypt(np.concatenate([b, b]).astype(np.uint32)) for b in x.reshape(c_i // c_n, -1)])
    g_batch = torch.stack([torch.stack([g for g, _ in im]) for im in imgs])
    outs = tw.gpu.conv_kg2_batch(g_batch, masks, dB, drs, 9, pair * c_n, taps, u_w * u_h, c_n)
    for i, im in enumerate(imgs):
        c_out = tw.cpu.conv_kg2(np.stack([c for _, c in im]), kern, u_w, u_h, pair, band_only=True)
        assert np.array_equal(tw.gpu.export_words(outs[i]), c_out)


@pytest.mark.parametrize("coef", ["1", "0"])
@pytest.mark.parametrize("tc", [False, True])
def test_mv_gala2_stream_host_words(tw, tc, coef, monkeypatch):
    """Streamed host entry point (S batches from host memory, copies overlapped with the layers) ==
    oracle o_mv_gala2 for every batch, word for word; key-folded layers with the coefficient-domain
    finish (k_moddown_coef, the default) and with the NTT-domain ModDown + export (GALA_STREAM_COEF=0)."""
    if coef == "0" and not tc:
        pytest.skip("the coefficient-domain finish only applies to key-folded layers")
    monkeypatch.setenv("GALA_STREAM_COEF", coef)
    n = tw.bfv.n
    T = min(8, n)
    b, steps = tw.gpu.bsgs_steps(T)
    tw.gpu.set_fc_tc_min_terms(1 if tc else 128)      # the key-folded tile at this small T (production: T >= 128)
    try:
        _stream_words(tw, tc, T, b, steps)
    finally:
        tw.gpu.set_fc_tc_min_terms(128)


def _stream_words(tw, tc, T, b, steps):
    import ctypes

    from paper_2105_01827_b200 import _lib

    if tc and (tw.N % 32 or not tw.gpu.fc_tc_supported(T, b)):
        pytest.skip("tensor-core path not applicable")
    tw.keys_for(steps)
    pts = tw.slots(T)
    pts2 = tw.gpu.encode_gala_weights(pts, b)
    wcan = tw.gpu.fc_tc_weights(pts2, T, b) if tc else None
    S, B = 3, (17 if tc else 2)
    xs = [[tw.encrypt(tw.slots()) for _ in range(B)] for _ in range(S)]
    rs = tw.slots(S * B).reshape(S, B, tw.N)
    host_ct = np.ascontiguousarray(np.stack([np.stack([tw.gpu.export_words(g) for g, _ in batch]) for batch in xs]))
    host_out = np.zeros_like(host_ct)
    r = np.ascontiguousarray(rs.astype(np.uint32))
    _lib.check(tw.gpu.lib.gala_mv_gala2_stream_host(
        tw.gpu._bind(), ctypes.c_void_p(host_ct.ctypes.data), S, B, ctypes.c_void_p(pts2.data_ptr()),
        ctypes.c_void_p(wcan.data_ptr() if wcan is not None else None), T, b, ctypes.c_void_p(r.ctypes.data),
        ctypes.c_void_p(host_out.ctypes.data)))
    for s in range(S):
        for i in (0, B - 1):
            _, c_masked = tw.cpu.mv_gala(xs[s][i][1], pts, rs[s, i], baby=b, schedule=2)
            assert np.array_equal(host_out[s, i], c_masked), f"batch {s} input {i}"


def test_conv_kg_batch_odd_rows_words(tw):
    """Batched first-Add with an odd accumulator-row count (c_n = 1, 3 outputs: the 2-row register
    tile's tail) and an odd image count == oracle per image."""
    n = tw.bfv.n
    if n < 16:
        pytest.skip("tiny")
    c_n, k, n_ib, n_obp, nimg = 1, 3, 2, 3, 3
    tap_steps = [0, 1, n - 1]
    tw.keys_for(tap_steps)
    imgs = [[tw.encrypt(tw.slots()) for _ in range(n_ib)] for _ in range(nimg)]
    pts = tw.slots(n_obp * n_ib * c_n * k).reshape(n_obp, n_ib, c_n, k, tw.N)
    import torch

    d_pts = tw.gpu.encode_plain(pts.reshape(-1, tw.N)).view(n_obp, n_ib, c_n, k, tw.L, tw.N)
    outs = tw.gpu.conv_kg_batch(torch.stack([torch.stack([g for g, _ in im]) for im in imgs]), d_pts, tap_steps, n)
    for b, im in enumerate(imgs):
        c_out = tw.cpu.conv_kg(np.stack([c for _, c in im]), pts, tap_steps, n)
        assert np.array_equal(tw.gpu.export_words(outs[b]), c_out), f"image {b}"
