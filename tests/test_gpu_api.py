"""Drop-in API on the GPU backend, against the reference's golden outputs and
the reference's own behavioural tests (pkg/tests/test_backend.py,
test_matvec.py, test_conv.py, test_sharing.py)."""
import os

import numpy as np
import pytest

from oracle.plain import conv2d_mod_p, dot_mod_p
from paper_2105_01827_b200 import (
    ConvTask,
    CostMeter,
    GalaFC,
    HEParams,
    KernelGroupingConv,
    MockCiphertext,
    MvTask,
    OpCounts,
    SlotVector,
    column_blocks,
    count_conv,
    count_mv,
    decrypt,
    encrypt,
    encrypt_inputs,
    gen_additive_share,
    he_add,
    he_decperm,
    he_hstperm,
    he_perm,
    he_scmult,
    mimo_kernel_grouping,
    mimo_output_rotation,
    pointwise,
    predict_noise,
    rotate_left,
    run_mv,
    siso_conv,
    subtract_plain,
    unpack_channels,
    with_overrides,
)
from paper_2105_01827_b200.errors import DimensionError, NoiseOverflowError

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
P = 1032193
BASE = HEParams()
PARAMS64 = with_overrides(BASE, n=64)


def fresh(rng, params=PARAMS64):
    return encrypt(SlotVector(rng.integers(0, P, params.n), P), params)


# --- golden fixtures from the reference ------------------------------------------
MV = np.load(os.path.join(GOLD, "mv_gala.npz"))
CV = np.load(os.path.join(GOLD, "conv_kg.npz"))
OPS = np.load(os.path.join(GOLD, "ops.npz"))


@pytest.mark.parametrize("idx", range(int(MV["count"][0])))
def test_run_mv_gala_matches_reference(idx):
    n, n_o, n_i, seed, rseed = (int(v) for v in MV[f"c{idx}_dims"])
    params = with_overrides(BASE, n=n)
    w = MV[f"c{idx}_w"].astype(np.int64) % P
    x = MV[f"c{idx}_x"].astype(np.int64)
    meter = CostMeter()
    out = run_mv("gala", MvTask(n_i, n_o, w, params), x, meter, rng=rseed)
    c = OpCounts.from_meter(meter)
    assert [c.perm, c.dec_perm, c.hst_perm, c.sc_mult, c.add, out.share_meter.add] == MV[f"c{idx}_counts"].tolist()
    assert out.output_cipher.noise == float(MV[f"c{idx}_noise"][0])
    assert np.array_equal(out.output_cipher.payload.slots, MV[f"c{idx}_payload"].astype(np.int64))
    assert np.array_equal(out.server_share.slots, MV[f"c{idx}_server"].astype(np.int64))
    assert np.array_equal(out.client_share.slots, MV[f"c{idx}_client"].astype(np.int64))
    assert out.seed == rseed


@pytest.mark.parametrize("idx", range(int(CV["count"][0])))
def test_mimo_kernel_grouping_matches_reference(idx):
    u, c_i, k, c_o, n, seed = (int(v) for v in CV[f"c{idx}_dims"])
    params = with_overrides(BASE, n=n)
    kern = CV[f"c{idx}_kernels"].astype(np.int64) % P
    ch = CV[f"c{idx}_channels"].astype(np.int64)
    task = ConvTask(u, u, c_i, k, k, c_o, kern, params)
    meter = CostMeter()
    outs = mimo_kernel_grouping(task, encrypt_inputs(task, ch), meter)
    c = OpCounts.from_meter(meter)
    assert [c.perm, c.dec_perm, c.hst_perm, c.sc_mult, c.add] == CV[f"c{idx}_counts"].tolist()
    assert [o.noise for o in outs] == CV[f"c{idx}_noise"].tolist()
    got = np.stack([decrypt(o).slots for o in outs])
    assert np.array_equal(got, CV[f"c{idx}_payloads"].astype(np.int64))


def test_ops_match_reference():
    x, y = OPS["x"], OPS["y"]
    meter = CostMeter()
    cx = encrypt(SlotVector(x, P), PARAMS64)
    for k in (1, 5, 17, 63):
        assert np.array_equal(he_perm(cx, k, meter).payload.slots, OPS[f"rot{k}"])
    assert np.array_equal(he_scmult(cx, SlotVector(y, P), meter).payload.slots, OPS["scmult"])
    assert np.array_equal(he_add(cx, encrypt(SlotVector(y, P), PARAMS64), meter).payload.slots, OPS["add"])
    assert np.array_equal(subtract_plain(cx, SlotVector(y, P), meter).payload.slots, OPS["sub"])


# --- reference behaviour: backend -----------------------------------------------------
def test_encrypt_fresh_noise_and_roundtrip():
    rng = np.random.default_rng(0)
    ct = encrypt(SlotVector.zeros(64, P), PARAMS64)
    assert ct.noise == PARAMS64.eta0 == 8.0 and decrypt(ct).tolist() == [0] * 64
    for _ in range(10):
        x = SlotVector(rng.integers(0, P, 64), P)
        assert decrypt(encrypt(x, PARAMS64)) == x
    with pytest.raises(DimensionError):
        encrypt(SlotVector.zeros(32, P), PARAMS64)


def test_decrypt_at_budget_fails():
    ct = MockCiphertext(SlotVector.zeros(64, P), PARAMS64.noise_budget, PARAMS64)
    with pytest.raises(NoiseOverflowError):
        decrypt(ct)


def test_chained_ras_overflow():
    tiny = HEParams(n=64, noise_budget=1e6)
    meter = CostMeter()
    eta, crossing = tiny.eta0, None
    for k in range(1, 41):
        eta = 2 * eta + tiny.eta_rot
        if crossing is None and eta >= tiny.noise_budget:
            crossing = k
    ct = encrypt(SlotVector.zeros(64, tiny.p), tiny)
    for k in range(1, crossing + 1):
        ct = he_add(ct, he_perm(ct, 1, meter), meter)
        if k == crossing - 1:
            assert decrypt(ct).tolist() == [0] * 64
    with pytest.raises(NoiseOverflowError):
        decrypt(ct)


def test_add_scmult_perm_semantics():
    rng = np.random.default_rng(1)
    meter = CostMeter()
    a, b = fresh(rng), fresh(rng)
    c = he_add(a, b, meter)
    assert c.payload == pointwise(a.payload, b.payload, "add") and c.noise == a.noise + b.noise
    ones = SlotVector.constant(1, 64, P)
    s = he_scmult(a, ones, meter)
    assert s.payload == a.payload and s.noise == PARAMS64.eta0 * PARAMS64.eta_mult
    assert he_perm(a, 0, meter) is a and he_perm(a, 64, meter) is a
    r5 = he_perm(a, 5, meter)
    assert r5.payload == rotate_left(a.payload, 5) and r5.noise == PARAMS64.eta0 + PARAMS64.eta_rot
    assert (meter.add, meter.sc_mult, meter.full_perm) == (1, 1, 1)


def test_decperm_hstperm_amortisation_and_words():
    rng = np.random.default_rng(6)
    m1, m2 = CostMeter(), CostMeter()
    a = fresh(rng)
    g = he_decperm(a, m1)
    for k in (0, 1, 17, 63):
        via_group = he_hstperm(g, k, m1)
        via_perm = he_perm(a, k, m2)
        assert via_group.payload == via_perm.payload and via_group.noise == via_perm.noise
        assert np.array_equal(via_group.words(), via_perm.words())   # same words, hoisted or not
    assert he_hstperm(g, 0, m1) is a
    assert m1.dec_perm == 1 and m1.hst_perm == 3 and g.source is a
    he_decperm(a, m1)
    assert m1.dec_perm == 2


def test_params_mismatch_rejected():
    other = HEParams(n=64, p=65537)
    a = encrypt(SlotVector.zeros(64, P), PARAMS64)
    b = encrypt(SlotVector.zeros(64, 65537), other)
    with pytest.raises(DimensionError):
        he_add(a, b, CostMeter())


def test_share_reconstruction_and_determinism():
    rng = np.random.default_rng(1)
    ct = fresh(rng, BASE)
    meter = CostMeter()
    r, masked = gen_additive_share(ct, np.random.default_rng(2), meter)
    assert pointwise(masked.payload, r, "add") == ct.payload
    assert meter.add == 1 and masked.noise == ct.noise + BASE.eta0
    r1, _ = gen_additive_share(ct, 42, CostMeter())
    r2, _ = gen_additive_share(ct, 42, CostMeter())
    assert r1 == r2


# --- schemes ---------------------------------------------------------------------------
@pytest.mark.parametrize("scheme", ["naive", "diagonal", "gazelle", "gala"])
def test_schemes_match_oracle_small_grid(scheme):
    params = with_overrides(BASE, n=256)
    rng = np.random.default_rng(99)
    for n_o, n_i in [(2, 1024), (16, 128), (4, 16)]:
        w = rng.integers(0, P, (n_o, n_i))
        x = rng.integers(0, P, n_i)
        meter = CostMeter()
        got = np.zeros(n_o, dtype=np.int64)
        for wb, xb in column_blocks(w, x, params.n):
            out = run_mv(scheme, MvTask(wb.shape[1], n_o, wb, params), xb, meter, rng=1)
            got = (got + out.server_share.slots + out.client_share.slots) % P
        assert np.array_equal(got, dot_mod_p(w, x, P)), (scheme, n_o, n_i)
    task = MvTask(16, 4, rng.integers(0, P, (4, 16)), params)
    meter = CostMeter()
    run_mv(scheme, task, rng.integers(0, P, 16), meter, rng=0)
    assert OpCounts.from_meter(meter) == count_mv(scheme, 16, 4, 256)


def test_gala_shares_reproducible_and_seed_recorded():
    rng = np.random.default_rng(2)
    task = MvTask(128, 16, rng.integers(0, P, (16, 128)), BASE)
    x = rng.integers(0, P, 128)
    a = run_mv("gala", task, x, CostMeter(), rng=123)
    b = run_mv("gala", task, x, CostMeter(), rng=123)
    assert a.seed == b.seed == 123 and a.server_share == b.server_share and a.client_share == b.client_share
    c = run_mv("gala", task, x, CostMeter(), rng=124)
    assert c.server_share != a.server_share


@pytest.mark.parametrize("u_w,u_h,c_i,k,c_o,n", [(4, 4, 4, 3, 8, 64), (4, 4, 8, 1, 8, 128), (4, 4, 8, 3, 8, 128)])
def test_mimo_schemes_agree(u_w, u_h, c_i, k, c_o, n):
    params = with_overrides(BASE, n=n)
    rng = np.random.default_rng(c_i * k + c_o)
    kern = rng.integers(0, P, (c_o, c_i, k, k))
    ch = rng.integers(0, P, (c_i, u_h, u_w))
    task = ConvTask(u_w, u_h, c_i, k, k, c_o, kern, params)
    want = conv2d_mod_p(ch, kern, P)
    for name, fn in (("gazelle", mimo_output_rotation), ("gala", mimo_kernel_grouping)):
        meter = CostMeter()
        outs = fn(task, encrypt_inputs(task, ch), meter)
        got = np.concatenate([unpack_channels(decrypt(o), task) for o in outs])
        assert np.array_equal(got, want), name
        assert OpCounts.from_meter(meter) == count_conv(name, u_w, u_h, c_i, c_o, k, k, n)
        eta = predict_noise(f"conv_{name}", (u_w, u_h, c_i, c_o, k, k), params)
        assert all(o.noise == eta for o in outs)


def test_siso_corner_term_and_identity():
    params = with_overrides(BASE, n=16)
    rng = np.random.default_rng(1)
    kern = rng.integers(0, P, (1, 1, 3, 3))
    img = rng.integers(0, P, (1, 3, 3))
    task = ConvTask(3, 3, 1, 3, 3, 1, kern, params)
    vec = np.zeros(16, dtype=np.int64)
    vec[:9] = img.ravel()
    meter = CostMeter()
    out = siso_conv(task, encrypt(SlotVector(vec, P), params), meter)
    m, f = img[0], kern[0, 0]
    want = (m[0, 0] * f[1, 1] + m[0, 1] * f[1, 2] + m[1, 0] * f[2, 1] + m[1, 1] * f[2, 2]) % P
    assert decrypt(out).slots[0] == want
    assert OpCounts.from_meter(meter) == OpCounts(dec_perm=1, hst_perm=8, sc_mult=9, add=8)


def test_channel_rotation_wraparound():
    n, u, c_n = 64, 4, 4
    params = with_overrides(BASE, n=n)
    kernels = np.zeros((c_n, c_n, 1, 1), dtype=np.int64)
    for o in range(c_n):
        for i in range(c_n):
            kernels[o, i, 0, 0] = 100 * o + i + 1
    task = ConvTask(u, u, c_n, 1, 1, c_n, kernels, params)
    for hot in range(c_n):
        channels = np.zeros((c_n, u, u), dtype=np.int64)
        channels[hot] = 1
        outs = mimo_kernel_grouping(task, encrypt_inputs(task, channels), CostMeter())
        got = unpack_channels(decrypt(outs[0]), task)
        for o in range(c_n):
            assert np.all(got[o] == 100 * o + hot + 1)


# --- BASELINE.json configs at full size (size-independent properties) ------------------
def _int8(rng, shape):
    return rng.integers(-128, 128, shape) % P


def test_cfg1_fc_16x2048_n4096():
    params = HEParams(n=2048, rns_limbs=1, seed=21)   # N = 4096, single 62-bit prime + special prime
    assert params.bfv().N == 4096 and params.bfv().L == 1
    rng = np.random.default_rng(1)
    w, x = _int8(rng, (16, 2048)), rng.integers(0, P, 2048)
    layer = GalaFC(w, params)
    assert layer.T == 8                          # two 8x2048 tasks paired on the hypercube rows
    masks = layer.draw_masks(7)
    masked = layer.forward_device(layer.encrypt_input(x), masks)
    got = (layer.client_shares(masked) + layer.server_shares(masks)) % P
    assert np.array_equal(got, dot_mod_p(w, x, P))


def test_cfg2_fc_1024x4096_n8192():
    params = HEParams(n=4096, rns_limbs=3, seed=22)
    rng = np.random.default_rng(2)
    w, x = _int8(rng, (1024, 4096)), rng.integers(0, P, 4096)
    layer = GalaFC(w, params)
    assert layer.T == 512 and layer.baby == 64      # schedule-2 baby count (Context.gala2_baby)
    masks = layer.draw_masks(8)
    masked = layer.forward_device(layer.encrypt_input(x), masks)
    got = (layer.client_shares(masked) + layer.server_shares(masks)) % P
    assert np.array_equal(got, dot_mod_p(w, x, P))


def test_cfg3_conv_16x16x64_n4096():
    params = HEParams(n=2048, rns_limbs=1, seed=23)
    rng = np.random.default_rng(3)
    kern, ch = _int8(rng, (64, 64, 3, 3)), rng.integers(0, P, (64, 16, 16))
    task = ConvTask(16, 16, 64, 3, 3, 64, kern, params)
    meter = CostMeter()
    outs = KernelGroupingConv(task)(encrypt_inputs(task, ch), meter)
    got = np.concatenate([unpack_channels(decrypt(o), task) for o in outs])
    assert np.array_equal(got, conv2d_mod_p(ch, kern, P))
    assert OpCounts.from_meter(meter) == OpCounts(perm=56, dec_perm=8, hst_perm=64, sc_mult=4608, add=4600)


def test_cfg4_conv_56x56x64_in_64x64_frame_n8192():
    params = HEParams(n=4096, rns_limbs=3, seed=24)
    rng = np.random.default_rng(4)
    kern, ch = _int8(rng, (64, 64, 3, 3)), rng.integers(0, P, (64, 56, 56))
    frame = np.zeros((64, 64, 64), dtype=np.int64)
    frame[:, :56, :56] = ch                      # zero-embedding
    task = ConvTask(64, 64, 64, 3, 3, 64, kern, params)
    meter = CostMeter()
    outs = KernelGroupingConv(task)(encrypt_inputs(task, frame), meter)
    got = np.concatenate([unpack_channels(decrypt(o), task) for o in outs])[:, :56, :56]
    assert np.array_equal(got, conv2d_mod_p(ch, kern, P))
    assert OpCounts.from_meter(meter) == OpCounts(perm=0, dec_perm=64, hst_perm=512, sc_mult=36864, add=36800)


@pytest.mark.parametrize("u,c_i,k,c_o,n", [(4, 8, 3, 16, 64), (16, 64, 3, 64, 2048), (8, 4, 5, 4, 64), (2, 4, 3, 4, 16)])
def test_gpu_weight_encoding_equals_host_encoding(u, c_i, k, c_o, n):
    """On-GPU coef_vectors + encode == the reference-order host construction, word for word."""
    params = with_overrides(BASE, n=n)
    rng = np.random.default_rng(u + c_i)
    task = ConvTask(u, u, c_i, k, k, c_o, rng.integers(0, P, (c_o, c_i, k, k)), params)
    for pair in (True, False):
        a = KernelGroupingConv(task, pair_rows=pair, schedule=1, drop_plaintexts=False)
        b = KernelGroupingConv(task, pair_rows=pair, host_encode=True)
        assert bool((a.pts == b.pts).all())


# --- config 5 building blocks: frames, halo tiling, strides, padded FC -----------------
def test_resnet_rules_small():
    from paper_2105_01827_b200.resnet import ConvLayer, FCLayer, LayerSpec

    params = HEParams(n=1024, seed=25)           # frames up to 32x32
    rng = np.random.default_rng(5)
    cases = [LayerSpec("tiled7x7s2", "conv", 3, 4, 7, 2, 70),      # 70 > 32: halo tiles, stride 2
             LayerSpec("s2", "conv", 4, 8, 3, 2, 14),              # 14 -> 16 frame, stride 2
             LayerSpec("ds1x1s2", "conv", 4, 8, 1, 2, 28),         # 1x1 downsample
             LayerSpec("s1", "conv", 16, 16, 3, 1, 7)]             # 7 -> 8 frame, c_n = 16
    for spec in cases:
        w = rng.integers(-128, 128, (spec.c_out, spec.c_in, spec.k, spec.k)) % P
        x = rng.integers(0, P, (spec.c_in, spec.size, spec.size))
        layer = ConvLayer(spec, w, params)
        got = layer.decrypt_output(layer.forward_device(layer.encrypt_frames(x)))
        want = conv2d_mod_p(x, w, P)[:, ::spec.stride, ::spec.stride]
        assert got.shape == (spec.c_out, spec.out_size, spec.out_size)
        assert np.array_equal(got, want), spec.name
    spec = LayerSpec("fc", "fc", 24, 40)
    w = rng.integers(-128, 128, (40, 24)) % P
    x = rng.integers(0, P, 24)
    fc = FCLayer(spec, w, params)
    masks = fc.layer.draw_masks(3)
    assert np.array_equal(fc.shares(fc.forward_device(fc.encrypt_frames(x), masks), masks), dot_mod_p(w, x, P))


def test_kg_schedule1_image_batch():
    """Schedule 1 over a batch of images sharing the weights (gala_conv_kg_batch) decrypts to
    conv2d mod p for every image and equals the one-image calls word for word."""
    import torch

    params = HEParams(n=256, seed=41)
    rng = np.random.default_rng(8)
    u, c_i, c_o, k = 8, 8, 8, 3                      # c_n = 4: 2 input cts, 2 output blocks
    kern = rng.integers(-128, 128, (c_o, c_i, k, k)) % P
    task = ConvTask(u, u, c_i, k, k, c_o, kern, params)
    layer = KernelGroupingConv(task, schedule=1, tensor_cores=False)
    assert layer.batchable
    imgs = [rng.integers(0, P, (c_i, u, u)) for _ in range(5)]
    cts = [encrypt_inputs(task, im) for im in imgs]
    outs = layer.forward_device_batch(torch.stack([torch.stack([c.data for c in cc]) for cc in cts]))
    ctx = layer.ctx
    n = params.n
    for b, im in enumerate(imgs):
        one = layer.forward_device(torch.stack([c.data for c in cts[b]]))
        assert np.array_equal(ctx.export_words(outs[b]), ctx.export_words(one))
        got = np.concatenate([ctx.decrypt_physical(outs[b][ob // 2])[(ob % 2) * n:(ob % 2 + 1) * n]
                              .reshape(layer.c_n, u, u) for ob in range(layer.n_ob)])
        assert np.array_equal(got, conv2d_mod_p(im, kern, P))


def test_sharded_conv_single_rank_is_the_layer():
    """ShardedKernelGroupingConv at world size 1 is mimo_kernel_grouping: same words, same counts,
    same noise (the multi-rank path is covered by the gloo world-2 test)."""
    from paper_2105_01827_b200.sharding import ShardedKernelGroupingConv

    params = HEParams(n=256, seed=42)
    rng = np.random.default_rng(9)
    u, c_i, c_o, k = 8, 8, 12, 3
    kern = rng.integers(-128, 128, (c_o, c_i, k, k)) % P
    task = ConvTask(u, u, c_i, k, k, c_o, kern, params)
    img = rng.integers(0, P, (c_i, u, u))
    cts = encrypt_inputs(task, img)
    m1, m2 = CostMeter(), CostMeter()
    want = mimo_kernel_grouping(task, cts, m1)
    got = ShardedKernelGroupingConv(task)(cts, m2)
    assert repr(m1) == repr(m2)
    for a, b in zip(want, got):
        assert a.noise == b.noise
        assert np.array_equal(decrypt(a).slots, decrypt(b).slots)
    dec = np.concatenate([unpack_channels(decrypt(o), task) for o in got])
    assert np.array_equal(dec, conv2d_mod_p(img, kern, P))


def test_real_noise_guard():
    """Real noise past Delta / 4 raises instead of returning wrong slots (GAZELLE's fold after the
    plaintext product at one 62-bit prime); the same circuit at L = 2 decrypts correctly."""
    from paper_2105_01827_b200.errors import NoiseOverflowError
    from paper_2105_01827_b200.matvec import mv_hybrid_gazelle, pack_input

    rng = np.random.default_rng(3)
    w = rng.integers(-128, 128, (16, 2048)) % P
    x = rng.integers(0, P, 2048)
    for L, ok in ((1, False), (2, True)):
        params = HEParams(n=2048, p=P, rns_limbs=L, seed=61)
        task = MvTask(2048, 16, w, params)
        ct = encrypt(pack_input(x, task), params)
        if ok:
            out = mv_hybrid_gazelle(task, ct, CostMeter(), rng=5)
            assert np.array_equal((out.client_share.slots + out.server_share.slots) % P, dot_mod_p(w, x, P))
            assert ct.ctx.last_noise_frac < 0.25
        else:
            with pytest.raises(NoiseOverflowError):
                mv_hybrid_gazelle(task, ct, CostMeter(), rng=5)
    # a fresh ciphertext is far below the limit
    assert decrypt(ct).slots is not None and ct.ctx.last_noise_frac < 1e-6
