"""Word-level parity at the BASELINE.json sizes: every output ciphertext of the product's layer
objects equals the CPU oracle's (oracle/bfv_oracle.c), word for word, given the same secret, keys
and encryption randomness (twins.Mirror replays the seeded context's streams).

* config 1 -- FC 16x2048, N = 4096, one prime: a batch of 64 layers (tensor-core schedule 2);
* config 2 -- FC 1024x4096, N = 8192, L = 3: inputs 0, 15 and 31 of a 32-input tensor-core tile;
* config 3 -- conv 16x16x64 -> 64, N = 4096, one prime: the row-paired layer, a 16-image batch
  (images 0 and 15) and the drop-in ``mimo_kernel_grouping`` (one block per ciphertext);
* config 4 -- conv 56x56x64 -> 64 in 64x64 frames, N = 8192, L = 3, c_n = 1: the production
  post-mask tcgen05 layer and the drop-in pre-mask path;
* config 5 -- ResNet-18 at 224x224: conv1 (16 halo tiles, batched), a c_n = 4 layer, a c_n = 64
  layer (tensor-core schedule 1) and the padded 1024x1024 FC.

Reference: matvec.py:305-320 (mv_gala), conv.py:268-293 (mimo_kernel_grouping).
"""
import zlib

import numpy as np
import pytest

from oracle.plain import conv2d_mod_p, dot_mod_p
from paper_2105_01827_b200.backend import Ciphertext, CostMeter, HEParams
from paper_2105_01827_b200.conv import (
    ConvTask,
    DiagonalPlan,
    KernelGroupingConv,
    centred_kernels,
    encode_channel_blocks,
    mimo_kernel_grouping,
    unpack_channels,
)
from paper_2105_01827_b200.matvec import GalaFC, gala_weight_slots
from twins import P, Mirror

pytestmark = pytest.mark.gpu


def _int8(rng, shape):
    return rng.integers(-128, 128, shape) % P


def kg1_slots(task, pair):
    """Physical slot plaintexts [n_obp][n_ib][c_n][k][N] of a schedule-1 layer (coef_vectors,
    conv.py:220-235; blocks ob = pair*obp + row on the hypercube rows)."""
    c_n, n = task.channels_per_ct, task.params.n
    n_ib, n_ob = task.c_i // c_n, task.c_o // c_n
    n_obp = (n_ob + pair - 1) // pair
    plan = DiagonalPlan(task, c_n)
    k = len(task.offsets())
    zeros = np.zeros((c_n, k, n), dtype=np.int64)
    pts = np.zeros((n_obp, n_ib, c_n, k, 2 * n), dtype=np.uint32)
    for obp in range(n_obp):
        for ib in range(n_ib):
            rows = [np.stack([plan.coef_slots(ob, ib, d) for d in range(c_n)]) if ob < n_ob else zeros
                    for ob in range(pair * obp, pair * obp + pair)]
            if pair == 1:
                rows.append(rows[0])
            pts[obp, ib] = np.concatenate(rows, axis=2)
    return pts


def oracle_kg(mir, layer, cts):
    """The oracle's output words for `layer` (its schedule, pairing and mask form) on cts [n_ib][2][L][N]."""
    task = layer.task
    if layer.schedule == 2:
        return mir.cpu.conv_kg2(cts, centred_kernels(task), task.u_w, task.u_h, layer.pair, band_only=layer.post)
    return mir.cpu.conv_kg(cts, kg1_slots(task, layer.pair), layer.tap_steps, layer.band)


def encrypt_blocks(mir, task, img):
    import torch

    g, c = [], []
    for b in encode_channel_blocks(task, img):
        gg, cc = mir.encrypt(np.concatenate([b.slots, b.slots]).astype(np.uint32))
        g.append(gg)
        c.append(cc)
    return torch.stack(g), np.stack(c)


def fc_case(mir, w, B, check):
    """B inputs through GalaFC.run_batch; words of inputs `check` == oracle o_mv_gala(2)."""
    import torch

    layer = GalaFC(w, mir.params)
    mir.sync_keys()
    ctx, rng = layer.ctx, np.random.default_rng(3)
    tasks = layer.blocks[0][0]
    phys_w = np.concatenate([gala_weight_slots(t) for t in tasks], axis=1).astype(np.uint32)
    xs = [rng.integers(0, P, layer.n_in) for _ in range(B)]
    enc = [mir.encrypt(ctx.physical(np.tile(x, tasks[0].copies))) for x in xs]
    rs = [ctx.physical(rng.integers(0, P, mir.params.n), rng.integers(0, P, mir.params.n)) for _ in range(B)]
    cts = torch.stack([g for g, _ in enc])
    _, masked = layer.run_batch(cts, layer.blocks[0][1], ctx.to_device_u32(np.stack(rs)), block=0)
    got = ctx.export_words(masked)
    for b in check:
        _, want = mir.cpu.mv_gala(enc[b][1], phys_w, rs[b], baby=layer.baby, schedule=layer.schedule)
        assert np.array_equal(got[b], want), b
    return layer, xs, rs, masked


def test_cfg1_fc_batch_words():
    mir = Mirror(HEParams(n=2048, rns_limbs=1, seed=301))
    w = _int8(np.random.default_rng(1), (16, 2048))
    layer, xs, rs, masked = fc_case(mir, w, 64, range(64))
    assert layer.T == 8 and mir.L == 1
    n = mir.params.n
    for b in (0, 63):   # and the shares reconstruct W x
        v = layer.client_shares([masked[b]])
        srv = layer.server_shares([[SV(rs[b][:n]), SV(rs[b][n:])]])
        assert np.array_equal((v + srv) % P, dot_mod_p(w, xs[b], P))


def SV(a):
    from paper_2105_01827_b200.ring import SlotVector

    return SlotVector(a.astype(np.int64), P)


def test_cfg2_fc_tensor_core_tile_words():
    mir = Mirror(HEParams(n=4096, rns_limbs=3, seed=302))
    w = _int8(np.random.default_rng(2), (1024, 4096))
    layer, _, _, _ = fc_case(mir, w, 32, (0, 15, 31))
    assert (layer.T, layer.baby, layer.schedule) == (512, 64, 2) and layer.wcan[0] is not None


def test_cfg3_conv_words_paired_batched_and_drop_in():
    import torch

    mir = Mirror(HEParams(n=2048, rns_limbs=1, seed=303))
    rng = np.random.default_rng(3)
    kern = _int8(rng, (64, 64, 3, 3))
    task = ConvTask(16, 16, 64, 3, 3, 64, kern, mir.params)
    layer = KernelGroupingConv(task)
    assert layer.schedule == 1 and layer.pair == 2
    mir.sync_keys()
    imgs = [rng.integers(0, P, (64, 16, 16)) for _ in range(16)]
    enc = [encrypt_blocks(mir, task, im) for im in imgs]
    out = layer.forward_device(enc[0][0])
    want0 = oracle_kg(mir, layer, enc[0][1])
    assert np.array_equal(layer.ctx.export_words(out), want0)
    # the 16-image batch (gala_conv_kg_batch)
    outb = layer.forward_device_batch(torch.stack([g for g, _ in enc]))
    assert np.array_equal(layer.ctx.export_words(outb[0]), want0)
    assert np.array_equal(layer.ctx.export_words(outb[15]), oracle_kg(mir, layer, enc[15][1]))
    # the drop-in: one output block per ciphertext, replicated
    cts = [Ciphertext._wrap(g, mir.params.eta0, mir.params, replicated=True) for g in enc[1][0]]
    outs = mimo_kernel_grouping(task, cts, CostMeter())
    single = KernelGroupingConv(task, pair_rows=False)
    want1 = oracle_kg(mir, single, enc[1][1])
    assert np.array_equal(np.stack([o.words() for o in outs]), want1)
    got = np.concatenate([unpack_channels(o.payload, task) for o in outs])
    assert np.array_equal(got, conv2d_mod_p(imgs[1], kern, P))


def test_cfg4_conv_production_and_drop_in_words():
    mir = Mirror(HEParams(n=4096, rns_limbs=3, seed=304))
    rng = np.random.default_rng(4)
    kern = _int8(rng, (64, 64, 3, 3))
    img = np.zeros((64, 64, 64), dtype=np.int64)
    img[:, :56, :56] = rng.integers(0, P, (64, 56, 56))
    task = ConvTask(64, 64, 64, 3, 3, 64, kern, mir.params)
    prod = KernelGroupingConv(task, band_only=True)          # production: post-mask, fused tcgen05 first-Add
    assert (prod.schedule, prod.post, prod.pair, prod.c_n) == (2, True, 2, 1)
    mir.sync_keys()
    g, c = encrypt_blocks(mir, task, img)
    assert np.array_equal(prod.ctx.export_words(prod.forward_device(g)), oracle_kg(mir, prod, c))
    # the drop-in mimo_kernel_grouping: pre-mask form (tap-validity masks), one block per ciphertext
    cts = [Ciphertext._wrap(x, mir.params.eta0, mir.params, replicated=True) for x in g]
    outs = mimo_kernel_grouping(task, cts, CostMeter())
    single = KernelGroupingConv(task, pair_rows=False)
    assert (single.schedule, single.post) == (2, False)
    assert np.array_equal(np.stack([o.words() for o in outs]), oracle_kg(mir, single, c))
    got = np.concatenate([unpack_channels(o.payload, task) for o in outs])[:, :56, :56]
    assert np.array_equal(got, conv2d_mod_p(img[:, :56, :56], kern, P))


@pytest.fixture(scope="module")
def resnet_mirror():
    return Mirror(HEParams(n=4096, rns_limbs=3, seed=305))


@pytest.mark.parametrize("name", ["conv1", "layer2.1.conv1", "layer4.1.conv1"])
def test_cfg5_resnet18_layer_words(resnet_mirror, name):
    import torch

    from paper_2105_01827_b200.resnet import ConvLayer, resnet18_224

    mir = resnet_mirror
    spec = next(s for s in resnet18_224() if s.name == name)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    w = _int8(rng, (spec.c_out, spec.c_in, spec.k, spec.k))
    x = rng.integers(0, P, (spec.c_in, spec.size, spec.size))
    layer = ConvLayer(spec, w, mir.params)
    kg = layer.kg
    mir.sync_keys()
    frames = [(oy, ox, encrypt_blocks(mir, layer.task, fr)) for oy, ox, fr in layer.frames(x)]
    outs = layer.forward_device([(oy, ox, g) for oy, ox, (g, _) in frames])
    for (oy, ox, (_, c)), (_, _, o) in zip(frames, outs):
        assert np.array_equal(layer.ctx.export_words(o), oracle_kg(mir, kg, c)), (name, oy, ox)
    got = layer.decrypt_output(outs)
    assert np.array_equal(got, conv2d_mod_p(x, w, P)[:, ::spec.stride, ::spec.stride])
    expect = {"conv1": (2, 1, 16), "layer2.1.conv1": (2, 4, 1), "layer4.1.conv1": (1, 64, 1)}[name]
    assert (kg.schedule, kg.c_n, len(frames)) == expect
    del torch


def test_cfg5_resnet18_fc_words(resnet_mirror):
    mir = resnet_mirror
    w = np.zeros((1024, 1024), dtype=np.int64)
    w[:1000, :512] = _int8(np.random.default_rng(5), (1000, 512))    # profiler._fc_padded rule
    layer, _, _, _ = fc_case(mir, w, 4, range(4))
    assert layer.T == 128
