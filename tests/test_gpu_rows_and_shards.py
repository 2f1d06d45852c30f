"""Hypercube-row bookkeeping of logical ciphertexts and the multi-rank KG layer on CUDA.

* Chained convolutions through the drop-in ``mimo_kernel_grouping`` (conv.py:268-293) give
  ``conv2d_mod_p`` of ``conv2d_mod_p``, and their outputs combine with every op (the reference
  accepts both).  Row-paired layer outputs are either used correctly (one row) or rejected with
  DimensionError -- never silently wrong.
* ``ShardedKernelGroupingConv`` with the real CUDA sub-layers on two gloo ranks (both on cuda:0,
  host-staged collectives): the gathered words equal the single-rank layer's, with uneven shards
  whose kernels alone would pick a different schedule than the full layer.
* ``ShardedGalaFC``: one schedule-2 FC layer split across 2 and 3 ranks by its BSGS giant groups;
  the exact u64 reduce of the QP partial sums and the root's single final ModDown give the
  single-GPU layer's words (backend.py:134-139).
"""
import os
import socket

import numpy as np
import pytest

from oracle.plain import conv2d_mod_p
from paper_2105_01827_b200 import (
    ConvTask,
    CostMeter,
    HEParams,
    KernelGroupingConv,
    decrypt,
    encrypt_inputs,
    he_add,
    mimo_kernel_grouping,
    unpack_channels,
)
from paper_2105_01827_b200.errors import DimensionError

pytestmark = pytest.mark.gpu

P = 1032193
# three 60-bit primes: a convolution of a convolution stays far inside Delta / 4 (one 62-bit prime
# would not: the second layer multiplies the first layer's rotation noise by full-range plaintexts)
DEEP = HEParams(n=64, p=P, rns_limbs=3, noise_budget=1e30)


def _dec(outs, task):
    return np.concatenate([unpack_channels(decrypt(o), task) for o in outs])


def test_drop_in_convolutions_chain():
    rng = np.random.default_rng(12)
    u = 4                                                 # c_n = 4
    k1 = rng.integers(-128, 128, (4, 4, 3, 3)) % P        # c_n -> c_n
    k2 = rng.integers(-128, 128, (8, 4, 3, 3)) % P        # c_n -> 2 c_n (two output blocks)
    k3 = rng.integers(-128, 128, (4, 8, 1, 1)) % P        # 2 c_n -> c_n (two input blocks)
    t1 = ConvTask(u, u, 4, 3, 3, 4, k1, DEEP)
    t2 = ConvTask(u, u, 4, 3, 3, 8, k2, DEEP)
    t3 = ConvTask(u, u, 8, 1, 1, 4, k3, DEEP)
    x = rng.integers(0, P, (4, u, u))
    meter = CostMeter()
    o1 = mimo_kernel_grouping(t1, encrypt_inputs(t1, x), meter)
    o2 = mimo_kernel_grouping(t2, o1, meter)
    assert len(o2) == 2 and all(o.replicated for o in o2)
    o3 = mimo_kernel_grouping(t3, o2, meter)
    y1 = conv2d_mod_p(x, k1, P)
    y2 = conv2d_mod_p(y1, k2, P)
    assert np.array_equal(_dec(o1, t1), y1)
    assert np.array_equal(_dec(o2, t2), y2)
    assert np.array_equal(_dec(o3, t3), conv2d_mod_p(y2, k3, P))
    s = he_add(o2[0], o2[1], meter)                        # blocks of one layer combine like the reference's
    assert np.array_equal(unpack_channels(decrypt(s), t2), (y2[:4] + y2[4:]) % P)


def test_row_paired_outputs_are_used_correctly_or_rejected():
    rng = np.random.default_rng(13)
    u = 4
    k1 = rng.integers(-128, 128, (8, 4, 3, 3)) % P        # paired layer: blocks 0 / 1 in rows 0 / 1
    t1 = ConvTask(u, u, 4, 3, 3, 8, k1, DEEP)
    x = rng.integers(0, P, (4, u, u))
    paired = KernelGroupingConv(t1)                       # pair_rows=True
    o = paired(encrypt_inputs(t1, x), CostMeter())
    assert [(c.row, c.replicated) for c in o] == [(0, False), (1, False)]
    y1 = conv2d_mod_p(x, k1, P)
    assert np.array_equal(_dec(o, t1), y1)
    # a single-row layer runs on either row's vector and answers in that row
    k2 = rng.integers(-128, 128, (4, 4, 3, 3)) % P
    t2 = ConvTask(u, u, 4, 3, 3, 4, k2, DEEP)
    single = KernelGroupingConv(t2, pair_rows=False)
    for blk in (0, 1):
        out = single([o[blk]], CostMeter())
        assert out[0].row == blk and not out[0].replicated
        assert np.array_equal(_dec(out, t2), conv2d_mod_p(y1[4 * blk:4 * blk + 4], k2, P))
    # rows that cannot be combined are rejected
    t3 = ConvTask(u, u, 8, 1, 1, 4, rng.integers(0, P, (4, 8, 1, 1)), DEEP)
    with pytest.raises(DimensionError):
        KernelGroupingConv(t3, pair_rows=False)(o, CostMeter())          # inputs in rows 0 and 1
    with pytest.raises(DimensionError):
        KernelGroupingConv(t2)([o[0]], CostMeter())                      # pairing needs replicated inputs
    with pytest.raises(DimensionError):
        he_add(o[0], o[1], CostMeter())


# --- two ranks, real CUDA sub-layers ----------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _kernels(rng, c_o, c_i, k):
    """int8 kernels everywhere except one large coefficient in the FIRST output block: the full layer
    (and rank 0's shard) must take schedule 1, while rank 1's shard alone would pick schedule 2."""
    kern = rng.integers(-128, 128, (c_o, c_i, k, k))
    kern[0, 0, 0, 0] = 5000
    return kern % P


def _shard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_01827_b200.conv import kg_schedule
        from paper_2105_01827_b200.sharding import ShardedKernelGroupingConv, sub_conv_task

        params = HEParams(n=1024, p=P, rns_limbs=3, seed=77)    # same seed: same secret and keys on both ranks
        rng = np.random.default_rng(5)
        u, c_i, c_o, k = 32, 8, 24, 3                            # c_n = 1: 8 inputs, 24 blocks -> 12 physical
        kern = _kernels(rng, c_o, c_i, k)
        task = ConvTask(u, u, c_i, k, k, c_o, kern, params)
        x = rng.integers(0, P, (c_i, u, u))
        layer = ShardedKernelGroupingConv(task)
        shard_sched = kg_schedule(sub_conv_task(task, layer.shards[1], 2), 1, 3)
        cts = encrypt_inputs(task, x)
        stacked = torch.stack([c.data for c in cts])
        if rank != 0:
            stacked = torch.zeros_like(stacked)                  # only the source rank holds the inputs
        out = layer.forward_device(stacked)
        res = {"sizes": layer.sizes, "schedule": layer.schedule, "local_schedule": layer.local.schedule,
               "shard_alone": shard_sched}
        if rank == 0:
            full = KernelGroupingConv(task)
            want = full.forward_device(torch.stack([c.data for c in cts]))
            ctx = full.ctx
            res["words_equal"] = bool(np.array_equal(ctx.export_words(out), ctx.export_words(want)))
            n = params.n
            got = np.concatenate([ctx.decrypt_physical(out[ob // 2])[(ob % 2) * n:(ob % 2 + 1) * n].reshape(1, u, u)
                                  for ob in range(c_o)])
            res["dec_ok"] = bool(np.array_equal(got, conv2d_mod_p(x, kern, P)))
        else:
            res["none_off_dst"] = out is None
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sharded_conv_two_ranks_cuda():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    r0, r1 = outs[0], outs[1]
    assert r0["sizes"] == [6, 6]
    assert r1["shard_alone"] == 2                    # the shard alone would have taken schedule 2 ...
    assert r0["schedule"] == r1["schedule"] == 1     # ... the plan of the full layer is imposed on both
    assert r0["local_schedule"] == r1["local_schedule"] == 1
    assert r0["words_equal"] and r0["dec_ok"]
    assert r1["none_off_dst"]


# --- one FC layer split across ranks by its giant groups ----------------------------------------
def _fc_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.plain import dot_mod_p
        from paper_2105_01827_b200.sharding import ShardedGalaFC

        params = HEParams(n=1024, p=P, rns_limbs=3, seed=78)     # same seed: same secret and keys everywhere
        rng = np.random.default_rng(8)
        w = rng.integers(-128, 128, (256, 1024)) % P
        sharded = ShardedGalaFC(w, params)
        lay, ctx = sharded.layer, sharded.ctx
        B = 3
        xs = [rng.integers(0, P, 1024) for _ in range(B)]
        masks = [lay.draw_masks(40 + b) for b in range(B)]
        cts = torch.stack([lay.encrypt_input(x)[0] for x in xs])
        d_r = ctx.to_device_u32(np.stack([ctx.physical(m[0][0].slots, m[0][1].slots) for m in masks]))
        if rank != 0:
            cts = torch.zeros_like(cts)                             # only the source rank holds the inputs
        res = sharded.forward_device(cts, d_r)
        out = {"groups": (sharded.groups.start, sharded.groups.stop), "G": sharded.G}
        if rank == 0:
            _, masked = res
            _, want = lay.run_batch(cts, lay.blocks[0][1], d_r, block=0)     # the single-GPU layer
            out["words_equal"] = bool(np.array_equal(ctx.export_words(masked), ctx.export_words(want)))
            out["dec_ok"] = all(bool(np.array_equal((lay.client_shares([masked[b]]) + lay.server_shares(masks[b])) % P,
                                                    dot_mod_p(w, xs[b], P))) for b in range(B))
        else:
            out["none_off_dst"] = res is None
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fc_giant_group_split_cuda(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fc_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    outs = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    G = outs[0]["G"]
    spans = sorted(outs[r]["groups"] for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == G and all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert outs[0]["words_equal"] and outs[0]["dec_ok"]
    assert all(outs[r]["none_off_dst"] for r in range(1, world))
