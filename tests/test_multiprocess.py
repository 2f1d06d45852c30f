"""World-size-2 gloo test of the multi-GPU host logic (CPU only)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_01827_b200.sharding import gather_objects, max_over_ranks, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 8, 1023):
        for world in (1, 2, 3, 8):
            got = [list(shard_range(n, world, r)) for r in range(world)]
            assert sum(got, []) == list(range(n))
            assert max(map(len, got)) - min(map(len, got)) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_01827_b200.matvec import MvTask
        from paper_2105_01827_b200.backend import HEParams
        from oracle.plain import dot_mod_p

        p = 1032193
        items = list(shard_range(10, world, rank))
        # each rank "serves" its own independent layer invocations (host-side layout work)
        rng = np.random.default_rng(0)
        w = rng.integers(0, p, (16, 128))
        res = {}
        for i in items:
            x = np.random.default_rng(100 + i).integers(0, p, 128)
            task = MvTask(128, 16, w, HEParams(n=2048))
            res[i] = (task.groups, dot_mod_p(w, x, p).tolist())
        t = max_over_ranks(float(rank + 1))
        allres = gather_objects(res)
        q.put((rank, t, allres))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_replicas():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, t, allres in outs:
        assert t == 2.0                      # max over ranks
        merged = {}
        for d in allres:
            assert not set(d) & set(merged)  # disjoint shards
            merged.update(d)
        assert sorted(merged) == list(range(10))


def test_partition_layers_balanced():
    from paper_2105_01827_b200.sharding import partition_layers

    costs = [5.0, 3.0, 3.0, 2.0, 2.0, 2.0, 1.0]
    for world in (1, 2, 3, 8):
        parts = partition_layers(costs, world)
        assert sorted(sum(parts, [])) == list(range(len(costs)))
        loads = [sum(costs[i] for i in p) for p in parts]
        # LPT bound: max load <= optimum * (4/3 - 1/(3 world)); optimum >= max(mean, max item)
        opt = max(sum(costs) / world, max(costs))
        assert max(loads) <= opt * (4 / 3) + 1e-9
    assert partition_layers(costs, 2) == partition_layers(costs, 2)   # every rank derives the same split


class _OracleKG:
    """CPU stand-in for one rank's fused KG layer: the oracle's o_conv_kg on the sub-task's
    physical-form plaintexts (the same construction as KernelGroupingConv._encode_on_host)."""

    def __init__(self, task, cpu):
        from paper_2105_01827_b200.conv import DiagonalPlan

        self.task, self.cpu = task, cpu
        c_n = task.channels_per_ct
        n = task.params.n
        n_ib, n_ob = task.c_i // c_n, task.c_o // c_n
        n_obp = (n_ob + 1) // 2
        plan = DiagonalPlan(task, c_n)
        k = len(task.offsets())
        zeros = np.zeros((c_n, k, n), dtype=np.int64)
        pts = np.zeros((n_obp, n_ib, c_n, k, 2 * n), dtype=np.uint32)
        for obp in range(n_obp):
            for ib in range(n_ib):
                rows = [np.stack([plan.coef_slots(ob, ib, d) for d in range(c_n)]) if ob < n_ob else zeros
                        for ob in (2 * obp, 2 * obp + 1)]
                pts[obp, ib] = np.concatenate(rows, axis=2)
        self.pts = pts
        self.taps = [rot for _, _, rot in task.offsets()]

    def forward_device(self, cts):
        import torch

        out = self.cpu.conv_kg(cts.numpy().view(np.uint64), self.pts, self.taps, self.task.image_slots)
        return torch.from_numpy(out.view(np.int64))

    batchable = True

    def forward_device_batch(self, cts_batch):
        import torch

        return torch.stack([self.forward_device(c) for c in cts_batch])


def _sharded_conv_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        from oracle.bfv import Oracle
        from oracle.plain import conv2d_mod_p
        from paper_2105_01827_b200 import sampling
        from paper_2105_01827_b200.backend import HEParams
        from paper_2105_01827_b200.conv import ConvTask, encode_channel_blocks, unpack_channels
        from paper_2105_01827_b200.ring import SlotVector
        from paper_2105_01827_b200.sharding import ShardedKernelGroupingConv

        p = 1032193
        params = HEParams(n=64, p=p, seed=3)
        bfv = params.bfv()
        rng = np.random.default_rng(7)            # same stream on every rank: same secret and keys
        s = sampling.secret(rng, bfv.N)
        cpu = Oracle(bfv)
        cpu.set_secret(s)
        c_i, c_o, u = 8, 24, 4                    # c_n = 4: 2 input cts, 6 output blocks -> 3 physical
        kern = rng.integers(-128, 128, (c_o, c_i, 3, 3)) % p
        task = ConvTask(u, u, c_i, 3, 3, c_o, kern, params)
        c_n = task.channels_per_ct
        steps = [rot for _, _, rot in task.offsets()] + [d * task.image_slots for d in range(1, c_n)]
        for st in sorted({st % params.n for st in steps} - {0}):
            a, e = sampling.rotation_key_randomness(rng, bfv)
            cpu.gen_rotkey(st, a, e)
        img = rng.integers(0, p, (c_i, u, u))
        cts = []
        for b in encode_channel_blocks(task, img):
            a, e = sampling.encryption_randomness(rng, bfv)
            phys = np.concatenate([b.slots, b.slots]).astype(np.uint32)
            cts.append(cpu.encrypt(phys, a, e))
        x = torch.from_numpy(np.stack(cts).view(np.int64))
        if rank != 0:
            x = torch.zeros_like(x)               # only the source rank holds the inputs
        layer = ShardedKernelGroupingConv(task, layer_factory=lambda t: _OracleKG(t, cpu))
        out = layer.forward_device(x)
        res = None
        if rank == 0:
            full = _OracleKG(task, cpu).forward_device(torch.from_numpy(np.stack(cts).view(np.int64)))
            words_equal = bool(torch.equal(out, full))
            got = []
            for ob in range(c_o // c_n):
                phys = cpu.decrypt(out[ob // 2].numpy().view(np.uint64))
                row = ob % 2
                got.append(unpack_channels(SlotVector(phys[row * 64:(row + 1) * 64].astype(np.int64), p), task))
            dec_ok = bool(np.array_equal(np.concatenate(got), conv2d_mod_p(img, kern, p)))
            res = (words_equal, dec_ok, layer.sizes)
        else:
            assert out is None
            res = (None, None, layer.sizes)
        # the batched form (halo tiles / images sharing the weights): gather along the output blocks
        xb = torch.stack([x, torch.flip(x, dims=[0])]) if rank == 0 else torch.zeros((2,) + tuple(x.shape), dtype=x.dtype)
        outb = layer.forward_device_batch(xb)
        if rank == 0:
            full = _OracleKG(task, cpu)
            ok_b = all(bool(torch.equal(outb[b], full.forward_device(xb[b]))) for b in range(2))
            res = res + (ok_b,)
        else:
            assert outb is None
            res = res + (None,)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_conv_output_blocks():
    """Output-block sharding of a KG convolution: broadcast inputs, per-rank sub-layers, gather of
    the output ciphertexts on rank 0 == the single-rank layer, word for word (uneven shards 2 + 1)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_conv_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    words_equal, dec_ok, sizes, batch_ok = outs[0]
    assert sizes == [2, 1]
    assert words_equal
    assert dec_ok
    assert batch_ok
