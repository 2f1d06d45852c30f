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
