"""Multi-GPU partitioning of independent GALA ciphertext work.

The GALA linear layers have no cross-ciphertext exchange inside a layer's output
blocks: each output ciphertext of a kernel-grouping convolution depends only on
the (shared) input ciphertexts and its own block of kernels (`conv.py:268-293`),
and independent layers / inputs share nothing at all.  So work is partitioned
across ranks, one process per GPU:

* **inputs / layers** (configs 1, 2, 5): replicas, or a cost-balanced assignment
  of whole layers to ranks (`partition_layers`); no data-path collective;
* **giant groups of one FC layer** (config 2; `ShardedGalaFC`): every rank takes a range of the
  BSGS giant groups, and the QP partial sums before the final ModDown meet in one exact modular
  reduce (an element-wise u64 sum: every word < q_j < 2^60 and at most 8 ranks) on the root, which
  finishes the layer -- the same words as one GPU;
* **output blocks of one convolution** (configs 3, 4, 5): `ShardedKernelGroupingConv`
  broadcasts the input ciphertexts from the source rank, every rank runs the fused
  layer on its contiguous range of physical output ciphertexts, and only the final
  output ciphertexts are gathered to the destination rank (NCCL over NVLink on
  GPUs, gloo on CPU).  The words of every output block equal the single-GPU
  layer's words for that block: the sub-layer is the same computation restricted
  to its kernels (`tests/test_multiprocess.py`).

The control-plane collectives are the max-over-ranks of the timed region and small
per-rank result objects.
"""
from __future__ import annotations

import heapq

import numpy as np


def shard_range(n_items: int, world: int, rank: int) -> range:
    """Contiguous, balanced block of item indices owned by `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def partition_layers(costs, world: int) -> list[list[int]]:
    """Longest-processing-time assignment of independent layers to `world` ranks.

    Returns, per rank, the layer indices in ascending order.  Deterministic (ties by
    index), so every rank computes the same assignment without communicating.
    """
    if world <= 0:
        raise ValueError("bad world")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(v) for v in out]


def _dist():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist
    return None


def world_rank(group=None) -> tuple[int, int]:
    dist = _dist()
    if dist is None:
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def max_over_ranks(value: float, device=None) -> float:
    """Maximum of a per-rank scalar (elapsed time) across the process group."""
    import torch

    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_objects(obj):
    """All ranks' small result objects (e.g. output shares) on every rank."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def _host_staged(dist, t, group=None) -> bool:
    """gloo moves host tensors only: CUDA tensors go through host memory (CPU tests of the
    multi-rank path with real CUDA layers); NCCL moves them over NVLink directly."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def broadcast_tensor(t, src: int = 0, group=None):
    """In-place broadcast of `t` from `src` (host-staged under gloo)."""
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return t
    if _host_staged(dist, t, group):
        h = t.cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)
    return t


def gather_blocks(local, sizes, dst: int = 0, group=None):
    """Gather per-rank ciphertext blocks [n_r][...] to `dst` -> [sum n_r][...] (None elsewhere).

    Blocks are padded to the largest shard so one fixed-size `gather` moves them; only
    `dst` receives data (the final result ciphertexts).
    """
    import torch

    dist = _dist()
    world, rank = world_rank(group)
    if dist is None or world == 1:
        return local
    m = max(sizes)
    if local.shape[0] < m:
        pad = torch.zeros((m - local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        local = torch.cat([local, pad])
    dev = local.device
    if _host_staged(dist, local, group):
        local = local.cpu()
    bufs = [torch.empty_like(local) for _ in range(world)] if rank == dst else None
    dist.gather(local.contiguous(), bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([b[:n] for b, n in zip(bufs, sizes)]).to(dev)


def sub_conv_task(task, obp: range, pair: int):
    """The ConvTask of physical output ciphertexts `obp` (output channels of blocks
    pair*obp.start .. pair*obp.stop, each block c_n channels)."""
    from .conv import ConvTask

    c_n = task.channels_per_ct
    lo = obp.start * pair * c_n
    hi = min(task.c_o, obp.stop * pair * c_n)
    return ConvTask(task.u_w, task.u_h, task.c_i, task.k_w, task.k_h, hi - lo, np.asarray(task.kernels)[lo:hi],
                    task.params)


class ShardedKernelGroupingConv:
    """`KernelGroupingConv` with its physical output ciphertexts partitioned across ranks.

    Every rank holds the encoded weights of its own output blocks only (HBM per GPU
    falls with the world size).  `forward_device` takes the physical inputs on the
    source rank (any tensor of the right shape elsewhere), broadcasts them, runs the
    local fused layer and gathers the outputs on `dst`.  ``layer_factory(sub_task)``
    builds the per-rank layer (default `KernelGroupingConv(sub_task, **kw)`).
    """

    def __init__(self, task, group=None, layer_factory=None, pair_rows: bool = True, **kw):
        self.task, self.group = task, group
        self.world, self.rank = world_rank(group)
        c_n = task.channels_per_ct
        self.pair = 2 if pair_rows else 1
        n_ob = task.c_o // c_n
        self.n_obp = (n_ob + self.pair - 1) // self.pair
        self.shards = [shard_range(self.n_obp, self.world, r) for r in range(self.world)]
        self.sizes = [len(s) for s in self.shards]
        mine = self.shards[self.rank]
        self.sub_task = sub_conv_task(task, mine, self.pair) if len(mine) else None
        # the schedule, mask form and first-Add engine are decided once from the FULL task and imposed
        # on every shard: a decision taken per shard (its kernels' int8 range, its row count, its
        # plaintext bytes) could differ between ranks, so the gathered words would not be the
        # single-GPU layer's and the ranks could reach the collectives with different shapes
        self.plan = kw.pop("plan", None)
        if layer_factory is None:
            from .backend import context
            from .conv import KernelGroupingConv, kg_plan

            if self.plan is None:
                ctx = context(task.params)
                plan_kw = {k: kw[k] for k in ("band_only", "tensor_cores", "host_encode", "schedule") if k in kw}
                self.plan = kg_plan(task, self.pair, ctx.L, ctx.N, **plan_kw)

            def layer_factory(t):
                return KernelGroupingConv(t, pair_rows=pair_rows, plan=self.plan, **kw)
        self.local = layer_factory(self.sub_task) if self.sub_task is not None else None
        # the layer geometry callers read (ConvLayer.decrypt_output)
        self.c_n, self.n_ob = c_n, n_ob
        self.schedule = self.plan.schedule if self.plan is not None else getattr(self.local, "schedule", None)

    @property
    def ctx(self):
        from .backend import context

        return context(self.task.params)

    @property
    def batchable(self) -> bool:
        """The full layer's batched form (rank-independent: every rank takes the same branch; a
        shard without the fused batched form runs its images one by one inside
        forward_device_batch)."""
        if self.plan is not None:
            return bool(self.plan.batchable)
        return bool(getattr(self.local, "batchable", True))

    def forward_device_batch(self, cts_batch, src: int = 0, dst: int = 0):
        """[B][n_ib][2][L][N] images on `src` -> [B][n_obp][2][L][N] on `dst` (None elsewhere)."""
        import torch

        if self.world > 1:
            cts_batch = broadcast_tensor(cts_batch.contiguous(), src=src, group=self.group)
        nb = cts_batch.shape[0]
        if self.local is not None:
            local = self.local.forward_device_batch(cts_batch)
        else:
            local = torch.empty((nb, 0) + tuple(cts_batch.shape[2:]), dtype=cts_batch.dtype, device=cts_batch.device)
        out = gather_blocks(local.transpose(0, 1).contiguous(), self.sizes, dst=dst, group=self.group)
        return None if out is None else out.transpose(0, 1).contiguous()

    def forward_device(self, cts_phys, src: int = 0, dst: int = 0):
        """[n_ib][2][L][N] on `src` -> [n_obp][2][L][N] on `dst` (None on the other ranks)."""
        import torch

        if self.world > 1:
            cts_phys = broadcast_tensor(cts_phys.contiguous(), src=src, group=self.group)
        if self.local is not None:
            local = self.local.forward_device(cts_phys)
        else:
            local = torch.empty((0,) + tuple(cts_phys.shape[1:]), dtype=cts_phys.dtype, device=cts_phys.device)
        return gather_blocks(local, self.sizes, dst=dst, group=self.group)

    def __call__(self, cts, meter, src: int = 0, dst: int = 0):
        """Drop-in form of `mimo_kernel_grouping` (conv.py:268-293): logical ciphertexts in
        on `src`, logical outputs on `dst` (None elsewhere); `dst` books the layer's counts."""
        import torch

        from .backend import Ciphertext
        from .conv import _check_mimo, _kg_book_and_noise
        from .errors import DimensionError

        c_n, n_ib, n_ob = _check_mimo(self.task, cts)
        if self.pair == 2 and not all(c.replicated for c in cts):
            raise DimensionError("row-paired kernel grouping expects replicated input ciphertexts")
        rows = {c.row for c in cts if not c.replicated}
        if len(rows) > 1:
            raise DimensionError("input ciphertexts hold their vectors in different hypercube rows")
        stacked = torch.stack([c.data for c in cts])
        outs = self.forward_device(stacked, src=src, dst=dst)
        if outs is None:
            return None
        noises = _kg_book_and_noise(self.task, [c.noise for c in cts], c_n, n_ib, n_ob, meter)
        if self.pair == 2:
            return [Ciphertext._wrap(outs[ob // 2], noises[ob], self.task.params, ob % 2) for ob in range(n_ob)]
        rep = not rows
        row = rows.pop() if rows else 0
        return [Ciphertext._wrap(outs[ob], noises[ob], self.task.params, row, replicated=rep) for ob in range(n_ob)]


def reduce_sum_u64(t, dst: int = 0, group=None):
    """Element-wise u64 sum of `t` over the ranks onto `dst` (in place there; int64 two's-complement
    addition is u64 addition).  The caller keeps every word < 2^64 / world (here < q_j < 2^60, at most
    8 ranks), so the sum is exact and one mod-q_j reduction after it gives the modular sum."""
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return t
    if _host_staged(dist, t, group):
        h = t.cpu()
        dist.reduce(h, dst=dst, op=dist.ReduceOp.SUM, group=group)
        if dist.get_rank(group) == dst:
            t.copy_(h)
    else:
        dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardedGalaFC:
    """One schedule-2 GALA FC layer (`matvec.GalaFC`) split across ranks by its giant groups
    (SURVEY.md 8(e), config 2).  Every rank holds the layer's weights and receives the inputs; rank r
    runs the baby-step sums and the giant-step key switches of its group range (`shard_range` over the
    G = T / b groups) and returns the QP sums before the final ModDown; `reduce_sum_u64` meets them on
    `dst`, which reduces mod q_j, applies the one final ModDown and the mask (gala_mv_gala2_finish).
    ModDown is linear only up to rounding, so it is applied once, to the total: the words equal the
    single-GPU layer's."""

    def __init__(self, w, params, group=None, tensor_cores: bool = True, **kw):
        from .matvec import GalaFC

        self.layer = GalaFC(w, params, tensor_cores=tensor_cores, **kw)
        if self.layer.schedule != 2:
            raise ValueError("the giant-group split needs the schedule-2 layer")
        self.group = group
        self.world, self.rank = world_rank(group)
        self.G = self.layer.T // self.layer.baby
        if self.world > self.G:
            raise ValueError(f"{self.world} ranks for {self.G} giant groups")
        self.groups = shard_range(self.G, self.world, self.rank)

    @property
    def ctx(self):
        return self.layer.ctx

    def forward_device(self, cts, d_r, block: int = 0, src: int = 0, dst: int = 0):
        """cts [B][2][L][N] and masks d_r [B][N] on `src` -> (outs, masked) on `dst`, None elsewhere."""
        if self.world > 1:
            cts = broadcast_tensor(cts.contiguous(), src=src, group=self.group)
        lay = self.layer
        tasks, pts2, T = lay.blocks[block]
        qp, qa = lay.ctx.mv_gala2_partial(cts, pts2, T, lay.baby, self.groups.start, self.groups.stop,
                                          wcan=lay.wcan[block])
        reduce_sum_u64(qp, dst=dst, group=self.group)
        reduce_sum_u64(qa, dst=dst, group=self.group)
        if self.rank != dst:
            return None
        return lay.ctx.mv_gala2_finish(qp, qa, d_r)
