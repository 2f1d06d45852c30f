#!/usr/bin/env python
"""Config 4 with its output ciphertexts sharded across GPUs, one process per GPU:

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        tools/bench_sharded_conv.py

Rank 0 encrypts the 64 input ciphertexts of a 56x56x64 -> 64 3x3 convolution (N = 8192, L = 3,
64x64 frames); each step broadcasts them (NCCL), every rank runs the fused kernel-grouping layer
on its range of the 32 physical output ciphertexts, and the outputs are gathered on rank 0.  The
step time is CUDA-event timed per rank and reported as the max over ranks; rank 0 decrypts the
gathered outputs and checks them against conv2d mod p.  Prints one JSON line.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from plain_check import conv2d_mod_p  # noqa: E402
from paper_2105_01827_b200 import ConvTask, HEParams  # noqa: E402
from paper_2105_01827_b200.conv import encrypt_inputs, unpack_channels  # noqa: E402
from paper_2105_01827_b200.sharding import ShardedKernelGroupingConv, gather_objects, max_over_ranks  # noqa: E402

P = 1032193


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    u, frame, c, k = 56, 64, 64, 3
    params = HEParams(n=4096, rns_limbs=3, seed=32)
    rng = np.random.default_rng(2)
    kern = rng.integers(-128, 128, (c, c, k, k)) % P
    ch = rng.integers(0, P, (c, u, u))
    img = np.zeros((c, frame, frame), dtype=np.int64)
    img[:, :u, :u] = ch
    task = ConvTask(frame, frame, c, k, k, c, kern, params)
    layer = ShardedKernelGroupingConv(task, band_only=True)
    if rank == 0:
        x = torch.stack([ct.data for ct in encrypt_inputs(task, img)])
    else:
        from paper_2105_01827_b200.backend import context

        ctx = context(params)
        x = torch.empty((c // task.channels_per_ct, 2, ctx.L, ctx.N), dtype=torch.int64, device=ctx.device)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    out = layer.forward_device(x)
    torch.cuda.synchronize()
    reps = []
    for _ in range(5):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = layer.forward_device(x)
        b.record()
        torch.cuda.synchronize()
        reps.append(a.elapsed_time(b))
    ms = max_over_ranks(float(np.median(reps)), device=torch.device("cuda"))
    local = gather_objects(layer.sizes[rank])
    if rank == 0:
        ctx = layer.local.ctx
        n = params.n
        got = []
        for ob in range(c // task.channels_per_ct):
            phys = ctx.decrypt_physical(out[ob // 2])
            got.append(phys[(ob % 2) * n:(ob % 2 + 1) * n].reshape(task.channels_per_ct, frame, frame))
        ok = bool(np.array_equal(np.concatenate(got)[:, :u, :u], conv2d_mod_p(ch, kern, P)))
        print(json.dumps({"workload": "cfg4 conv 56x56x64->64 3x3 (64x64 frames), output ciphertexts sharded",
                          "n_gpus": world, "physical_outputs_per_rank": local, "ms_per_layer": round(ms, 4),
                          "layers_per_s": round(1e3 / ms, 1), "correct": ok,
                          "timing": "CUDA events per rank incl. input broadcast and output gather, max over ranks, "
                                    "L2 flushed before each step"}), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
