#!/usr/bin/env python
"""Config 5 (BASELINE.json configs[4]): all ResNet-18 linear layers at 224x224x3, N=8192, L=3.

Encodes every layer's weights into HBM once, then for each layer: encrypts a
fresh random input (frames/tiles), times the fused layer on the device (CUDA
events, weights and inputs resident), decrypts and checks the result against
the plaintext truth (stride-1 conv then subsample / W x).  Prints one JSON line
per layer and a summary line (whole-network linear latency = sum of layers).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2105_01827_b200.resnet import ResNet18Linear, layer_costs, resnet18_224  # noqa: E402
from paper_2105_01827_b200.sharding import gather_objects, max_over_ranks, partition_layers  # noqa: E402
from plain_check import conv2d_mod_p, dot_mod_p  # noqa: E402


def plain_layer(spec, x, w, p):
    if spec.kind == "fc":
        return dot_mod_p(w, x, p)
    return conv2d_mod_p(x, w, p, spec.stride)


def _measured_costs():
    path = os.path.join(ROOT, "profiles", "r1_resnet18_224.jsonl")
    out = {}
    if os.path.exists(path):
        for line in open(path):
            d = json.loads(line)
            if "layer" in d:
                out[d["layer"]] = d["ms"]
    return out


def main():
    """One process per GPU under torchrun: the layers are partitioned across ranks (LPT on the
    measured per-layer times, `sharding.partition_layers`); each rank holds and runs its own
    layers.  The pipelined network period is the max over ranks of the per-rank sums."""
    check = "--no-check" not in sys.argv
    blocks = "--shard-blocks" in sys.argv     # latency form: every conv's output blocks split across ranks
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    specs = resnet18_224()
    if "--net" in sys.argv:       # layers from a network file (reference layer-list format)
        from paper_2105_01827_b200.netfile import load_network, network_layers

        names = [sp.name for sp in specs]
        specs = network_layers(load_network(sys.argv[sys.argv.index("--net") + 1]), names=names)
    if blocks:   # every rank holds a slice of every conv; the FC runs on rank 0
        parts = [list(range(len(specs)))] + [[i for i, sp in enumerate(specs) if sp.kind == "conv"]] * (world - 1)
    else:
        parts = partition_layers(layer_costs(specs, _measured_costs()), world)
    mine = parts[rank]
    t0 = time.perf_counter()
    net = ResNet18Linear(only=mine, shard_blocks=blocks and world > 1, layers=specs)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    ctx = net.ctx
    rng = np.random.default_rng(7)
    total_ms, ok_all = 0.0, True
    for i, (spec, layer) in enumerate(zip(net.specs, net.layers)):
        x = net.random_input(i, rng)        # drawn on every rank: the same inputs as one GPU
        if layer is None:
            continue
        if spec.kind == "fc":
            cts = layer.encrypt_frames(x)
            masks = layer.layer.draw_masks(11 + i)
            run = lambda: layer.forward_device(cts, masks)  # noqa: E731
        else:
            enc = layer.encrypt_frames(x)
            run = lambda: layer.forward_device(enc)  # noqa: E731
        out = run()
        torch.cuda.synchronize()
        reps = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = run()
            b.record()
            torch.cuda.synchronize()
            reps.append(a.elapsed_time(b))
        ms = float(np.median(reps))
        breakdown = None
        if "--profile" in sys.argv:   # one extra traced run: per-kernel CUDA-event times of this layer
            ctx.profile(True)
            out = run()
            prof = ctx.profile_read()
            ctx.profile(False)
            breakdown = {k: round(v["ms"], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}
        if blocks and world > 1 and spec.kind == "conv":   # every rank ran a slice of this layer
            ms = max_over_ranks(ms, device=torch.device("cuda"))
        total_ms += ms
        res = {"layer": spec.name, "shape": [spec.c_in, spec.c_out, spec.k, spec.stride, spec.size], "ms": round(ms, 3),
               "ms_reps": [round(v, 3) for v in reps],
               "plaintext_GB": round(layer.plaintext_bytes / 1e9, 3)}
        if spec.kind == "conv":
            res.update(frame=layer.frame, c_n=layer.kg.c_n, tiles=layer.tiles ** 2, schedule=layer.kg.schedule)
        if breakdown is not None:
            res["breakdown_ms"] = breakdown
        if check and (not blocks or rank == 0):   # sharded outputs are gathered on rank 0
            got = layer.shares(out, masks) if spec.kind == "fc" else layer.decrypt_output(out)
            ok = bool(np.array_equal(got, plain_layer(spec, x, net.weights[i], net.params.p)))
            res["correct"] = ok
            ok_all &= ok
        res["rank"] = rank
        print(json.dumps(res), flush=True)
    period = max_over_ranks(total_ms, device=torch.device("cuda"))
    sums = gather_objects((total_ms, ok_all))
    if rank == 0 and blocks:
        print(json.dumps({"summary": "resnet18_224_linear_latency", "layers": len(net.specs), "n_gpus": world,
                          "mode": "every conv's output ciphertexts sharded across ranks (inputs broadcast, "
                                  "outputs gathered on rank 0); per-layer time = max over ranks",
                          "latency_ms": round(total_ms, 2), "all_correct": ok_all if check else None,
                          "N": ctx.N, "L": ctx.L}), flush=True)
    elif rank == 0:
        print(json.dumps({"summary": "resnet18_224_linear", "layers": len(net.specs), "n_gpus": world,
                          "partition": parts, "per_rank_ms": [round(t, 2) for t, _ in sums],
                          "total_ms": round(sum(t for t, _ in sums), 2),
                          "pipelined_period_ms": round(period, 2),
                          "networks_per_s": round(1e3 / period, 3),
                          "all_correct": all(o for _, o in sums) if check else None,
                          "plaintext_GB_rank0": round(net.plaintext_bytes / 1e9, 2), "weight_setup_s": round(setup, 1),
                          "N": ctx.N, "L": ctx.L, "key_MB": round(ctx.key_bytes() / 1e6, 1)}), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
