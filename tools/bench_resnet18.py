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

from paper_2105_01827_b200.resnet import ResNet18Linear  # noqa: E402
from plain_check import conv2d_mod_p, dot_mod_p  # noqa: E402


def plain_layer(spec, x, w, p):
    if spec.kind == "fc":
        return dot_mod_p(w, x, p)
    return conv2d_mod_p(x, w, p, spec.stride)


def main():
    check = "--no-check" not in sys.argv
    t0 = time.perf_counter()
    net = ResNet18Linear()
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    ctx = net.ctx
    rng = np.random.default_rng(7)
    total_ms, ok_all = 0.0, True
    for i, (spec, layer) in enumerate(zip(net.specs, net.layers)):
        x = net.random_input(i, rng)
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
        total_ms += ms
        res = {"layer": spec.name, "shape": [spec.c_in, spec.c_out, spec.k, spec.stride, spec.size], "ms": round(ms, 3),
               "ms_reps": [round(v, 3) for v in reps],
               "plaintext_GB": round(layer.plaintext_bytes / 1e9, 3)}
        if spec.kind == "conv":
            res.update(frame=layer.frame, c_n=layer.kg.c_n, tiles=layer.tiles ** 2, schedule=layer.kg.schedule)
        if check:
            got = layer.shares(out, masks) if spec.kind == "fc" else layer.decrypt_output(out)
            ok = bool(np.array_equal(got, plain_layer(spec, x, net.weights[i], net.params.p)))
            res["correct"] = ok
            ok_all &= ok
        print(json.dumps(res), flush=True)
    print(json.dumps({"summary": "resnet18_224_linear", "layers": len(net.specs), "total_ms": round(total_ms, 2),
                      "networks_per_s": round(1e3 / total_ms, 3), "all_correct": ok_all if check else None,
                      "plaintext_GB": round(net.plaintext_bytes / 1e9, 2), "weight_setup_s": round(setup, 1),
                      "N": ctx.N, "L": ctx.L, "key_MB": round(ctx.key_bytes() / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
