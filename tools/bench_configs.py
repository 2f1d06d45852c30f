#!/usr/bin/env python
"""Side benchmark of every BASELINE config's fused layer on one GPU (not the driver's bench line).

cfg1: GALA FC 16x2048, N=4096 L=1          cfg2: GALA FC 1024x4096, N=8192 L=3
cfg3: KG conv 16x16x64->64 3x3, N=4096 L=1  cfg4: KG conv 56x56x64->64 3x3 (64x64 frame), N=8192 L=3
Prints one JSON object per config: ms per layer (CUDA events, L2 flushed between reps), layers/s,
kernel breakdown, algorithmic modmuls, and a decrypted-result check against the plaintext truth.
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
from plain_check import conv2d_mod_p, dot_mod_p  # noqa: E402
from paper_2105_01827_b200 import ConvTask, CostMeter, GalaFC, HEParams, KernelGroupingConv  # noqa: E402
from paper_2105_01827_b200.conv import encrypt_inputs, unpack_channels  # noqa: E402
from paper_2105_01827_b200.backend import decrypt  # noqa: E402
from paper_2105_01827_b200.analytics import (  # noqa: E402
    executed_roofline,
    fc_executed_work,
    kg2_executed_work,
    survey_conv_roofline,
    survey_fc_roofline,
)

P = 1032193
dev = torch.device("cuda", 0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def fc(name, n, L, n_out, n_in, B):
    params = HEParams(n=n, rns_limbs=L, seed=31)
    rng = np.random.default_rng(1)
    w = rng.integers(-128, 128, (n_out, n_in)) % P
    layer = GalaFC(w, params)
    ctx = layer.ctx
    xs = [rng.integers(0, P, n_in) for _ in range(B)]
    cts = torch.stack([layer.encrypt_input(x)[0] for x in xs])
    masks = [layer.draw_masks(100 + b) for b in range(B)]
    d_r = ctx.to_device_u32(np.stack([ctx.physical(m[0][0].slots, m[0][1].slots if layer.paired else None)
                                      for m in masks]))
    pts = layer.blocks[0][1]
    outs, masked = ctx.empty_ct(B), ctx.empty_ct(B)
    run = lambda: layer.run_batch(cts, pts, d_r, outs=outs, masked=masked)  # noqa: E731
    ms = timeit(run)
    ctx.profile(True)
    run()
    prof = ctx.profile_read()
    ctx.profile(False)
    ok = all(np.array_equal((layer.client_shares([masked[b]]) + layer.server_shares(masks[b])) % P,
                            dot_mod_p(w, xs[b], P)) for b in range(min(B, 2)))
    return {"config": name, "N": ctx.N, "L": ctx.L, "T": layer.T, "schedule": layer.schedule, "batch": B,
            "ms_per_layer": ms / B,
            "layers_per_s": 1e3 * B / ms, "correct": ok,
            "breakdown_ms_per_layer": {k: round(v["ms"] / B, 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])},
            "roofline": roofline(survey_fc_roofline(ctx.N, ctx.L, layer.T), ms / B, ctx),
            "roofline_executed": fc_exec(layer, ctx, B, ms)}


def fc_exec(layer, ctx, B, ms):
    if layer.schedule != 2:
        return None
    T, b = layer.T, layer.baby
    if ctx.fc_key_folded():
        tc = "kf" if layer.wcan[0] is not None and B >= 16 and T >= 128 else False
    else:
        tc = layer.wcan[0] is not None and B >= 16 and (B <= 32 or (T >= 128 and (B % 32 == 0 or B % 32 >= 16)))
    w = fc_executed_work(ctx.N, ctx.L, T, b, B, tc)
    return exec_roof(w, w["bytes"], ms, ctx)


def conv_exec(layer, ctx, ms, images=1):
    """Schedule 2: analytics.kg2_executed_work; schedule 1 on the CUDA cores is the survey model itself."""
    if layer.schedule != 2:
        return None
    L, N = ctx.L, ctx.N
    w = kg2_executed_work(N, L, layer.n_ib, layer.k, layer.pair * layer.c_n, layer.n_obp * layer.c_n, layer.c_n,
                          layer.n_obp, layer.post, images)
    keys = (layer.k - 1 + layer.c_n - 1) * 2 * L * (L + 1) * N * 8
    nbytes = images * (layer.n_ib + layer.n_obp) * 2 * L * N * 8 + keys + layer.resident_bytes
    return exec_roof(w, nbytes, ms, ctx)


def conv(name, n, L, u, frame, c_i, c_o, k, B=1):
    params = HEParams(n=n, rns_limbs=L, seed=32)
    rng = np.random.default_rng(2)
    kern = rng.integers(-128, 128, (c_o, c_i, k, k)) % P
    ch = rng.integers(0, P, (c_i, u, u))
    img = np.zeros((c_i, frame, frame), dtype=np.int64)
    img[:, :u, :u] = ch
    task = ConvTask(frame, frame, c_i, k, k, c_o, kern, params)
    t0 = time.perf_counter()
    layer = KernelGroupingConv(task, schedule=SCHED, band_only=frame - u >= k // 2)
    setup = time.perf_counter() - t0
    ctx = layer.ctx
    cts = encrypt_inputs(task, img)
    model = survey_conv_roofline(ctx.N, ctx.L, layer.n_ib, layer.n_obp, layer.c_n, layer.k)
    stacked = torch.stack([c.data for c in cts])
    run = lambda: layer.forward_device(stacked)  # noqa: E731
    ms = timeit(run, reps=3)
    batch = None
    if B > 1 and layer.batchable:
        # B images sharing the weights: one pass (rotations, first-Add, second-Perm batched)
        chs = [rng.integers(0, P, (c_i, u, u)) for _ in range(B - 1)]
        imgs = [img]
        for c2 in chs:
            im2 = np.zeros_like(img)
            im2[:, :u, :u] = c2
            imgs.append(im2)
        bt = torch.stack([torch.stack([c.data for c in encrypt_inputs(task, im)]) for im in imgs])
        runb = lambda: layer.forward_device_batch(bt)  # noqa: E731
        msb = timeit(runb, reps=3)
        from paper_2105_01827_b200 import _lib
        torch.cuda.synchronize()
        l0, h0 = _lib.launch_count(), time.perf_counter()
        runb()
        host_ms = (time.perf_counter() - h0) * 1e3
        launches = _lib.launch_count() - l0
        torch.cuda.synchronize()
        ctx.profile(True)
        runb()
        profb = ctx.profile_read()
        ctx.profile(False)
        ob = runb()
        okb = True
        for bi in (0, B - 1):
            outs_b = [ob[bi][o // layer.pair] for o in range(layer.n_ob)]
            got = np.concatenate([ctx.decrypt_physical(ob[bi][o // layer.pair])[(o % layer.pair) * n:(o % layer.pair + 1) * n]
                                  .reshape(layer.c_n, frame, frame) for o in range(layer.n_ob)])[:, :u, :u]
            want = conv2d_mod_p(ch if bi == 0 else chs[bi - 1], kern, P)
            okb = okb and bool(np.array_equal(got, want))
            del outs_b
        batch = {"roofline": roofline(model, msb / B, ctx), "roofline_executed": conv_exec(layer, ctx, msb, B), "images": B, "ms_per_batch": msb, "host_enqueue_ms": round(host_ms, 3), "launches": launches, "ms_per_layer": msb / B, "layers_per_s": 1e3 * B / msb,
                 "correct": okb,
                 "breakdown_ms_per_layer": {k2: round(v["ms"] / B, 4)
                                            for k2, v in sorted(profb.items(), key=lambda kv: -kv[1]["ms"])}}
    ctx.profile(True)
    run()
    prof = ctx.profile_read()
    ctx.profile(False)
    meter = CostMeter()
    outs = layer(cts, meter)
    got = np.concatenate([unpack_channels(decrypt(o), task) for o in outs])[:, :u, :u]
    ok = bool(np.array_equal(got, conv2d_mod_p(ch, kern, P)))
    return {"config": name, "N": ctx.N, "L": ctx.L, "c_n": layer.c_n, "n_ib": layer.n_ib, "n_obp": layer.n_obp,
            "ms_per_layer": ms, "layers_per_s": 1e3 / ms, "correct": ok, "weight_encode_s": round(setup, 2),
            "schedule": layer.schedule, "post_mask": layer.post,
            "plaintext_bytes": layer.resident_bytes, "meter": repr(meter),
            "breakdown_ms": {k: round(v["ms"], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])},
            "roofline": roofline(model, ms, ctx), "roofline_executed": conv_exec(layer, ctx, ms), "batch": batch}


SCHED = int(os.environ["KG_SCHED"]) if os.environ.get("KG_SCHED") else None
HBM_PEAK = 6536.0   # GB/s, MEASURED_PEAKS.json (fallback)
try:
    HBM_PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", HBM_PEAK))
except Exception:
    pass
_PEAK_MM = []


def exec_roof(work, nbytes, ms_per_layer, ctx):
    """The schedule as executed (analytics.*_executed_work) against every roof: CUDA-core modmuls at the
    measured modmul peak, int8 MACs at the measured tcgen05 i8 rate (analytics.tensor_i8_peak_ops), bytes at HBM."""
    import torch

    from paper_2105_01827_b200.analytics import tensor_i8_peak_ops

    if not _PEAK_MM:
        _PEAK_MM.append(ctx.bench_modmul())
    bf16, mhz = 1639.9, 1965.0
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        bf16, mhz = float(pk.get("bf16_tflops", bf16)), float(pk.get("sm_max_mhz", mhz))
    except Exception:
        pass
    i8 = tensor_i8_peak_ops(torch.cuda.get_device_properties(ctx.device).multi_processor_count, mhz, bf16)
    r = executed_roofline(work, nbytes, ms_per_layer / 1e3, _PEAK_MM[0], i8, HBM_PEAK * 1e9)
    return {"bound": r["bound"], "frac": r["frac"], "roofline_us": r["roofline_us"], "modmuls": r["modmuls"],
            "int8_macs": r["int8_macs"], "bytes": r["bytes"]}


def roofline(model, ms_per_layer, ctx):
    """roofline time = max(modmuls / measured modmul peak, bytes / HBM peak), with the
    survey's per-operation counts (the reference's schedule: one key switch per rotation)."""
    if not _PEAK_MM:
        _PEAK_MM.append(ctx.bench_modmul())
    t_int = model["modmuls"] / _PEAK_MM[0]
    t_hbm = model["bytes"] / (HBM_PEAK * 1e9)
    return {"modmuls": model["modmuls"], "bytes": model["bytes"], "peak_gmodmul_s": round(_PEAK_MM[0] / 1e9, 1),
            "peak_hbm_gbs": HBM_PEAK, "bound": "int" if t_int >= t_hbm else "hbm",
            "roofline_us": round(max(t_int, t_hbm) * 1e6, 2), "frac": round(max(t_int, t_hbm) / (ms_per_layer / 1e3), 4)}

if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4"]
    for w in which:
        if w == "cfg1":
            r = fc("cfg1", 2048, 1, 16, 2048, int(os.environ.get("CFG1_BATCH", "1024")))
        elif w == "cfg2":
            r = fc("cfg2", 4096, 3, 1024, 4096, int(os.environ.get("CFG2_BATCH", "256")))
        elif w == "cfg3":
            r = conv("cfg3", 2048, 1, 16, 16, 64, 64, 3, B=int(os.environ.get("CFG3_BATCH", "16")))
        elif w == "cfg4":
            r = conv("cfg4", 4096, 3, 56, 64, 64, 64, 3, B=int(os.environ.get("CFG4_BATCH", "4")))
        elif w.startswith("conv:"):     # conv:n:L:u:frame:c_i:c_o:k
            a = [int(v) for v in w.split(":")[1:]]
            r = conv(w, *a)
        print(json.dumps(r), flush=True)
