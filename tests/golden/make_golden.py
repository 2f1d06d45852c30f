"""Generate golden fixtures by running the REFERENCE package (mock backend).

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
Outputs tests/golden/*.npz.  The GPU box never reads /root/reference; the
tests load these fixtures instead.  p = 1032193 (batching-friendly; the
reference accepts any prime < 2^31, backend.py:103-106).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
P = 1032193


def main():
    sys.path.insert(0, REF)
    from gala.analytics import OpCounts
    from gala.backend import CostMeter, HEParams, encrypt, with_overrides
    from gala.conv import ConvTask, encrypt_inputs, mimo_kernel_grouping, mimo_output_rotation
    from gala.matvec import MvTask, column_blocks, encode_gala_weights, pack_input, run_mv

    base = with_overrides(HEParams(), p=P)

    # ---- GALA dot products: (n, n_o, n_i, seed) -------------------------------
    mv_cases = [(64, 4, 16, 1), (64, 64, 64, 2), (256, 16, 128, 3), (256, 8, 256, 4), (2048, 1, 2048, 5),
                (2048, 2, 1024, 6), (2048, 16, 128, 7), (2048, 16, 2048, 8), (2048, 8, 2048, 9),
                (1024, 4, 16, 11), (512, 256, 512, 12)]
    mv = {}
    for idx, (n, n_o, n_i, seed) in enumerate(mv_cases):
        params = with_overrides(base, n=n)
        rng = np.random.default_rng(seed)
        w = rng.integers(-128, 128, (n_o, n_i), dtype=np.int64) % P
        x = rng.integers(0, P, n_i, dtype=np.int64)
        task = MvTask(n_i, n_o, w, params)
        meter = CostMeter()
        out = run_mv("gala", task, x, meter, rng=1000 + seed)
        c = OpCounts.from_meter(meter)
        pref = f"c{idx}_"
        mv[pref + "dims"] = np.array([n, n_o, n_i, seed, 1000 + seed])
        mv[pref + "w"] = ((w + 128) % P - 128).astype(np.int8)  # int8 weights, mapped into Z_p by % P
        mv[pref + "x"] = x.astype(np.uint32)
        mv[pref + "payload"] = out.output_cipher.payload.slots.astype(np.uint32)
        mv[pref + "server"] = out.server_share.slots.astype(np.uint32)
        mv[pref + "client"] = out.client_share.slots.astype(np.uint32)
        mv[pref + "counts"] = np.array([c.perm, c.dec_perm, c.hst_perm, c.sc_mult, c.add, out.share_meter.add])
        mv[pref + "noise"] = np.array([out.output_cipher.noise])
        print("mv", n, n_o, n_i, "T", task.groups, c)
    mv["count"] = np.array([len(mv_cases)])
    np.savez_compressed(os.path.join(HERE, "mv_gala.npz"), **mv)

    # ---- kernel-grouping convolutions: (u, c_i, k, c_o, n, seed) --------------
    conv_cases = [(4, 4, 1, 4, 64, 1), (4, 8, 3, 8, 64, 2), (4, 4, 3, 8, 64, 3), (4, 8, 3, 8, 128, 4),
                  (4, 8, 1, 8, 128, 5), (8, 8, 3, 16, 256, 6), (2, 4, 3, 4, 16, 7), (16, 64, 3, 64, 2048, 8),
                  (8, 4, 5, 4, 64, 9)]
    cv = {}
    for idx, (u, c_i, k, c_o, n, seed) in enumerate(conv_cases):
        params = with_overrides(base, n=n)
        rng = np.random.default_rng(seed)
        kern = rng.integers(-128, 128, (c_o, c_i, k, k), dtype=np.int64) % P
        ch = rng.integers(0, P, (c_i, u, u), dtype=np.int64)
        task = ConvTask(u, u, c_i, k, k, c_o, kern, params)
        meter = CostMeter()
        outs = mimo_kernel_grouping(task, encrypt_inputs(task, ch), meter)
        c = OpCounts.from_meter(meter)
        pref = f"c{idx}_"
        cv[pref + "dims"] = np.array([u, c_i, k, c_o, n, seed])
        cv[pref + "kernels"] = ((kern + 128) % P - 128).astype(np.int8)
        cv[pref + "channels"] = ch.astype(np.uint32)
        cv[pref + "payloads"] = np.stack([o.payload.slots for o in outs]).astype(np.uint32)
        cv[pref + "counts"] = np.array([c.perm, c.dec_perm, c.hst_perm, c.sc_mult, c.add])
        cv[pref + "noise"] = np.array([o.noise for o in outs])
        print("conv", u, c_i, k, c_o, n, c)
    cv["count"] = np.array([len(conv_cases)])
    np.savez_compressed(os.path.join(HERE, "conv_kg.npz"), **cv)

    # ---- op-level: rotations / scmult / add on a 64-slot vector --------------
    from gala.backend import he_add, he_perm, he_scmult, subtract_plain
    from gala.ring import SlotVector

    params = with_overrides(base, n=64)
    rng = np.random.default_rng(77)
    x = rng.integers(0, P, 64)
    y = rng.integers(0, P, 64)
    meter = CostMeter()
    cx = encrypt(SlotVector(x, P), params)
    ops = {"x": x, "y": y}
    for k in (1, 5, 17, 63):
        ops[f"rot{k}"] = he_perm(cx, k, meter).payload.slots
    ops["scmult"] = he_scmult(cx, SlotVector(y, P), meter).payload.slots
    ops["add"] = he_add(cx, encrypt(SlotVector(y, P), params), meter).payload.slots
    ops["sub"] = subtract_plain(cx, SlotVector(y, P), meter).payload.slots
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **ops)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
