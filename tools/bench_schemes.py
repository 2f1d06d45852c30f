#!/usr/bin/env python
"""GALA vs GAZELLE on the same B200 backend: the paper's comparison, measured.

For each shape, on the GPU backend:
  * the GAZELLE baseline op by op (`mv_hybrid_gazelle` / `mimo_output_rotation`, conv.py:247-265);
  * GALA op by op -- the reference's own loops over the same he_* primitives
    (matvec.py:305-320: sum_t perm(scmult(x, p_t), t); conv.py:268-293: first-Add, second-Perm);
  * GALA fused (`mv_gala` / `mimo_kernel_grouping`: one library call per layer).
Op-by-op times are wall clock around the call with a device synchronize on both sides (every he_*
call is a library call on the GPU; host overhead included, as in an op-by-op deployment).  Also
measures the per-op costs and writes them as a `load_cost_config` calibration
(backend.py:314-334 keys), then compares the analytic estimate (analytics.estimate_time on the
reference's op counts) with the measured op-by-op time.  Every result is decrypted and checked.
Prints JSON lines; `--out DIR` also writes DIR/r1_schemes.jsonl and DIR/r1_cost_config_gpu_*.json.
"""
import argparse
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
from paper_2105_01827_b200 import (  # noqa: E402
    ConvTask, CostMeter, HEParams, MvTask, decrypt, encrypt, encrypt_inputs, he_add, he_decperm, he_hstperm,
    he_perm, he_scmult, mimo_kernel_grouping, mimo_output_rotation, unpack_channels)
from paper_2105_01827_b200.analytics import count_conv, count_mv, estimate_time  # noqa: E402
from paper_2105_01827_b200.backend import CostModel  # noqa: E402
from paper_2105_01827_b200.errors import NoiseOverflowError  # noqa: E402
from paper_2105_01827_b200.conv import DiagonalPlan, _diag_conv, _input_rotations  # noqa: E402
from paper_2105_01827_b200.matvec import (  # noqa: E402
    _finish_single, encode_gala_weights, mv_gala, mv_hybrid_gazelle, pack_input)
from paper_2105_01827_b200.ring import SlotVector  # noqa: E402

P = 1032193


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts)), out


def op_costs(params):
    """Per-op milliseconds of the he_* primitives on this backend (CostModel fields)."""
    rng = np.random.default_rng(0)
    x = encrypt(SlotVector(rng.integers(0, P, params.n), P), params)
    v = SlotVector(rng.integers(0, P, params.n), P)
    m = CostMeter()
    g = he_decperm(x, m)
    he_perm(x, 1, m)
    he_hstperm(g, 1, m)
    reps = 50

    def t(fn):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / reps

    return CostModel(t_perm=t(lambda: he_perm(x, 1, m)), t_scmult=t(lambda: he_scmult(x, v, m)),
                     t_add=t(lambda: he_add(x, x, m)), t_decperm=t(lambda: he_decperm(x, m)),
                     t_hstperm=t(lambda: he_hstperm(g, 1, m)))


def gala_mv_op_by_op(task, ct, meter, rng):
    """The reference's mv_gala loop (matvec.py:305-320) over the he_* primitives."""
    lin = CostMeter(meter.cost_model)
    acc = None
    for t, p_t in enumerate(encode_gala_weights(task)):
        term = he_scmult(ct, p_t, lin)
        if t:
            term = he_perm(term, t, lin)
        acc = term if acc is None else he_add(acc, term, lin)
    meter.merge(lin)
    return _finish_single(task, "gala", acc, task.fold_spec(), task.slot_map(), lin, rng)


def kg_op_by_op(task, cts, meter):
    """The reference's mimo_kernel_grouping loops (conv.py:268-293) over the he_* primitives."""
    c_n = task.channels_per_ct
    n_ib, n_ob, b = task.c_i // c_n, task.c_o // c_n, task.image_slots
    plan = DiagonalPlan(task, c_n)
    rots = [_input_rotations(task, ct, meter) for ct in cts]
    out = []
    for ob in range(n_ob):
        res = None
        for diag in range(c_n):
            acc = None
            for ib in range(n_ib):
                v = _diag_conv(rots[ib], plan.coef_vectors(ob, ib, diag), meter)
                acc = v if acc is None else he_add(acc, v, meter)
            if diag:
                acc = he_perm(acc, diag * b, meter)
            res = acc if res is None else he_add(res, acc, meter)
        out.append(res)
    return out


def fc_case(n, L, n_o, n_i, model):
    params = HEParams(n=n, p=P, rns_limbs=L, seed=61)
    rng = np.random.default_rng(3)
    w = rng.integers(-128, 128, (n_o, n_i)) % P
    x = rng.integers(0, P, n_i)
    task = MvTask(n_i, n_o, w, params)
    ct = encrypt(pack_input(x, task), params)
    want = dot_mod_p(w, x, P)
    res = {"kind": "fc", "n": n, "L": L, "n_o": n_o, "n_i": n_i}
    for name, fn in (("gazelle_op_by_op", lambda m: mv_hybrid_gazelle(task, ct, m, rng=5)),
                     ("gala_op_by_op", lambda m: gala_mv_op_by_op(task, ct, m, 5)),
                     ("gala_fused", lambda m: mv_gala(task, ct, m, rng=5))):
        meter = CostMeter()
        try:
            ms, out = wall(lambda: fn(CostMeter()))
        except NoiseOverflowError as e:   # the real-noise guard of decrypt
            res[name] = {"error": f"NoiseOverflowError: {e}"}
            continue
        fn(meter)
        ok = bool(np.array_equal((out.client_share.slots + out.server_share.slots) % P, want))
        res[name] = {"ms": round(ms, 3), "correct": ok, "counts": repr(meter)}
    gz, ga = count_mv("gazelle", n_i, n_o, n), count_mv("gala", n_i, n_o, n)
    res["estimate_ms"] = {"gazelle": round(estimate_time(gz, model), 3), "gala": round(estimate_time(ga, model), 3)}
    if all("ms" in res[k] for k in ("gazelle_op_by_op", "gala_op_by_op", "gala_fused")):
        res["speedup_op_by_op"] = round(res["gazelle_op_by_op"]["ms"] / res["gala_op_by_op"]["ms"], 2)
        res["speedup_fused"] = round(res["gazelle_op_by_op"]["ms"] / res["gala_fused"]["ms"], 2)
    return res


def conv_case(n, L, u, c_i, c_o, k, model):
    params = HEParams(n=n, p=P, rns_limbs=L, seed=62)
    rng = np.random.default_rng(4)
    kern = rng.integers(-128, 128, (c_o, c_i, k, k)) % P
    img = rng.integers(0, P, (c_i, u, u))
    task = ConvTask(u, u, c_i, k, k, c_o, kern, params)
    cts = encrypt_inputs(task, img)
    want = conv2d_mod_p(img, kern, P)
    res = {"kind": "conv", "n": n, "L": L, "u": u, "c_i": c_i, "c_o": c_o, "k": k}
    for name, fn in (("gazelle_op_by_op", lambda m: mimo_output_rotation(task, cts, m)),
                     ("gala_op_by_op", lambda m: kg_op_by_op(task, cts, m)),
                     ("gala_fused", lambda m: mimo_kernel_grouping(task, cts, m))):
        meter = CostMeter()
        ms, out = wall(lambda: fn(CostMeter()), reps=1)
        fn(meter)
        got = np.concatenate([unpack_channels(decrypt(o), task) for o in out])
        res[name] = {"ms": round(ms, 3), "correct": bool(np.array_equal(got, want)), "counts": repr(meter)}
    gz, ga = (count_conv(s, u, u, c_i, c_o, k, k, n) for s in ("gazelle", "gala"))
    res["estimate_ms"] = {"gazelle": round(estimate_time(gz, model), 3), "gala": round(estimate_time(ga, model), 3)}
    res["speedup_op_by_op"] = round(res["gazelle_op_by_op"]["ms"] / res["gala_op_by_op"]["ms"], 2)
    res["speedup_fused"] = round(res["gazelle_op_by_op"]["ms"] / res["gala_fused"]["ms"], 2)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lines = []
    models = {}
    for n, L in ((2048, 1), (2048, 2), (4096, 3)):
        model = op_costs(HEParams(n=n, p=P, rns_limbs=L, seed=60))
        models[(n, L)] = model
        cfg = {"n": n, "rns_limbs": L, "p": P, "t_perm": model.t_perm, "t_scmult": model.t_scmult,
               "t_add": model.t_add, "t_decperm": model.t_decperm, "t_hstperm": model.t_hstperm}
        lines.append({"kind": "op_costs_ms", **cfg})
        if args.out:
            with open(os.path.join(args.out, f"r1_cost_config_gpu_n{n}_L{L}.json"), "w") as f:
                json.dump(cfg, f, indent=1)
    for n, L, n_o, n_i in ((2048, 1, 1, 2048), (2048, 1, 16, 128), (2048, 1, 16, 2048), (2048, 2, 16, 2048),
                           (2048, 1, 128, 2048), (2048, 2, 128, 2048), (4096, 3, 1024, 4096)):
        lines.append(fc_case(n, L, n_o, n_i, models[(n, L)]))
        print(json.dumps(lines[-1]), flush=True)
    for n, L, u, c_i, c_o, k in ((2048, 1, 16, 64, 64, 3), (2048, 1, 16, 128, 128, 3), (4096, 3, 16, 64, 64, 3)):
        lines.append(conv_case(n, L, u, c_i, c_o, k, models[(n, L)]))
        print(json.dumps(lines[-1]), flush=True)
    for l in lines[:3]:
        print(json.dumps(l))
    if args.out:
        with open(os.path.join(args.out, "r1_schemes.jsonl"), "w") as f:
            for l in lines:
                f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()
