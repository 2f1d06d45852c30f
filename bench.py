#!/usr/bin/env python
"""bench.py -- GALA FC dot product at scale on B200 (BASELINE.json configs[1]).

Workload (one "layer"): a 1024 x 4096 int8 weight matrix (mapped into Z_p,
p = 1032193) against one encrypted input vector of 4096 values, RNS-BFV with
N = 8192, three 60-bit ciphertext primes + one special prime.  The layer is
split into two reference MvTasks (512 x 4096 each, n = 4096, T = 512) paired
on the two hypercube rows of one ciphertext; every layer runs the fused GALA
product (T ScMult, T-1 key-switched rotations on a BSGS tree, lazy ModDown)
and the share-mask subtraction.  A step = one pass over a batch of
independent encrypted inputs already resident in HBM.

Output: one JSON line (driver contract); see DESIGN.md "Measurement".
  --impl reference : the CPU path (oracle/ port of the same algorithm, all host
                     threads) on the same config/metric -- the reference package
                     itself is a pure-Python mock without HE arithmetic.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HE linear-layer throughput (layers/s, rotations/s) + % of INT/HBM roofline"
P = 1032193
N_OUT, N_IN, SLOTS = 1024, 4096, 4096   # configs[1]
WORKLOAD = "gala_fc_1024x4096_N8192_L3"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=512,
                    help="independent layers (inputs) per step per GPU (key-folded tensor-core tiles of 256)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--stream-steps", type=int, default=32,
                    help="batches per streamed e2e call (pinned host staging: ~0.2 GB per batch of 256)")
    ap.add_argument("--baby", type=int, default=0, help="BSGS baby-step count (0: library default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tensor-cores", action="store_true", help="CUDA-core baby-step sums (k_gala_mac2)")
    ap.add_argument("--profile-only", action="store_true", help="run one profiled step and print the breakdown")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def weights(seed=2105):
    rng = np.random.default_rng(seed)
    return rng.integers(-128, 128, (N_OUT, N_IN), dtype=np.int64) % P


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "10"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def modmul_model(N, L, T, baby, schedule):
    from paper_2105_01827_b200.analytics import ks_modmuls, ntt_modmuls, physical_mv_counts

    G = T // baby
    h = ntt_modmuls(N)
    M = L + 1
    rot_items = G * (baby - 1) + (G - 1)
    groups = G + (1 if G > 1 else 0)
    if schedule == 2:
        giant = G - 1
        # ModDowns as executed: the c1 of each giant group g >= 1 (one component) + one final
        # two-component ModDown per input ("Deferred c0 ModDown")
        md_comps = giant + 2
        per_kernel = {
            "k_gala_e": (baby - 1) * 2 * L * M * N,
            "k_gala_mac2": G * (baby - 1) * (2 * M * N + L * N) + G * 2 * L * N,
            "k_gala_tc": G * 2 * L * N,                      # step-0 products; the sums run on the tensor cores
            "k_gala_kf": G * 2 * M * N,                      # rebuild + REDC per group-sum word (sums: tensor cores)
            "k_digits_intt": (1 + giant) * L * h,
            "k_digits_perm": (1 + giant) * L * L * h,
            "k_ks_mac": giant * 2 * L * M * N,
            "k_ntt_inv[moddown]": md_comps * h,
            "k_moddown": md_comps * (L * h + L * N),
        }
        return per_kernel, physical_mv_counts(N, L, T, baby, 2)["modmuls"]
    per_kernel = {
        "k_ct_mul_pts": 2 * L * N * T,
        "k_digits_intt": rot_items * L * h + 2 * L * N * rot_items,
        "k_digits_perm": rot_items * L * L * h,          # digit i into the L other primes (j != i)
        "k_ks_mac": rot_items * 2 * L * M * N,
        "k_ntt_inv[moddown]": groups * 2 * h,
        "k_moddown": groups * (2 * L * h + 2 * L * N),
    }
    total = physical_mv_counts(N, L, T, baby, 1)["modmuls"]
    return per_kernel, total


def ks_modmuls_one(N, L):
    """one full Perm, hybrid key switching, K = 1, D = L digits."""
    from paper_2105_01827_b200.analytics import ntt_modmuls

    h, K, D = ntt_modmuls(N), 1, L
    return (L + D * (L + K - 1) + 2 * K + 2 * L) * h + (2 * D * (L + K) + 2 * L) * N


def hbm_model(N, L, T, baby, B, tc):
    """Algorithmic DRAM bytes per step of the schedule-2 baby-step kernels (batch of B inputs).

    SURVEY.md 8(d) counts the layer's own objects only -- input ciphertexts, weight plaintexts,
    keys, outputs -- and no intermediates (they are the fusion target).  Per kernel that leaves:
    k_gala_e (-> E_jj, an intermediate): the inputs' identity digit blocks and the baby-step keys
    (read once per 32-input tile); k_gala_tc / k_gala_mac2: the weights and the inputs' c1 (the
    step-0 product).  The group sums U, C they write are intermediates too (the giant steps consume
    them).  `traffic` (ncu) against these shows the round trips still to remove."""
    M = L + 1
    MN = M * N
    dig = B * (L * M + L) * N * 8                                 # identity digit blocks (of the inputs)
    keys = (baby - 1) * L * 2 * MN * 8
    x_c1 = B * L * N * 8
    if tc == "kf":
        # k_gala_kf: the inputs' digit blocks (reordered by k_gala_dq) and the weights + baby-step keys it
        # folds (k_gala_kfw re-encodes them offline; the folded form is read once per 256-input tile)
        from paper_2105_01827_b200.analytics import kf_tiles

        return {"k_gala_kf": dig + (T * MN * 8 + keys) * kf_tiles(B), "k_gala_dq": dig}
    if tc:
        tiles = (B + 31) // 32                                    # one e_can / tc pair per 32 inputs
        return {"k_gala_e": dig + keys * tiles, "k_gala_tc": T * MN * 8 * tiles + x_c1}
    return {"k_gala_e": dig + keys, "k_gala_mac2": T * MN * 8 + x_c1}


def layer_config(N, L, T, baby, schedule):
    """The headline layer (BASELINE.json configs[1]) -- the same dict in both arms' lines."""
    return {"workload": WORKLOAD, "layer": "GALA FC 1024x4096 (2 paired MvTasks of 512x4096, T=512)",
            "N": N, "L": L, "special_primes": 1, "p": P, "T": T, "bsgs_baby": baby, "gala_schedule": schedule}


def run_ours(args):
    import torch

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2105_01827_b200 import _lib
    from paper_2105_01827_b200.backend import HEParams
    from paper_2105_01827_b200.matvec import GalaFC

    params = HEParams(n=SLOTS, p=P, rns_limbs=3, device=local, seed=7)
    t_setup = time.perf_counter()
    layer = GalaFC(weights(), params, baby=args.baby or None, tensor_cores=not args.no_tensor_cores)
    ctx = layer.ctx
    N, L, T, baby = ctx.N, ctx.L, layer.T, layer.baby
    B = args.batch
    rng = np.random.default_rng(1000 + rank)
    xs = [rng.integers(0, P, N_IN) for _ in range(B)]
    cts = [layer.encrypt_input(x)[0] for x in xs]                     # client side, resident in HBM
    masks = [layer.draw_masks(5000 + 100 * rank + b) for b in range(B)]
    phys_r = [ctx.physical(m[0][0].slots, m[0][1].slots) for m in masks]
    d_r = ctx.to_device_u32(np.stack(phys_r))
    pts = layer.blocks[0][1]
    cts_b = torch.stack(cts)
    outs = ctx.empty_ct(B)
    masked = ctx.empty_ct(B)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    def step():
        # one batched library call: all B layers share every launch
        layer.run_batch(cts_b, pts, d_r, outs=outs, masked=masked)

    # correctness gate before timing: decrypted shares == W x mod p
    w = weights()
    step()
    for b in range(min(B, 2)):
        got = (layer.client_shares([masked[b]]) + layer.server_shares(masks[b])) % P
        want = (w @ xs[b]) % P
        if not np.array_equal(got, want):
            raise SystemExit(f"parity gate failed on input {b}")

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MB > 126 MB L2
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # profile pass (untimed): per-kernel CUDA-event breakdown of one step
    ctx.profile(True)
    step()
    prof = ctx.profile_read()
    ctx.profile(False)
    if args.profile_only and rank == 0:
        print(json.dumps(prof, indent=1))
        return

    stream = torch.cuda.current_stream(dev)
    launches0 = _lib.launch_count()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = _lib.launch_count() - launches0
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    layers = B * args.steps * world
    value = layers / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # e2e: host buffers through the C-ABI host entry point (H2D ct + r, fused layer, D2H masked)
    import ctypes

    host_ct = torch.from_numpy(ctx.export_words(cts_b).view(np.int64)).pin_memory()
    host_r = torch.from_numpy(np.stack(phys_r).view(np.int32)).pin_memory()
    host_out = torch.empty((B, 2, L, N), dtype=torch.int64).pin_memory()
    h = ctx._bind()

    def e2e_step():
        # one C-ABI call per step: H2D of B canonical ciphertexts + masks, fused layers, D2H of masked words
        if layer.schedule == 2 and layer.wcan[0] is not None:
            _lib.check(ctx.lib.gala_mv_gala2_batch_tc_host(h, ctypes.c_void_p(host_ct.data_ptr()), B,
                                                           ctypes.c_void_p(pts.data_ptr()),
                                                           ctypes.c_void_p(layer.wcan[0].data_ptr()), T, baby,
                                                           ctypes.c_void_p(host_r.data_ptr()),
                                                           ctypes.c_void_p(host_out.data_ptr())))
            return
        host_fn = ctx.lib.gala_mv_gala2_batch_host if layer.schedule == 2 else ctx.lib.gala_mv_gala_batch_host
        _lib.check(host_fn(h, ctypes.c_void_p(host_ct.data_ptr()), B,
                                                   ctypes.c_void_p(pts.data_ptr()), T, baby,
                                                   ctypes.c_void_p(host_r.data_ptr()),
                                                   ctypes.c_void_p(host_out.data_ptr())))

    e2e_step()
    # e2e parity: host-path masked words equal the device-path masked words
    if not np.array_equal(host_out.numpy().view(np.uint64), ctx.export_words(masked)):
        raise SystemExit("e2e host path disagrees with device path")
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_times.append(e0.elapsed_time(e1))
    e2e_ms = sum(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_sync_value = layers / (e2e_ms / 1e3)

    # e2e, streamed (the serving form): one C-ABI call takes all K steps' inputs from pinned host memory and
    # returns all K steps' masked words there; each step's H2D and D2H overlap the neighbouring steps' layers
    # (gala_mv_gala2_stream_host).  Every step's copies are inside the timed region.
    K = args.steps
    S = max(1, min(K, args.stream_steps))   # batches per streamed call (pinned staging bounded); K steps = ceil(K / S) calls
    stream_ct = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(host_ct.numpy()[None], (S,) + tuple(host_ct.shape)))).pin_memory()
    stream_r = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(host_r.numpy()[None], (S,) + tuple(host_r.shape)))).pin_memory()
    stream_out = torch.empty((S, B, 2, L, N), dtype=torch.int64).pin_memory()
    wc = layer.wcan[0] if layer.schedule == 2 and layer.wcan[0] is not None else None

    def e2e_stream(nsteps):
        _lib.check(ctx.lib.gala_mv_gala2_stream_host(h, ctypes.c_void_p(stream_ct.data_ptr()), nsteps, B,
                                                     ctypes.c_void_p(pts.data_ptr()),
                                                     ctypes.c_void_p(wc.data_ptr() if wc is not None else None),
                                                     T, baby, ctypes.c_void_p(stream_r.data_ptr()),
                                                     ctypes.c_void_p(stream_out.data_ptr())))

    e2e_stream_value = None
    if layer.schedule == 2:
        e2e_stream(min(S, 3))
        torch.cuda.synchronize()
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done = 0
        while done < K:
            e2e_stream(min(S, K - done))
            done += S
        e1.record(stream)
        torch.cuda.synchronize()
        st_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([st_ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            st_ms = float(t.item())
        want = host_out.numpy()
        for k in sorted({0, S // 2, S - 1}):
            if not np.array_equal(stream_out[k].numpy(), want):
                raise SystemExit(f"streamed e2e step {k} disagrees with the device path")
        e2e_stream_value = layers / (st_ms / 1e3)
    e2e_value = e2e_stream_value if e2e_stream_value is not None else e2e_sync_value

    # raw key-switch probe: hoisted full rotations of the batch's inputs, 8 steps each
    ks_steps = [1, 2, 3, 5, 8, 13, 21, 34]
    rot_outs = ctx.rotate_batch(cts_b, ks_steps)
    torch.cuda.synchronize()
    ks_ms = []
    for _ in range(5):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        ctx.rotate_batch(cts_b, ks_steps)
        a1.record(stream)
        torch.cuda.synchronize()
        ks_ms.append(a0.elapsed_time(a1))
    ks_ms_med = float(np.median(ks_ms))
    ks_rot_per_s = B * len(ks_steps) / (ks_ms_med / 1e3)
    del rot_outs

    # roofline: integer-multiply bound (modmul count) -- peak measured live with the library's own modmul
    peak_modmul = ctx.bench_modmul()
    per_kernel, layer_modmuls = modmul_model(N, L, T, baby, layer.schedule)
    dominant = max(prof.items(), key=lambda kv: kv[1]["ms"])
    dom_name, dom = dominant
    step_ms_prof = sum(v["ms"] for v in prof.values())
    dom_work = per_kernel.get(dom_name, 0) * B
    dom_achieved = dom_work / (dom["ms"] / 1e3) if dom["ms"] else 0.0
    layer_achieved = layer_modmuls * layers / world / (total_ms / 1e3)

    kf_on = "k_gala_kf" in prof            # key-folded tensor-core baby steps (the library's default form)
    tc_on = layer.wcan[0] is not None and B >= 16 and (kf_on or B <= 32 or (T >= 128 and (B % 32 == 0 or B % 32 >= 16)))
    tc_form = "kf" if kf_on else tc_on
    traffic = None    # DRAM bytes per launch of the dominant kernel from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            tj = json.load(f)
        # per launch: a capture of one full tile stands for every batch of full tiles
        ent = tj.get("kernels", {}).get(dom_name)
        if ent and B % int(ent["tile"]) == 0:
            traffic = int(ent["bytes"])
    except Exception:
        pass
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    pt_bytes = T * L * N * 8
    key_bytes = ctx.key_bytes()
    ct_bytes = 2 * L * N * 8
    layer_bytes = pt_bytes / B + key_bytes / B + 3 * ct_bytes + N * 4   # weights/keys amortised over the batch

    # int8 tensor roof: the measured tcgen05 kind::i8 issue rate (tools/mma_bench.cu, profiles/r2_mma_bench.txt:
    # 8192 MACs per clock per SM) at the maximum SM clock -- higher than 2x the cuBLAS bf16 figure, so the
    # stricter roof
    from paper_2105_01827_b200.analytics import tensor_i8_peak_ops

    i8_peak = tensor_i8_peak_ops(torch.cuda.get_device_properties(dev).multi_processor_count,
                                 peaks.get("sm_max_mhz", 1965.0), peaks.get("bf16_tflops", 1639.9))
    # dominant kernel against every roof it has (integer multiplies, HBM bytes, int8 tensor MACs);
    # the reported bound is the tightest one (highest fraction)
    dom_s = dom["ms"] / 1e3 if dom["ms"] else 0.0          # profile pass = one step
    # the tensor-core pair runs once per tile of 32 inputs: per-launch figures divide by the tiles
    from paper_2105_01827_b200.analytics import KF_MACS_PER_POSITION, kf_tiles, kf_useful_mac_frac

    if kf_on and dom_name in ("k_gala_kf", "k_gala_dq"):
        launches_per_step = kf_tiles(B)
    elif tc_on and dom_name in ("k_gala_e", "k_gala_tc"):
        launches_per_step = (B + 31) // 32
    else:
        launches_per_step = 1
    roofs = {}
    if per_kernel.get(dom_name):
        a = per_kernel[dom_name] * B / dom_s if dom_s else 0.0
        roofs["int"] = {"achieved": round(a / 1e9, 2), "peak": round(peak_modmul / 1e9, 2), "unit": "Gmodmul/s",
                        "frac": round(a / peak_modmul, 4), "peak_source": "measured live: gala_bench_modmul"}
    hb = hbm_model(N, L, T, baby, B, tc_form).get(dom_name)
    if hb:
        a = hb / dom_s if dom_s else 0.0
        roofs["hbm"] = {"achieved": round(a / 1e9, 2), "peak": hbm_peak, "unit": "GB/s", "frac": round(a / 1e9 / hbm_peak, 4),
                        "algorithmic_bytes_per_launch": int(hb / launches_per_step),
                        "launches_per_step": launches_per_step, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    if dom_name == "k_gala_tc":
        macs = (L + 1) * N * 128 * 128 * 512 * launches_per_step  # issued int8 MACs (byte-convolution tiles)
        int8_peak = i8_peak
        a = 2 * macs / dom_s if dom_s else 0.0
        # useful share of the issued MACs: 96 of the 128 M rows carry data (3 streams x 32 inputs), and of
        # the 16 byte shifts x 8 byte positions of each (row, group, rotation) only the 64 with
        # 0 <= s' - a < 8 are non-zero Toeplitz entries
        roofs["tensor"] = {"achieved": round(a / 1e12, 2), "peak": round(int8_peak / 1e12, 1), "unit": "TOP/s",
                           "frac": round(a / int8_peak, 4), "useful_mac_frac": 0.375,
                           "useful_frac_of_peak": round(0.375 * a / int8_peak, 4),
                           "peak_source": "tcgen05 kind::i8 issue rate measured by tools/mma_bench.cu x SMs x sm_max_mhz"}
    if dom_name == "k_gala_kf":
        macs = (L + 1) * N * KF_MACS_PER_POSITION * launches_per_step   # issued int8 MACs (CTA-pair MMAs)
        int8_peak = i8_peak
        a = 2 * macs / dom_s if dom_s else 0.0
        uf = kf_useful_mac_frac(B, L, T // baby, baby)
        roofs["tensor"] = {"achieved": round(a / 1e12, 2), "peak": round(int8_peak / 1e12, 1), "unit": "TOP/s",
                           "frac": round(a / int8_peak, 4), "useful_mac_frac": round(uf, 4),
                           "useful_frac_of_peak": round(uf * a / int8_peak, 4),
                           "peak_source": "tcgen05 kind::i8 issue rate measured by tools/mma_bench.cu (8192 MAC/clk/SM) "
                                          "x SMs x MEASURED_PEAKS.json sm_max_mhz"}
    bound = max(roofs, key=lambda r: roofs[r]["frac"]) if roofs else "int"
    br = roofs.get(bound, {"achieved": 0.0, "peak": 0.0, "unit": "", "frac": 0.0})
    # the whole step against SURVEY.md 8(d)'s formula with the work the schedule executes
    # (analytics.fc_executed_work: CUDA-core modmuls at the modmul peak, int8 MACs at 2x the bf16 peak,
    # bytes at HBM): the slowest roof over the measured step time
    from paper_2105_01827_b200.analytics import executed_roofline, fc_executed_work

    work = fc_executed_work(N, L, T, baby, B, tc_form)
    lr = executed_roofline(work, work["bytes"], ms_per_step / 1e3, peak_modmul, i8_peak, hbm_peak * 1e9)
    layer_roof = {"bound": lr["bound"], "frac": lr["frac"], "roofline_us_per_step": lr["roofline_us"],
                  "measured_us_per_step": round(ms_per_step * 1e3, 1), "modmuls_per_step": lr["modmuls"],
                  "int8_macs_per_step": lr["int8_macs"], "bytes_per_step": lr["bytes"],
                  "roof_times_us": {k: round(v * 1e6, 2) for k, v in lr["times_s"].items()},
                  "model": "analytics.fc_executed_work (schedule 2 as executed; SURVEY 8(d) formula)"}

    result = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "layers/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64 (RNS residues mod 60-bit primes)",
        "data": "synthetic (seeded int8 weights mapped to Z_p, uniform Z_p inputs)",
        # the layer both arms compute (identical dict in the reference arm's line); how this arm runs it
        # (batching, tensor cores, L2 policy) is under "run"
        "config": layer_config(N, L, T, baby, layer.schedule),
        "run": {"batch_per_gpu": B,
                "baby_step_sums": ("tcgen05 int8 MMA, key-folded weights, CTA pairs (k_gala_kf)" if kf_on else
                                   "tcgen05 int8 MMA (k_gala_e_can + k_gala_tc)" if tc_on else "CUDA cores"),
                "parallelism": f"replicas x{world} (independent inputs per GPU)",
                "l2": "flushed (256 MB write) before every timed step"},
        "rotations_per_s": round(value * (T - 1), 1),
        "ks_probe": {"rotations_per_s": round(ks_rot_per_s, 1), "batch": B, "steps_per_input": len(ks_steps),
                     "ms": round(ks_ms_med, 4),
                     "modmuls_per_rotation": ks_modmuls_one(N, L),
                     "achieved_gmodmul_s": round(ks_rot_per_s * ks_modmuls_one(N, L) / 1e9, 1),
                     "note": "hoisted full key switches (one decomposition per input, one ModDown per output), "
                             "gala_rotate_batch; SURVEY 8(d) count per rotation"},
        "roofline": {
            "bound": bound,
            "kernel": dom_name,
            "achieved": br["achieved"],
            "peak": br["peak"],
            "unit": br["unit"],
            "frac": br["frac"],
            "traffic": traffic,
            "traffic_unit": "bytes per launch (dram read + write, ncu --set full, profiles/r2_ncu_summary.md)",
            "kernel_share_of_step": round(dom["ms"] / step_ms_prof, 4) if step_ms_prof else None,
            "roofs": roofs,
            "layer": layer_roof,
            "hbm": {"algorithmic_bytes_per_layer": int(layer_bytes),
                    "achieved_gbs": round(layer_bytes * layers / world / (total_ms / 1e3) / 1e9, 2),
                    "peak_gbs": hbm_peak},
        },
        "kernel_breakdown_ms_per_step": {k: round(v["ms"], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])},
        "e2e": {"value": round(e2e_value, 3), "unit": "layers/s",
                "h2d_bytes_per_step": B * (ct_bytes + N * 4), "d2h_bytes_per_step": B * ct_bytes,
                "path": ("gala_mv_gala2_stream_host (C-ABI, pinned host buffers, canonical words; one call per "
                         f"{S} steps, each step's H2D and D2H overlapped with the neighbouring steps' layers; "
                         "words of the first, middle and last batch of a call checked against the device path)")
                        if e2e_stream_value is not None else
                        (f"gala_mv_gala{layer.schedule if layer.schedule == 2 else ''}_batch_host"
                         " (C-ABI, pinned host buffers, canonical words, one call per step)"),
                "sync_per_step": {"value": round(e2e_sync_value, 3),
                                  "path": ("gala_mv_gala2_batch_tc_host" if tc_on else
                                           f"gala_mv_gala{layer.schedule if layer.schedule == 2 else ''}_batch_host")
                                          + " (one blocking call per step: copies not overlapped)"}},
        "gpu_launches": int(launches),
        "setup_s": round(setup_s, 2),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(ctx, layer, cts[0], phys_r[0], masked[0])
    if rank == 0:
        print(json.dumps(result))
    if world > 1:
        torch.distributed.destroy_process_group()


def _oracle_for(bfv, seed):
    """CPU oracle with the GPU context's secret and rotation keys (same host randomness)."""
    from oracle.bfv import Oracle
    from paper_2105_01827_b200 import sampling

    o = Oracle(bfv)
    o.set_secret(sampling.secret(np.random.default_rng([seed, 0]), bfv.N))
    return o


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_MOCK_SNIPPET = r"""
import sys, time, json
import numpy as np
sys.path.insert(0, sys.argv[1])
from gala.backend import CostMeter, HEParams
from gala.matvec import MvTask, run_mv
P, reps = int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(2105)
w = rng.integers(-128, 128, (1024, 4096), dtype=np.int64) % P
x = rng.integers(0, P, 4096, dtype=np.int64)
params = HEParams(n=4096, p=P)
task = MvTask(4096, 1024, w, params)
run_mv("gala", task, x, CostMeter(), rng=1)
ts = []
for i in range(reps):
    t0 = time.perf_counter()
    run_mv("gala", task, x, CostMeter(), rng=i)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"median_s": float(np.median(ts)), "T": task.groups}))
"""


def reference_mock_baseline(reps: int = 3):
    """SURVEY.md 8(d) baseline 1: the reference package itself (baseline/_ref, unmodified), its own
    run_mv("gala") on the config-2 matrix at n = 4096 (T = 1024), single-threaded NumPy.  It times
    slot arithmetic on a mock backend -- no HE -- so it is reported, not compared."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gala")):
        return {"unavailable": "baseline/_ref not installed (see DESIGN.md section 8)"}
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    try:
        r = subprocess.run([sys.executable, "-c", _MOCK_SNIPPET, ref, str(P), str(reps)], capture_output=True,
                           text=True, timeout=300, env=env)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        return {"unavailable": f"reference mock run failed: {e}"}
    return {"value": round(1.0 / d["median_s"], 3), "unit": "layers/s", "cores": 1, "kind": "reference",
            "sample": f"reference run_mv('gala') on the 1024x4096 matrix, HEParams(n=4096, p={P}) (T={d['T']}), "
                      f"median of {reps}; NumPy slot mock, no HE arithmetic"}


def cpu_baseline(ctx, layer, ct, phys_r, masked_gpu):
    """Oracle port of the same fused layer, timed on the host cores (one layer = the sample)."""
    from oracle.bfv import num_threads
    from paper_2105_01827_b200 import sampling

    bfv = ctx.bfv
    o = _oracle_for(bfv, ctx.seed)
    for s in layer.steps:
        a, e = sampling.rotation_key_randomness(np.random.default_rng([ctx.seed, 1, s]), bfv)
        o.gen_rotkey(s, a, e)
    tasks = layer.blocks[0][0]
    from paper_2105_01827_b200.matvec import gala_weight_slots

    pts = np.concatenate([gala_weight_slots(tasks[0]), gala_weight_slots(tasks[1])], axis=1).astype(np.uint32)
    words = ctx.export_words(ct)
    t0 = time.perf_counter()
    _, m = o.mv_gala(words, pts, phys_r, baby=layer.baby, schedule=layer.schedule)
    dt = time.perf_counter() - t0
    match = bool(np.array_equal(m, ctx.export_words(masked_gpu)))
    return {"value": round(1.0 / dt, 4), "unit": "layers/s", "cores": num_threads(), "kind": "port",
            "sample": "1 layer (same input ct, keys and mask as GPU input 0); oracle/bfv_oracle.c, OpenMP",
            "words_match_gpu": match, "host_cpus": os.cpu_count(), "cpu_model": cpu_model(),
            "reference_mock": reference_mock_baseline()}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.bfv import num_threads
    from paper_2105_01827_b200 import sampling
    from paper_2105_01827_b200.matvec import MvTask, gala_weight_slots, pack_input
    from paper_2105_01827_b200.params import derive

    bfv = derive(SLOTS, P, 3)
    seed = 7
    o = _oracle_for(bfv, seed)
    w = weights()
    from paper_2105_01827_b200.backend import HEParams

    params = HEParams(n=SLOTS, p=P, rns_limbs=3, seed=seed)
    tasks = [MvTask(N_IN, N_OUT // 2, w[:N_OUT // 2], params), MvTask(N_IN, N_OUT // 2, w[N_OUT // 2:], params)]
    pts = np.concatenate([gala_weight_slots(tasks[0]), gala_weight_slots(tasks[1])], axis=1).astype(np.uint32)
    T = pts.shape[0]
    # the GPU arm's baby-step split (Context.gala2_baby: b = 2^round(log2 sqrt(7 T)), 64 at T = 512)
    baby = 1 << int(round(math.log2(math.sqrt(7 * T))))
    G = T // baby
    for s in sorted({j for j in range(1, baby)} | {g * baby for g in range(1, G)}):
        a, e = sampling.rotation_key_randomness(np.random.default_rng([seed, 1, s]), bfv)
        o.gen_rotkey(s, a, e)
    rng = np.random.default_rng(1000)
    x = rng.integers(0, P, N_IN)
    xs = pack_input(x, tasks[0]).slots
    phys = np.concatenate([xs, xs]).astype(np.uint32)
    a, e = sampling.encryption_randomness(np.random.default_rng([seed, 2, 0]), bfv)
    ct = o.encrypt(phys, a, e)
    r = np.random.default_rng(5000).integers(0, P, 2 * SLOTS).astype(np.uint32)
    schedule = 2   # the production schedule for L = 3 (same algorithm as the GPU arm)
    if args.warmup > 0:
        o.mv_gala(ct, pts, r, baby=baby, schedule=schedule)   # one warm-up layer (bounded CPU sample)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.mv_gala(ct, pts, r, baby=baby, schedule=schedule)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = args.steps / total
    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "layers/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues mod 60-bit primes)",
        "data": "synthetic", "impl": "reference",
        "config": layer_config(bfv.N, bfv.L, T, baby, schedule),
        "run": {"layers_per_step": 1, "threads": num_threads()},
        "cpu_baseline": {"value": round(value, 4), "unit": "layers/s", "cores": num_threads(), "kind": "port",
                         "sample": "1 layer per step: oracle/bfv_oracle.c (same algorithm), OpenMP, all host threads",
                         "cpu_model": cpu_model(), "host_cpus": os.cpu_count()},
        "e2e": {"value": round(value, 4), "unit": "layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference package's own backend is a pure-Python slot mock without HE arithmetic; "
                "the CPU arm runs the restated RNS-BFV algorithm (oracle/) on the host cores",
    }
    print(json.dumps(out))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
