"""Packed-HE matrix-vector products on the GPU backend (reference: pkg/src/gala/matvec.py).

``mv_gala`` -- the hot path -- is one fused library call
(``gala_mv_gala``): all T plaintext products, the BSGS rotation tree with
lazy ModDown, and the share-mask subtraction run on the GPU in a handful of
launches; the caller's meter receives the reference's logical counts
(T ScMult, T-1 Perm, T-1 Add; matvec.py:305-320, analytics.count_mv).
The three baselines (naive, diagonal, gazelle) run op by op through the same
GPU backend, exactly as the reference composes them.

``GalaFC`` is the throughput form: a resident-weight layer whose logical
MvTasks are paired on the two hypercube rows of each ciphertext.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .backend import (
    Ciphertext,
    CostMeter,
    HEParams,
    context,
    decrypt,
    encrypt,
    he_add,
    he_decperm,
    he_hstperm,
    he_perm,
    he_scmult,
)
from .errors import DimensionError, ParameterError
from .ring import SlotVector, fold_ras, is_power_of_two, read_slots, rotate_left
from .sharing import draw_mask, gen_additive_share


@dataclass
class MvTask:
    """One n_o x n_i dot product with n_o <= n_i <= n (matvec.py:41-98)."""

    n_i: int
    n_o: int
    w: np.ndarray
    params: HEParams

    def __post_init__(self):
        for name, v in (("n_i", self.n_i), ("n_o", self.n_o)):
            if not is_power_of_two(v):
                raise ParameterError(f"{name} must be a power of two, got {v}")
        if not self.n_o <= self.n_i <= self.params.n:
            raise ParameterError(f"need n_o <= n_i <= n, got {self.n_o}x{self.n_i} with n={self.params.n}")
        w = np.asarray(self.w, dtype=np.int64)
        if w.shape != (self.n_o, self.n_i):
            raise DimensionError(f"w has shape {w.shape}, expected {(self.n_o, self.n_i)}")
        self.w = w % self.params.p

    @property
    def copies(self) -> int:
        return self.params.n // self.n_i

    @property
    def n_o_padded(self) -> int:
        return max(self.n_o, self.copies)

    @property
    def groups(self) -> int:
        return self.n_i * self.n_o_padded // self.params.n

    def padded_matrix(self) -> np.ndarray:
        if self.n_o_padded == self.n_o:
            return self.w
        out = np.zeros((self.n_o_padded, self.n_i), dtype=np.int64)
        out[: self.n_o] = self.w
        return out

    def slot_map(self) -> list[int]:
        t = self.groups
        return [(r // t) * self.n_i + (r % t) for r in range(self.n_o)]

    def fold_spec(self) -> tuple[int, int]:
        return (self.n_i, self.groups)


@dataclass
class MvOutcome:
    scheme: str
    output_cipher: Ciphertext | list
    server_share: SlotVector
    client_share: SlotVector
    slot_map: list
    fold_spec: tuple
    meter: CostMeter
    share_meter: CostMeter
    seed: int | None = None


def _resolve_rng(rng):
    return np.random.default_rng(rng), (rng if isinstance(rng, int) else None)


def pack_input(x, task: MvTask) -> SlotVector:
    """x tiled n/n_i times (matvec.py:126-131)."""
    x = np.asarray(x, dtype=np.int64)
    if x.shape != (task.n_i,):
        raise DimensionError(f"x has shape {x.shape}, expected ({task.n_i},)")
    return SlotVector(np.tile(x, task.copies), task.params.p)


def embed_input(x, task: MvTask) -> SlotVector:
    x = np.asarray(x, dtype=np.int64)
    if x.shape != (task.n_i,):
        raise DimensionError(f"x has shape {x.shape}, expected ({task.n_i},)")
    out = np.zeros(task.params.n, dtype=np.int64)
    out[: task.n_i] = x % task.params.p
    return SlotVector._wrap(out, task.params.p)


def column_blocks(w, x, n: int):
    """(w_block, x_block) pairs of at most n columns (matvec.py:144-159)."""
    w, x = np.asarray(w), np.asarray(x)
    n_i = w.shape[1]
    if n_i <= n:
        yield w, x
        return
    if n_i % n:
        raise ParameterError(f"n_i={n_i} is not a multiple of the block width {n}")
    for lo in range(0, n_i, n):
        yield w[:, lo:lo + n], x[lo:lo + n]


def gala_weight_slots(task: MvTask) -> np.ndarray:
    """[T][n] slot values of the row-wise (GALA) encoding.

    Slot j of plaintext t holds w[r((j - t) mod n)][j mod n_i] with row class
    r(j) = (j // n_i) T + (j mod T)  (matvec.py:162-182), vectorised.
    """
    n, T = task.params.n, task.groups
    wp = task.padded_matrix()
    j = np.arange(n)
    src = (j[None, :] - np.arange(T)[:, None]) % n
    rows = (src // task.n_i) * T + (src % T)
    return wp[rows, (j % task.n_i)[None, :]]


def encode_gala_weights(task: MvTask) -> list[SlotVector]:
    return [SlotVector._wrap(row.copy(), task.params.p) for row in gala_weight_slots(task)]


def _encode_cyclic_diagonals(task: MvTask) -> list[SlotVector]:
    n, p = task.params.n, task.params.p
    j = np.arange(n)
    rows = j % task.n_o
    return [SlotVector._wrap(task.w[rows, (j + k) % task.n_i], p) for k in range(task.n_i)]


def _he_fold(ct, start, end, meter):
    s = start // 2
    while s >= end:
        ct = he_add(ct, he_perm(ct, s, meter), meter)
        s //= 2
    return ct


def _acc(acc, term, meter):
    return term if acc is None else he_add(acc, term, meter)


def _finish_single(task, scheme, ct, fold_spec, slot_map, lin, rng):
    from .backend import CostMeter as _CM

    gen, seed = _resolve_rng(rng)
    share_meter = _CM(lin.cost_model)
    r, masked = gen_additive_share(ct, gen, share_meter)
    start, end = fold_spec
    client = read_slots(fold_ras(decrypt(masked), start, end), slot_map)
    server = read_slots(fold_ras(r, start, end), slot_map)
    return MvOutcome(scheme, ct, server, client, slot_map, fold_spec, lin, share_meter, seed)


def mv_naive(task: MvTask, ct_x: Ciphertext, meter: CostMeter, rng=None) -> MvOutcome:
    """Baseline: one row plaintext + full fold per output (matvec.py:230-264)."""
    p, n = task.params.p, task.params.n
    lin = CostMeter(meter.cost_model)
    outs = []
    for i in range(task.n_o):
        row = np.zeros(n, dtype=np.int64)
        row[: task.n_i] = task.w[i]
        outs.append(_he_fold(he_scmult(ct_x, SlotVector._wrap(row, p), lin), task.n_i, 1, lin))
    meter.merge(lin)
    gen, seed = _resolve_rng(rng)
    share_meter = CostMeter(meter.cost_model)
    server = np.empty(task.n_o, dtype=np.int64)
    client = np.empty(task.n_o, dtype=np.int64)
    for i, ct in enumerate(outs):
        r, masked = gen_additive_share(ct, gen, share_meter)
        server[i] = r.slots[0]
        client[i] = decrypt(masked).slots[0]
    return MvOutcome("naive", outs, SlotVector._wrap(server, p), SlotVector._wrap(client, p), [0] * task.n_o,
                     (1, 1), lin, share_meter, seed)


def mv_diagonal(task: MvTask, ct_xpack: Ciphertext, meter: CostMeter, rng=None) -> MvOutcome:
    """Baseline: n_i hoisted input rotations, no fold (matvec.py:267-282)."""
    lin = CostMeter(meter.cost_model)
    group = he_decperm(ct_xpack, lin) if task.n_i > 1 else None
    acc = None
    for k, d_k in enumerate(_encode_cyclic_diagonals(task)):
        x_rot = ct_xpack if k == 0 else he_hstperm(group, k, lin)
        acc = _acc(acc, he_scmult(x_rot, d_k, lin), lin)
    meter.merge(lin)
    return _finish_single(task, "diagonal", acc, (1, 1), list(range(task.n_o)), lin, rng)


def mv_hybrid_gazelle(task: MvTask, ct_xpack: Ciphertext, meter: CostMeter, rng=None) -> MvOutcome:
    """Baseline: rotated inputs + ciphertext-domain fold (matvec.py:285-302)."""
    lin = CostMeter(meter.cost_model)
    plains = encode_gala_weights(task)
    group = he_decperm(ct_xpack, lin) if task.groups > 1 else None
    acc = None
    for t, p_t in enumerate(plains):
        x_rot = ct_xpack if t == 0 else he_hstperm(group, t, lin)
        acc = _acc(acc, he_scmult(x_rot, rotate_left(p_t, t), lin), lin)
    folded = _he_fold(acc, task.n_i, task.groups, lin)
    meter.merge(lin)
    return _finish_single(task, "gazelle", folded, (1, 1), task.slot_map(), lin, rng)


def _gala_noise(x_noise: float, T: int, params: HEParams) -> float:
    """Mock noise of sum_t perm(scmult(x, p_t), t) in the reference's order."""
    acc = None
    for t in range(T):
        term = x_noise * params.eta_mult
        if t % params.n:
            term = term + params.eta_rot
        acc = term if acc is None else acc + term
    return acc


def book_gala(meter: CostMeter, T: int) -> None:
    meter.sc_mult += T
    meter.full_perm += T - 1
    meter.add += T - 1


def mv_gala(task: MvTask, ct_xpack: Ciphertext, meter: CostMeter, rng=None) -> MvOutcome:
    """GALA dot product, fused on the GPU (matvec.py:305-320 + sharing.py:34-45)."""
    params = task.params
    ctx = ct_xpack.ctx
    lin = CostMeter(meter.cost_model)
    slots = gala_weight_slots(task)
    T = slots.shape[0]
    phys = np.concatenate([slots, slots], axis=1)
    gen, seed = _resolve_rng(rng)
    r = draw_mask(gen, params.p, params.n)
    if ctx.gala_schedule(T) == 2:
        baby, _ = ctx.bsgs_steps(T)
        pts2 = ctx.encode_gala_weights(phys, baby)
        outs, masked_b = ctx.mv_gala2_batch(ct_xpack.data.unsqueeze(0), pts2, T,
                                            ctx.to_device_u32(ctx.physical(r.slots)[None, :]), baby)
        out, masked = outs[0], masked_b[0]
    else:
        out, masked = ctx.mv_gala(ct_xpack.data, ctx.encode_plain(phys), T, ctx.physical(r.slots))
    book_gala(lin, T)
    meter.merge(lin)
    out_noise = _gala_noise(ct_xpack.noise, T, params)
    ct_out = Ciphertext._wrap(out, out_noise, params, ct_xpack.row, ct_xpack.replicated)
    ct_masked = Ciphertext._wrap(masked, out_noise + params.eta0, params, ct_xpack.row, ct_xpack.replicated)
    share_meter = CostMeter(lin.cost_model)
    share_meter.add += 1
    start, end = task.fold_spec()
    slot_map = task.slot_map()
    client = read_slots(fold_ras(decrypt(ct_masked), start, end), slot_map)
    server = read_slots(fold_ras(r, start, end), slot_map)
    return MvOutcome("gala", ct_out, server, client, slot_map, (start, end), lin, share_meter, seed)


MV_RUNNERS = {"naive": mv_naive, "diagonal": mv_diagonal, "gazelle": mv_hybrid_gazelle, "gala": mv_gala}


def run_mv(scheme: str, task: MvTask, x, meter: CostMeter, rng=None) -> MvOutcome:
    """Encrypt x in the layout `scheme` expects and run it (matvec.py:331-337)."""
    if scheme not in MV_RUNNERS:
        raise ParameterError(f"unknown scheme {scheme!r}")
    layout = embed_input if scheme == "naive" else pack_input
    return MV_RUNNERS[scheme](task, encrypt(layout(x, task), task.params), meter, rng)


# ---------------------------------------------------------------------------
# resident-weight layer (throughput form)


class GalaFC:
    """A GALA FC layer with weights encoded once into HBM.

    W (n_out x n_in) is split into logical reference MvTasks: column blocks
    of n (column_blocks) and, per block, row blocks paired on the two
    hypercube rows of one physical ciphertext (both rows share T, hence one
    BSGS schedule).  forward() consumes one encrypted input per column block
    and returns the masked output ciphertexts plus the server's folded shares.
    """

    def __init__(self, w, params: HEParams, pair_rows: bool = True, baby: int | None = None,
                 tensor_cores: bool = True):
        self.params = params
        self.ctx = context(params)
        w = np.asarray(w, dtype=np.int64) % params.p
        n = params.n
        self.n_out, self.n_in = w.shape
        if not (is_power_of_two(self.n_out) and is_power_of_two(self.n_in)):
            raise ParameterError("layer dims must be powers of two (pad first)")
        self.n_cb = max(1, self.n_in // n)
        cb_w = min(self.n_in, n)
        # row split: two halves when each half is still a valid MvTask
        half = self.n_out // 2
        self.paired = pair_rows and half >= 1 and half <= cb_w and self.n_out >= 2
        rows = [(0, half), (half, self.n_out)] if self.paired else [(0, self.n_out)]
        if not self.paired and self.n_out > cb_w:
            raise ParameterError("n_out exceeds the column-block width; use pair_rows=True")
        self.blocks = []  # per column block: (tasks, pts tensor, T)
        for b in range(self.n_cb):
            wb = w[:, b * cb_w:(b + 1) * cb_w]
            tasks = [MvTask(cb_w, hi - lo, wb[lo:hi], params) for lo, hi in rows]
            s0 = gala_weight_slots(tasks[0])
            s1 = gala_weight_slots(tasks[1]) if self.paired else s0
            if s0.shape != s1.shape:
                raise ParameterError("paired row blocks must share T")
            self.blocks.append([tasks, np.concatenate([s0, s1], axis=1), s0.shape[0]])
        self.T = self.blocks[0][2]
        self.schedule = self.ctx.gala_schedule(self.T)
        if baby is None and self.schedule == 2:
            baby = self.ctx.gala2_baby(self.T)
        self.baby, self.steps = self.ctx.bsgs_steps(self.T, baby)
        for blk in self.blocks:    # resident encoded weights, in the layout of the chosen schedule
            blk[1] = (self.ctx.encode_gala_weights(blk[1], self.baby) if self.schedule == 2
                      else self.ctx.encode_plain(blk[1]))
        self.ctx.ensure_keys(self.steps)
        # tensor-core baby-step sums (schedule 2): the weights with the baby-step rotation keys folded in
        # (gala_fc_tc_weights), per block -- after the keys exist
        self.wcan = [None] * len(self.blocks)
        if tensor_cores and self.schedule == 2 and self.ctx.fc_tc_supported(self.T, self.baby):
            self.wcan = [self.ctx.fc_tc_weights(blk[1], self.T, self.baby) for blk in self.blocks]

    def encrypt_input(self, x) -> list:
        """Client side: one physical ciphertext per column block."""
        x = np.asarray(x, dtype=np.int64)
        cts = []
        for b, (tasks, _, _) in enumerate(self.blocks):
            xs = pack_input(x[b * tasks[0].n_i:(b + 1) * tasks[0].n_i], tasks[0]).slots
            cts.append(self.ctx.encrypt_physical(self.ctx.physical(xs)))
        return cts

    def draw_masks(self, rng) -> list:
        gen = np.random.default_rng(rng)
        out = []
        for tasks, _, _ in self.blocks:
            rs = [draw_mask(gen, self.params.p, self.params.n) for _ in tasks]
            out.append(rs)
        return out

    def forward_device(self, cts, masks) -> list:
        """Server side, device only: masked output ciphertexts (one per block)."""
        outs = []
        for bidx, ((tasks, pts, T), ct, rs) in enumerate(zip(self.blocks, cts, masks)):
            phys_r = self.ctx.physical(rs[0].slots, rs[1].slots if self.paired else None)
            _, masked = self.run_batch(ct.unsqueeze(0), pts, self.ctx.to_device_u32(phys_r[None, :]), block=bidx)
            outs.append(masked[0])
        return outs

    def run_batch(self, cts, pts, d_r, outs=None, masked=None, block: int | None = None):
        """Fused layer over a batch of inputs (cts [B][2][L][N], d_r [B][N]) for one column block."""
        if self.schedule == 2:
            if block is None:   # locate the block by its weights tensor
                block = next((i for i, b in enumerate(self.blocks) if b[1] is pts), None)
            wcan = self.wcan[block] if block is not None else None
            return self.ctx.mv_gala2_batch(cts, pts, self.T, d_r, self.baby, outs=outs, masked=masked, wcan=wcan)
        return self.ctx.mv_gala_batch(cts, pts, self.T, d_r, self.baby, outs=outs, masked=masked)

    def server_shares(self, masks) -> np.ndarray:
        res = np.zeros(self.n_out, dtype=np.int64)
        for (tasks, _, _), rs in zip(self.blocks, masks):
            parts = [read_slots(fold_ras(r, *t.fold_spec()), t.slot_map()).slots for t, r in zip(tasks, rs)]
            res = (res + np.concatenate(parts)) % self.params.p
        return res

    def client_shares(self, masked_cts) -> np.ndarray:
        res = np.zeros(self.n_out, dtype=np.int64)
        n = self.params.n
        for (tasks, _, _), ct in zip(self.blocks, masked_cts):
            full = self.ctx.decrypt_physical(ct)
            parts = []
            for row, t in enumerate(tasks):
                v = SlotVector._wrap(full[row * n:(row + 1) * n].copy(), self.params.p)
                parts.append(read_slots(fold_ras(v, *t.fold_spec()), t.slot_map()).slots)
            res = (res + np.concatenate(parts)) % self.params.p
        return res

    def book(self, meter: CostMeter) -> None:
        for tasks, _, T in self.blocks:
            for _ in tasks:
                book_gala(meter, T)
