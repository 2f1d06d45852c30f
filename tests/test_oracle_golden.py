"""Pin the CPU BFV oracle to the reference package (no GPU needed).

The golden fixtures (tests/golden/*.npz) were produced by running the
reference `gala` package (mock backend) -- see tests/golden/make_golden.py.
The oracle must decrypt every fused schedule to exactly the reference's
payloads, and its op-level semantics must match the reference ops.
"""
import os

import numpy as np
import pytest

from oracle.bfv import Oracle, bsgs_baby
from oracle.plain import conv2d_mod_p, dot_mod_p
from paper_2105_01827_b200 import sampling
from paper_2105_01827_b200.backend import HEParams
from paper_2105_01827_b200.conv import ConvTask, DiagonalPlan, encode_channel_blocks
from paper_2105_01827_b200.matvec import MvTask, gala_weight_slots, pack_input

GOLD = os.path.join(os.path.dirname(__file__), "golden")
P = 1032193


def load(name):
    return np.load(os.path.join(GOLD, name))


def twin_oracle(n, L=None, seed=3):
    params = HEParams(n=n, p=P, rns_limbs=L)
    bfv = params.bfv()
    o = Oracle(bfv)
    rng = np.random.default_rng(seed)
    o.set_secret(sampling.secret(rng, bfv.N))
    return params, bfv, o, rng


def add_keys(o, bfv, rng, steps):
    for s in sorted(set(int(x) % bfv.n for x in steps) - {0}):
        a, e = sampling.rotation_key_randomness(rng, bfv)
        o.gen_rotkey(s, a, e)


def enc(o, bfv, rng, phys):
    a, e = sampling.encryption_randomness(rng, bfv)
    return o.encrypt(phys, a, e)


MV = load("mv_gala.npz")
MV_CASES = list(range(int(MV["count"][0])))


@pytest.mark.parametrize("schedule", [1, 2])
@pytest.mark.parametrize("idx", MV_CASES)
def test_oracle_mv_gala_matches_reference_payload(idx, schedule):
    """Both oracle schedules (1: per-term key switches, as the reference; 2: digits hoisted across the
    plaintext product, deferred c0 ModDown) decrypt to the reference's payload and shares."""
    n, n_o, n_i, seed, rseed = (int(v) for v in MV[f"c{idx}_dims"])
    if n > 1024 and idx % 2:
        pytest.skip("large cases: every other one on CPU")
    params, bfv, o, rng = twin_oracle(n)
    w = MV[f"c{idx}_w"].astype(np.int64) % P
    x = MV[f"c{idx}_x"].astype(np.int64)
    task = MvTask(n_i, n_o, w, params)
    slots = gala_weight_slots(task)
    T = slots.shape[0]
    b = bsgs_baby(T)
    add_keys(o, bfv, rng, list(range(1, b)) + [g * b for g in range(1, T // b)])
    xs = pack_input(x, task).slots
    ct = enc(o, bfv, rng, np.concatenate([xs, xs]).astype(np.uint32))
    r = np.random.default_rng(rseed).integers(0, P, n, dtype=np.int64)
    out, masked = o.mv_gala(ct, np.concatenate([slots, slots], axis=1).astype(np.uint32),
                            np.concatenate([r, r]).astype(np.uint32), schedule=schedule)
    dec = o.decrypt(out).astype(np.int64)
    assert np.array_equal(dec[:n], MV[f"c{idx}_payload"].astype(np.int64))
    assert np.array_equal(dec[n:], MV[f"c{idx}_payload"].astype(np.int64))
    # shares: client = fold(decrypt(masked)), server = fold(r); reference shares reproduce exactly
    from paper_2105_01827_b200.ring import SlotVector, fold_ras, read_slots

    dm = o.decrypt(masked).astype(np.int64)[:n]
    client = read_slots(fold_ras(SlotVector(dm, P), *task.fold_spec()), task.slot_map()).slots
    server = read_slots(fold_ras(SlotVector(r, P), *task.fold_spec()), task.slot_map()).slots
    assert np.array_equal(client, MV[f"c{idx}_client"].astype(np.int64))
    assert np.array_equal(server, MV[f"c{idx}_server"].astype(np.int64))
    assert np.array_equal((client + server) % P, dot_mod_p(w, x, P))


CV = load("conv_kg.npz")
CONV_CASES = list(range(int(CV["count"][0])))


@pytest.mark.parametrize("idx", CONV_CASES)
def test_oracle_conv_kg_matches_reference_payload(idx):
    u, c_i, k, c_o, n, seed = (int(v) for v in CV[f"c{idx}_dims"])
    params, bfv, o, rng = twin_oracle(n)
    kern = CV[f"c{idx}_kernels"].astype(np.int64) % P
    ch = CV[f"c{idx}_channels"].astype(np.int64)
    task = ConvTask(u, u, c_i, k, k, c_o, kern, params)
    c_n = task.channels_per_ct
    n_ib, n_ob = c_i // c_n, c_o // c_n
    n_obp = (n_ob + 1) // 2
    plan = DiagonalPlan(task, c_n)
    kk = k * k
    pts = np.zeros((n_obp, n_ib, c_n, kk, 2 * n), np.uint32)
    for ob in range(n_ob):
        row = ob % 2
        for ib in range(n_ib):
            for d in range(c_n):
                pts[ob // 2, ib, d, :, row * n:(row + 1) * n] = plan.coef_slots(ob, ib, d)
    steps = [rot for _, _, rot in task.offsets()]
    B = u * u
    add_keys(o, bfv, rng, steps + [d * B for d in range(1, c_n)])
    cts = np.stack([enc(o, bfv, rng, np.concatenate([v.slots, v.slots]).astype(np.uint32))
                    for v in encode_channel_blocks(task, ch)])
    outs = o.conv_kg(cts, pts, steps, B)
    want = CV[f"c{idx}_payloads"].astype(np.int64)
    for ob in range(n_ob):
        d = o.decrypt(outs[ob // 2]).astype(np.int64)
        row = ob % 2
        assert np.array_equal(d[row * n:(row + 1) * n], want[ob]), ob
    full = np.concatenate([want[ob].reshape(c_n, u, u) for ob in range(n_ob)])
    assert np.array_equal(full, conv2d_mod_p(ch, kern, P))


def test_oracle_ops_match_reference_ops():
    ops = load("ops.npz")
    params, bfv, o, rng = twin_oracle(64)
    x, y = ops["x"].astype(np.int64), ops["y"].astype(np.int64)
    phys = lambda v: np.concatenate([v, v]).astype(np.uint32)  # noqa: E731
    ct = enc(o, bfv, rng, phys(x))
    add_keys(o, bfv, rng, [1, 5, 17, 63])
    for k in (1, 5, 17, 63):
        assert np.array_equal(o.decrypt(o.rotate(ct, k))[:64].astype(np.int64), ops[f"rot{k}"])
    assert np.array_equal(o.decrypt(o.scmult(ct, phys(y)))[:64].astype(np.int64), ops["scmult"])
    assert np.array_equal(o.decrypt(o.add(ct, enc(o, bfv, rng, phys(y))))[:64].astype(np.int64), ops["add"])
    assert np.array_equal(o.decrypt(o.sub_plain(ct, phys(y)))[:64].astype(np.int64), ops["sub"])


@pytest.mark.parametrize("n,L", [(4, 1), (64, 1), (64, 2), (1024, 3), (4096, 3)])
def test_oracle_ntt_roundtrip_and_encoding(n, L):
    params, bfv, o, rng = twin_oracle(n, L)
    for idx in list(range(bfv.L + 1)) + [-1]:
        q = bfv.all_primes[idx] if idx >= 0 else bfv.p
        a = rng.integers(0, q, bfv.N, dtype=np.uint64)
        assert np.array_equal(o.ntt(o.ntt(a, idx), idx, inverse=True), a)
    s = rng.integers(0, P, bfv.N).astype(np.uint32)
    assert np.array_equal(o.decode_p(o.encode_p(s)), s)


def test_oracle_rotation_is_rowwise_rotate_left():
    params, bfv, o, rng = twin_oracle(32, 2)
    x = rng.integers(0, P, 64).astype(np.uint32)
    ct = enc(o, bfv, rng, x)
    add_keys(o, bfv, rng, [1, 7, 31])
    outs = o.rotate_hoisted(ct, [1, 7, 31])
    xs = x.astype(np.int64)
    for k, oc in zip([1, 7, 31], outs):
        want = np.concatenate([np.roll(xs[:32], -k), np.roll(xs[32:], -k)])
        assert np.array_equal(o.decrypt(oc).astype(np.int64), want)
        assert np.array_equal(o.rotate(ct, k), oc)   # DecPerm+HstPerm == full Perm, word for word


def test_oracle_linearity_and_noise_margin_cfg3_shape():
    """Real noise stays under Delta/2 at the single-prime N=4096 conv shape (cfg3)."""
    import os as _os

    idx = [i for i in CONV_CASES if int(CV[f"c{i}_dims"][4]) == 2048][0]
    u, c_i, k, c_o, n, seed = (int(v) for v in CV[f"c{idx}_dims"])
    assert (u, c_i, c_o, n) == (16, 64, 64, 2048)
    # the full decryption check of this case runs in test_oracle_conv_kg_matches_reference_payload;
    # here: the margin of the single-prime parameter set
    bfv = HEParams(n=2048, p=P, rns_limbs=1).bfv()
    assert bfv.L == 1 and bfv.primes[0] % (2 * bfv.N * P) == 1 and bfv.log2_budget() > 40.9
