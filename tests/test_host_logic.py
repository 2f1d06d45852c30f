"""Host-side logic of the drop-in API (no GPU): layouts, encodings, meters,
noise recurrences, parameter derivation, ring semantics.  Known-answer
vectors follow the reference's own tests (pkg/tests/test_matvec.py,
test_conv.py, test_ring.py, test_analytics.py)."""
import json

import numpy as np
import pytest

from paper_2105_01827_b200 import params as bp
from paper_2105_01827_b200.analytics import OpCounts, count_conv, count_mv, physical_mv_counts, predict_noise
from paper_2105_01827_b200.backend import CostMeter, CostModel, HEParams, load_cost_config, with_overrides
from paper_2105_01827_b200.conv import ConvTask, DiagonalPlan, _kg_book_and_noise, build_offset_masks
from paper_2105_01827_b200.errors import DimensionError, ParameterError
from paper_2105_01827_b200.matvec import (
    MvTask,
    _gala_noise,
    book_gala,
    column_blocks,
    encode_gala_weights,
    gala_weight_slots,
    pack_input,
)
from paper_2105_01827_b200.ring import SlotVector, fold_ras, negate, pointwise, read_slots, rotate_left

P = 1032193
PARAMS = HEParams()


def test_default_params_batch():
    assert PARAMS.p == P and PARAMS.n == 2048
    b = PARAMS.bfv()
    assert b.N == 4096 and b.L == 2 and (P - 1) % (2 * b.N) == 0
    assert all(q < 2**60 for q in b.primes) and b.special < 2**60
    one = HEParams(rns_limbs=1).bfv()          # configs 1 and 3: a single 62-bit prime, q = 1 mod 2N p
    assert one.L == 1 and one.primes[0] % (2 * one.N * P) == 1 and one.primes[0] < 2**62 and one.special < 2**62
    assert with_overrides(PARAMS, n=4096).bfv().L == 3


def test_params_reject_nonbatching_p():
    with pytest.raises(ParameterError):
        HEParams(p=1048573).bfv()  # the reference default is not 1 mod 2N
    with pytest.raises(ParameterError):
        HEParams(n=100)
    with pytest.raises(ParameterError):
        HEParams(p=1048575)
    with pytest.raises(ParameterError):
        HEParams(eta_rot=1.0)
    with pytest.raises(ParameterError):
        HEParams(noise_budget=1.0)
    assert HEParams().noise_budget == pytest.approx(2**59 / P)


@pytest.mark.parametrize("N", [8, 64, 4096, 8192])
def test_primes_and_roots(N):
    for L in (1, 3):
        b = bp.derive(N // 2, P, L)
        for m, psi in zip(b.all_primes, b.psis):
            assert bp.is_prime(m) and (m - 1) % (2 * N) == 0
            assert pow(psi, N, m) == m - 1
        assert pow(b.psi_p, N, P) == P - 1
        assert len(set(b.all_primes)) == L + 1


def test_galois_element_is_rotation_generator():
    N = 64
    g = bp.galois_element(1, N)
    assert g == 3 and bp.galois_element(N // 2, N) == 1 and bp.galois_element(-1, N) == pow(3, N // 2 - 1, 2 * N)


# --- layouts / encodings (reference KATs) ---------------------------------------
def test_encode_small_square_case():
    params = with_overrides(PARAMS, n=4)
    task = MvTask(4, 2, np.array([[11, 12, 13, 14], [21, 22, 23, 24]]), params)
    p0, p1 = encode_gala_weights(task)
    assert p0.tolist() == [11, 22, 13, 24]
    assert p1.tolist() == [21, 12, 23, 14]


def test_encode_two_copies():
    task = MvTask(2, 2, np.array([[1, 2], [3, 4]]), with_overrides(PARAMS, n=4))
    (p0,) = encode_gala_weights(task)
    assert p0.tolist() == [1, 2, 3, 4]
    assert task.slot_map() == [0, 2]


@pytest.mark.parametrize("n,n_o,n_i", [(2048, 16, 128), (256, 16, 128), (256, 8, 256), (2048, 4, 16)])
def test_exact_cover(n, n_o, n_i):
    params = with_overrides(PARAMS, n=n)
    rng = np.random.default_rng(5)
    task = MvTask(n_i, n_o, rng.integers(0, P, (n_o, n_i)), params)
    plains = gala_weight_slots(task)
    T = task.groups
    w = task.padded_matrix()
    for j0 in range(n_o):
        base = (j0 // T) * n_i + (j0 % T)
        cols = []
        for kk in range(n_i // T):
            j = base + kk * T
            for t in range(T):
                col = (j + t) % n_i
                cols.append(col)
                assert plains[t][(j + t) % n] == w[j0][col]
        assert sorted(cols) == list(range(n_i))


def test_slot_map_padded_case_and_validation():
    task = MvTask(16, 4, np.zeros((4, 16)), PARAMS)
    assert task.n_o_padded == 128 and task.groups == 1 and task.slot_map() == [0, 16, 32, 48]
    with pytest.raises(ParameterError):
        MvTask(3, 2, np.zeros((2, 3)), PARAMS)
    with pytest.raises(ParameterError):
        MvTask(16, 32, np.zeros((32, 16)), PARAMS)
    with pytest.raises(ParameterError):
        MvTask(4096, 1, np.zeros((1, 4096)), PARAMS)
    with pytest.raises(DimensionError):
        MvTask(16, 4, np.zeros((4, 8)), PARAMS)


def test_pack_and_column_blocks():
    task = MvTask(16, 4, np.zeros((4, 16)), PARAMS)
    x = np.arange(16)
    packed = pack_input(x, task)
    assert packed.slots[:16].tolist() == packed.slots[16:32].tolist()
    rng = np.random.default_rng(17)
    w = rng.integers(0, P, (2, 1024))
    xx = rng.integers(0, P, 1024)
    blocks = list(column_blocks(w, xx, 256))
    assert len(blocks) == 4
    with pytest.raises(ParameterError):
        list(column_blocks(w[:, :1000], xx[:1000], 256))


# --- conv host logic ----------------------------------------------------------------
def test_offset_masks_kats():
    params = with_overrides(PARAMS, n=16)
    k = np.arange(1, 10).reshape(1, 1, 3, 3)
    task = ConvTask(3, 3, 1, 3, 3, 1, k, params)
    masks = build_offset_masks(task, task.kernels[0, 0])
    m = next(m for m in masks if m.offset == (1, 1))
    board = m.mask.slots[:9].reshape(3, 3)
    assert not board[2].any() and not board[:, 2].any() and board[:2, :2].all() and m.rotation == 4
    center = next(m for m in masks if m.offset == (0, 0))
    assert all(v == 5 for v in center.mask.slots[:9])


def test_diagonal_plan_band_layout():
    params = with_overrides(PARAMS, n=64)
    rng = np.random.default_rng(3)
    kern = rng.integers(0, P, (8, 8, 3, 3))
    task = ConvTask(4, 4, 8, 3, 3, 8, kern, params)
    plan = DiagonalPlan(task, 4)
    sl = plan.coef_slots(1, 0, 2)            # [k][n]
    for ch in range(4):
        o = 1 * 4 + (ch - 2) % 4
        i = 0 * 4 + ch
        # centre tap (index 4) is valid everywhere in the band
        assert np.all(sl[4, ch * 16:(ch + 1) * 16] == kern[o, i, 1, 1] % P)


def test_kg_bookkeeping_matches_analytics():
    for (u, c_i, k, c_o, n) in [(4, 4, 1, 4, 64), (4, 8, 3, 8, 64), (4, 8, 3, 8, 128), (16, 64, 3, 64, 2048)]:
        params = with_overrides(PARAMS, n=n)
        task = ConvTask(u, u, c_i, k, k, c_o, np.zeros((c_o, c_i, k, k)), params)
        c_n = task.channels_per_ct
        meter = CostMeter()
        noises = _kg_book_and_noise(task, [params.eta0] * (c_i // c_n), c_n, c_i // c_n, c_o // c_n, meter)
        assert OpCounts.from_meter(meter) == count_conv("gala", u, u, c_i, c_o, k, k, n)
        eta = predict_noise("conv_gala", (u, u, c_i, c_o, k, k), params)
        assert all(v == eta for v in noises)


def test_gala_bookkeeping_matches_analytics():
    for n in (2048, 256):
        params = with_overrides(PARAMS, n=n)
        for n_o, n_i in [(1, 2048), (2, 1024), (16, 128), (8, 256), (4, 16)]:
            if n_i > n:
                continue
            task = MvTask(n_i, n_o, np.zeros((n_o, n_i)), params)
            meter = CostMeter()
            book_gala(meter, task.groups)
            assert OpCounts.from_meter(meter) == count_mv("gala", n_i, n_o, n)
            assert _gala_noise(params.eta0, task.groups, params) == predict_noise("mv_gala", (n_i, n_o), params)
    assert predict_noise("mv_gala", (2048, 2), PARAMS) == 2 * 8.0 * 1024.0 + 2048.0


def test_table_v_counts():
    assert count_mv("gala", 2048, 1, 2048) == OpCounts(sc_mult=1)
    assert count_mv("gazelle", 2048, 1, 2048) == OpCounts(perm=11, sc_mult=1, add=11)
    assert count_mv("gazelle", 128, 16, 2048) == OpCounts(perm=7, sc_mult=1, add=7)
    assert count_conv("gala", 16, 16, 128, 128, 3, 3, 2048).paired() == OpCounts(
        0, 128, 240, 18432, 18416, "paired")


def test_physical_work_model():
    w = physical_mv_counts(8192, 3, 512, 32)
    assert w["rotations"] == 511 and w["moddowns"] == 17 and w["modmuls"] > 4e8
    # schedule 2 as executed (b = 64, G = 8): 7 one-component inner ModDowns (the giant groups' c1)
    # + one final two-component ModDown = 9 ModDown components, not 9 two-component ModDowns
    w2 = physical_mv_counts(8192, 3, 512, 64, schedule=2)
    assert w2["moddown_components"] == 9 and w2["moddowns"] == 8
    h = 8192 // 2 * 13
    one = 4 * h + 3 * 8192
    decomp, giant = (3 + 9) * h, 7 * ((3 + 9) * h + 2 * 3 * 4 * 8192)
    baby = 63 * 2 * 3 * 4 * 8192 + 8 * 63 * (2 * 4 * 8192 + 3 * 8192) + 8 * 2 * 3 * 8192
    mask = h + 3 * h + 3 * 8192
    assert w2["modmuls"] == decomp + baby + giant + 9 * one + mask


# --- meters / config -----------------------------------------------------------------
def test_meter_views_and_merge():
    meter = CostMeter()
    meter.full_perm, meter.dec_perm, meter.hst_perm, meter.sc_mult, meter.add = 2, 1, 3, 4, 5
    m = meter.cost_model
    assert meter.estimated_ms() == pytest.approx(2 * m.t_perm + m.t_decperm + 3 * m.t_hstperm + 4 * m.t_scmult
                                                 + 5 * m.t_add)
    paired = meter.as_dict("paired")
    assert paired["perm"] == 0 and paired["dec_perm"] == 3 and paired["hst_perm"] == 5
    other = CostMeter()
    other.add = 10
    other.merge(meter)
    assert other.add == 15 and other.full_perm == 2
    with pytest.raises(ParameterError):
        meter.as_dict("bogus")
    c = CostModel()
    assert 50 <= c.t_perm / c.t_add <= 60 and 30 <= c.t_perm / c.t_scmult <= 38


def test_load_cost_config(tmp_path):
    cfg = tmp_path / "cost.json"
    cfg.write_text(json.dumps({"t_perm": 0.2, "eta0": 4.0, "n": 1024, "rns_limbs": 3}))
    params, model = load_cost_config(cfg)
    assert params.n == 1024 and params.eta0 == 4.0 and params.rns_limbs == 3 and model.t_perm == 0.2
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"t_perm": 0.2, "bogus": 1}))
    with pytest.raises(ParameterError):
        load_cost_config(bad)


# --- ring semantics (reference ring.py) --------------------------------------------
def test_ring_semantics():
    v = SlotVector(np.arange(8), 7)
    assert rotate_left(v, 3).tolist() == [3, 4, 5, 6, 0, 0, 1, 2]   # result[j] = v[(j + 3) mod 8]
    assert rotate_left(v, 8) is v
    assert pointwise(v, v, "add").tolist() == [(2 * i) % 7 for i in range(8)]
    with pytest.raises(ParameterError):
        pointwise(v, v, "sub")
    with pytest.raises(DimensionError):
        pointwise(v, SlotVector(np.arange(4), 7), "add")
    with pytest.raises(DimensionError):
        SlotVector(np.arange(6), 7)
    assert read_slots(v, [0, 2, 5, 7]).tolist() == [0, 2, 5, 0]
    with pytest.raises(DimensionError):
        read_slots(v, [0, 8])


def test_fold_linearity():
    rng = np.random.default_rng(6)
    for _ in range(20):
        m = SlotVector(rng.integers(0, P, 32), P)
        r = SlotVector(rng.integers(0, P, 32), P)
        masked = pointwise(m, negate(r), "add")
        lhs = pointwise(fold_ras(masked, 8, 2), fold_ras(r, 8, 2), "add")
        assert lhs == fold_ras(m, 8, 2)
    with pytest.raises(ParameterError):
        fold_ras(SlotVector(np.zeros(8), P), 16, 1)


@pytest.mark.parametrize("n,u,c_o,c_i,pair", [(64, 4, 12, 8, 2), (64, 4, 8, 8, 1), (256, 16, 3, 2, 2)])
def test_kg2_coefficients_factor_the_convolution(n, u, c_o, c_i, pair):
    """Band masks x int8 coefficient matrix, evaluated on slot vectors, is the convolution (mod p)."""
    from oracle.plain import conv2d_mod_p
    from paper_2105_01827_b200.backend import HEParams
    from paper_2105_01827_b200.conv import ConvTask, kg2_coefficients

    P = 1032193
    rng = np.random.default_rng(1)
    kern = rng.integers(-128, 128, (c_o, c_i, 3, 3))
    t = ConvTask(u, u, c_i, 3, 3, c_o, kern, HEParams(n=n, p=P))
    c_n, B = n // (u * u), u * u
    nb = pair * c_n
    A, rowsum, K = kg2_coefficients(t, c_n, pair)
    assert A.shape[1] % 16 == 0 and K == (c_i // c_n) * 9 * nb
    assert np.array_equal(rowsum, A.astype(np.int64).sum(axis=1))
    x = rng.integers(0, P, (c_i, u, u))
    phys = [np.concatenate([b, b]) for b in x.reshape(c_i // c_n, -1)]

    def rot(v, s):
        return np.concatenate([np.roll(v[:n], -s), np.roll(v[n:], -s)])

    s = np.arange(2 * n)
    row, cs = s // n, s % n
    ch, pos = cs // B, cs % B
    yy, xx = pos // u, pos % u
    band = row * c_n + ch if pair == 2 else ch
    out = []
    for o in range(A.shape[0] // c_n):
        tot = np.zeros(2 * n, np.int64)
        for d in range(c_n):
            acc = np.zeros(2 * n, np.int64)
            for ib, v in enumerate(phys):
                for ti, (dw, dh, r) in enumerate(t.offsets()):
                    R = rot(v, r)
                    ok = (xx + dw >= 0) & (xx + dw < u) & (yy + dh >= 0) & (yy + dh < u)
                    for beta in range(nb):
                        m = ((band == beta) & ok).astype(np.int64)
                        acc = (acc + int(A[o * c_n + d, (ib * 9 + ti) * nb + beta]) * R * m) % P
            tot = (tot + rot(acc, d * B)) % P
        out.append(tot)
    want = conv2d_mod_p(x, kern, P).reshape(c_o // c_n, -1)
    for ob in range(c_o // c_n):
        r = ob % pair if pair == 2 else 0
        assert np.array_equal(out[ob // pair][r * n:(r + 1) * n], want[ob])


def test_kg2_post_coefficients_are_a_column_regrouping():
    """Post-mask matrix [(m, beta)][(ib, tap)] holds exactly the pre-mask entries A[m][(ib, tap, beta)]."""
    from paper_2105_01827_b200.backend import HEParams
    from paper_2105_01827_b200.conv import ConvTask, kg2_coefficients, kg2_post_coefficients

    rng = np.random.default_rng(4)
    n, u, c_i, c_o = 64, 4, 8, 12
    t = ConvTask(u, u, c_i, 3, 3, c_o, rng.integers(-128, 128, (c_o, c_i, 3, 3)), HEParams(n=n, p=1032193))
    c_n = n // (u * u)
    for pair in (1, 2):
        nb = pair * c_n
        A, _, K = kg2_coefficients(t, c_n, pair)
        B, rs = kg2_post_coefficients(A, K, nb)
        Kq = K // nb
        assert B.shape == (A.shape[0] * nb, (Kq + 31) // 32 * 32)
        assert np.array_equal(rs, B.astype(np.int64).sum(axis=1))
        for m in range(A.shape[0]):
            for beta in range(nb):
                assert np.array_equal(B[m * nb + beta, :Kq], A[m, beta:K:nb])
        assert not B[:, Kq:].any()


def test_kg_schedule_selection():
    """Schedule 2 needs L >= 2, int8 kernels and c_n <= KG2_MAX_CN; otherwise schedule 1."""
    from paper_2105_01827_b200.backend import HEParams
    from paper_2105_01827_b200.conv import KG2_MAX_CN, ConvTask, kg_schedule

    p = 1032193
    params = HEParams(n=64, p=p)
    small = ConvTask(8, 8, 2, 3, 3, 2, np.ones((2, 2, 3, 3), dtype=np.int64), params)
    assert kg_schedule(small, 1, 3) == 2
    assert kg_schedule(small, 1, 1) == 1                       # one 62-bit prime: noise budget
    assert kg_schedule(small, KG2_MAX_CN * 2, 3) == 1          # too many bands
    big = ConvTask(8, 8, 2, 3, 3, 2, np.full((2, 2, 3, 3), 300, dtype=np.int64), params)
    assert kg_schedule(big, 1, 3) == 1                         # not int8 after centring
    neg = ConvTask(8, 8, 2, 3, 3, 2, np.full((2, 2, 3, 3), p - 128, dtype=np.int64), params)
    assert kg_schedule(neg, 1, 3) == 2                         # -128 mod p centres into int8


def test_system_rng_samplers():
    """Default (seed=None) contexts draw secrets, keys and encryption randomness from the OS CSPRNG:
    the samplers' ranges and moments hold, and two draws differ."""
    from paper_2105_01827_b200 import sampling

    g = sampling.SystemRng()
    assert HEParams().seed is None
    s = sampling.secret(g, 1 << 14)
    assert set(np.unique(s).tolist()) == {-1, 0, 1}
    assert abs(float(np.mean(s == 0)) - 1 / 3) < 0.03
    q = (1 << 60) - 93
    u = sampling.uniform(g, [q, 1032193], 4096)
    assert u.dtype == np.uint64 and u.shape == (2, 4096)
    assert int(u[0].max()) < q and int(u[1].max()) < 1032193
    assert abs(float(u[1].astype(np.float64).mean()) / 1032193 - 0.5) < 0.03
    e = sampling.gaussian(g, 1 << 15, 3.2)
    assert abs(float(e.std()) - 3.2) < 0.15 and abs(float(e.mean())) < 0.15 and int(np.abs(e).max()) <= 20
    assert not np.array_equal(sampling.secret(g, 256), sampling.secret(g, 256))
    # the seeded (insecure, reproducible) stream stays available for word-parity tests
    a = sampling.secret(np.random.default_rng([5, 0]), 64)
    assert np.array_equal(a, sampling.secret(np.random.default_rng([5, 0]), 64))


def test_kg_plan_is_taken_from_the_full_task():
    """Schedule / mask form / first-Add engine come from the full layer: a shard whose kernels alone
    fit int8 still follows the full layer's schedule (sharding.ShardedKernelGroupingConv)."""
    from paper_2105_01827_b200.conv import kg_plan, kg_schedule
    from paper_2105_01827_b200.sharding import shard_range, sub_conv_task

    params = HEParams(n=1024, rns_limbs=3)
    rng = np.random.default_rng(5)
    kern = rng.integers(-128, 128, (24, 8, 3, 3))
    kern[0, 0, 0, 0] = 5000
    task = ConvTask(32, 32, 8, 3, 3, 24, kern % P, params)
    assert kg_plan(task, 2, 3, 2048).schedule == 1
    sub = sub_conv_task(task, shard_range(12, 2, 1), 2)
    assert kg_schedule(sub, 1, 3) == 2
    p2 = kg_plan(ConvTask(32, 32, 8, 3, 3, 24, rng.integers(-128, 128, (24, 8, 3, 3)) % P, params), 2, 3, 2048,
                 band_only=True)
    assert (p2.schedule, p2.post, p2.batchable) == (2, True, True)


# --- network files (reference layer-list format, profiler.py:9-17, 61-88) -------------------------
def test_parse_network_format_and_errors():
    from paper_2105_01827_b200.errors import NetworkParseError
    from paper_2105_01827_b200.netfile import parse_network

    assert parse_network("") == [] and parse_network("# only a comment\n\n") == []
    specs = parse_network("conv 8 8 4 3 3 16  # a conv\nnonlinear relu\nfc 128 10\n")
    assert [s.kind for s in specs] == ["conv", "nonlinear", "fc"]
    assert (specs[0].u_w, specs[0].c_i, specs[0].k_h, specs[0].c_o) == (8, 4, 3, 16)
    assert (specs[2].n_i, specs[2].n_o) == (128, 10) and specs[1].label == "relu"
    for bad, line in (("conv 8 8 4 3 3\n", 1), ("fc 1 2\npool 2\n", 2), ("\nfc x 2\n", 2), ("conv 0 8 4 3 3 16", 1)):
        with pytest.raises(NetworkParseError) as e:
            parse_network(bad)
        assert e.value.line_no == line


def test_resnet18_224_network_file_is_the_config5_layer_list():
    from paper_2105_01827_b200.netfile import fc_padded, load_network, network_layers
    from paper_2105_01827_b200.resnet import resnet18_224

    got = network_layers(load_network("resnet18_224.net"))
    want = resnet18_224()
    assert [(s.kind, s.c_in, s.c_out, s.k, s.stride, s.size) for s in got] == \
           [(s.kind, s.c_in, s.c_out, s.k, s.stride, s.size) for s in want]
    assert fc_padded(512, 1000, 4096) == (1024, 1024)          # profiler._fc_padded
    assert fc_padded(24, 40, 4096) == (64, 64)
    with pytest.raises(ParameterError):
        fc_padded(8, 5000, 4096)


@pytest.mark.skipif(not __import__("os").path.isdir("/root/reference/pkg/src/gala"),
                    reason="reference not mounted (it is only present in the build container)")
def test_network_file_parses_identically_with_the_reference_parser():
    import sys

    from paper_2105_01827_b200.netfile import NETWORKS, parse_network

    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from gala.profiler import parse_network as ref_parse
    finally:
        sys.path.pop(0)
        for m in [m for m in sys.modules if m == "gala" or m.startswith("gala.")]:
            del sys.modules[m]
    text = open(f"{NETWORKS}/resnet18_224.net").read()
    ours, ref = parse_network(text), ref_parse(text)
    assert [(s.kind, s.u_w, s.u_h, s.c_i, s.k_w, s.k_h, s.c_o, s.n_i, s.n_o, s.label) for s in ours] == \
           [(s.kind, s.u_w, s.u_h, s.c_i, s.k_w, s.k_h, s.c_o, s.n_i, s.n_o, s.label) for s in ref]
