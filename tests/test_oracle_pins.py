"""Pins for the oracle: each check ties oracle/ to something
other than itself -- values the paper prints, closed forms, invariants, exact integer
brute force, and library special cases -- so that a dropped term, wrong sign or
index, or transposed operand anywhere in oracle/ fails at least one of them.
All CPU-only (no GPU marker)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kv(path):
    out = {}
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = line.split("=", 1)
        out[k] = v
    return out


def _nums(s):
    return [float(t) for t in s.split()]


def _rand_problem(seed, H_in=24, H_out=20, S=7, max_len=4, max_rank=9, n_ad=4, p_none=0.15):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len + 1, size=S)
    ip = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = np.array([int(rng.integers(0, n_ad)) if rng.random() > p_none else -1 for _ in range(S)], np.int32)
    T = int(ip[-1])
    ads = []
    for a in range(n_ad):
        r = int(rng.integers(1, max_rank + 1))
        ads.append((a, r, float(rng.choice([1.0, 0.5, 2.0, 0.3])), rng.standard_normal((r, H_in)),
                    rng.standard_normal((r, H_out))))
    x = rng.standard_normal((T, H_in))
    y = rng.standard_normal((T, H_out))
    return H_in, H_out, ip, ids, ads, x, y


# ---------------------------------------------------------------- P1
def test_p1_hand_example_spec_s51():
    g = _kv(os.path.join(GOLDEN, "p1_hand_example.txt"))
    H_in, H_out, r = int(g["H_in"]), int(g["H_out"]), int(g["rank"])
    A = np.array(_nums(g["A_rank_major"])).reshape(r, H_in)
    B = np.array(_nums(g["B"])).reshape(r, H_out)
    y = O.delta(H_in, H_out, [0, 1], [7], [(7, r, float(g["scale"]), A, B)],
                np.array([_nums(g["x"])]), np.array([_nums(g["y_in"])]))
    assert y.tolist() == [_nums(g["y_expected"])]


# ---------------------------------------------------------------- P2
def test_p2_merged_weight_identity_eq1():
    """Eq. 1: xW + x(sA)B == x(W + sAB), fp64, rel <= 1e-12."""
    for seed in range(20):
        H_in, H_out, ip, ids, ads, x, _ = _rand_problem(seed, p_none=0.0)
        rng = np.random.default_rng(1000 + seed)
        W = rng.standard_normal((H_in, H_out))
        y_base = x @ W
        y = O.delta(H_in, H_out, ip, ids, ads, x, y_base)
        tab = {a[0]: a for a in ads}
        for i in range(len(ids)):
            _, r, s, A_st, B = tab[int(ids[i])]
            W_merged = W + s * (A_st.T @ B)          # paper A = A_st^T (H_in x r)
            for t in range(ip[i], ip[i + 1]):
                ref = x[t] @ W_merged
                assert np.linalg.norm(y[t] - ref) <= 1e-12 * max(1.0, np.linalg.norm(ref))


# ---------------------------------------------------------------- P3
def test_p3_numpy_blas_per_segment():
    """Library special case: per segment s*((X_seg @ A_st^T) @ B) + y_in, different
    summation order (BLAS), rel <= 1e-12."""
    for seed in range(20):
        H_in, H_out, ip, ids, ads, x, y0 = _rand_problem(seed + 50, H_in=64, H_out=48, max_len=9, max_rank=17)
        y = O.delta(H_in, H_out, ip, ids, ads, x, y0)
        tab = {a[0]: a for a in ads}
        ref = y0.copy()
        for i in range(len(ids)):
            if ids[i] < 0:
                continue
            _, r, s, A_st, B = tab[int(ids[i])]
            sl = slice(ip[i], ip[i + 1])
            ref[sl] = y0[sl] + s * ((x[sl] @ A_st.T) @ B)
        den = max(np.linalg.norm(ref - y0), 1e-300)
        assert np.linalg.norm(y - ref) <= 1e-12 * den + 1e-300


# ---------------------------------------------------------------- exact integers
def test_exact_integer_bruteforce():
    """Small-integer inputs make every fp64 operation exact; compare bit for bit with a
    pure-Python integer brute force of y_t = y_in_t + s * sum_j (sum_k x_t[k] A[k][j]) B[j][n]."""
    rng = np.random.default_rng(7)
    for trial in range(30):
        H_in, H_out, S = int(rng.integers(1, 9)), int(rng.integers(1, 9)), int(rng.integers(0, 6))
        lens = rng.integers(0, 4, size=S)
        ip = [0] + list(np.cumsum(lens).astype(int))
        ids = [int(rng.integers(-1, 3)) for _ in range(S)]
        ads = []
        for a in range(3):
            r = int(rng.integers(1, 6))
            A = rng.integers(-4, 5, size=(r, H_in))
            B = rng.integers(-4, 5, size=(r, H_out))
            s = int(rng.choice([1, 2, 4]))
            ads.append((a, r, s, A, B))
        T = ip[-1]
        x = rng.integers(-5, 6, size=(T, H_in))
        y0 = rng.integers(-9, 10, size=(T, H_out))
        y = O.delta(H_in, H_out, ip, ids, [(a, r, float(s), A.astype(float), B.astype(float)) for a, r, s, A, B in ads],
                    x.astype(float), y0.astype(float))
        for i in range(S):
            for t in range(ip[i], ip[i + 1]):
                for n in range(H_out):
                    if ids[i] < 0:
                        exp = int(y0[t][n])
                    else:
                        _, r, s, A, B = ads[ids[i]]
                        exp = int(y0[t][n])
                        for j in range(r):
                            vj = 0
                            for k in range(H_in):
                                vj += int(x[t][k]) * int(A[j][k])
                            exp += s * vj * int(B[j][n])
                    assert y[t][n] == float(exp), (trial, t, n)


# ---------------------------------------------------------------- P4
def test_p4_zero_padded_rank_is_bitwise_identical():
    """BGMV pads smaller ranks to the max rank; MBGMV does not;
    the delta is the same.  Padding with exact zeros leaves the fp64 oracle bitwise equal."""
    for seed in range(10):
        H_in, H_out, ip, ids, ads, x, y0 = _rand_problem(seed + 200)
        y = O.delta(H_in, H_out, ip, ids, ads, x, y0)
        R = 32
        padded = []
        for (a, r, s, A, B) in ads:
            Ap = np.zeros((R, H_in)); Ap[:r] = A
            Bp = np.zeros((R, H_out)); Bp[:r] = B
            padded.append((a, R, s, Ap, Bp))
        yp = O.delta(H_in, H_out, ip, ids, padded, x, y0)
        assert np.array_equal(y, yp)


# ---------------------------------------------------------------- P5
@pytest.mark.parametrize("which", ["A", "B"])
def test_p5_zero_adapter_gives_zero_delta(which):
    H_in, H_out, ip, ids, ads, x, y0 = _rand_problem(300, p_none=0.0)
    z = []
    for (a, r, s, A, B) in ads:
        z.append((a, r, s, A * 0 if which == "A" else A, B * 0 if which == "B" else B))
    y = O.delta(H_in, H_out, ip, ids, z, x, y0)
    assert np.all(y == y0)


# ---------------------------------------------------------------- P6
def test_p6_segment_permutation_bitwise():
    rng = np.random.default_rng(9)
    for seed in range(10):
        H_in, H_out, ip, ids, ads, x, y0 = _rand_problem(seed + 400)
        y = O.delta(H_in, H_out, ip, ids, ads, x, y0)
        perm = rng.permutation(len(ids))
        lens = np.diff(ip)
        ip2 = np.concatenate([[0], np.cumsum(lens[perm])]).astype(np.int32)
        rows = np.concatenate([np.arange(ip[i], ip[i + 1]) for i in perm]).astype(int) if len(perm) else np.zeros(0, int)
        y2 = O.delta(H_in, H_out, ip2, ids[perm], ads, x[rows], y0[rows])
        assert np.array_equal(y2, y[rows])


# ---------------------------------------------------------------- P7
def test_p7_segment_split_merge_bitwise():
    H_in, H_out = 32, 16
    rng = np.random.default_rng(11)
    ads = [(5, 7, 0.5, rng.standard_normal((7, H_in)), rng.standard_normal((7, H_out)))]
    x = rng.standard_normal((40, H_in)); y0 = rng.standard_normal((40, H_out))
    y_one = O.delta(H_in, H_out, [0, 40], [5], ads, x, y0)
    for cuts in ([1], [1, 2, 3], [13, 13, 27], [39]):
        ip = [0] + list(cuts) + [40]
        y_split = O.delta(H_in, H_out, ip, [5] * (len(ip) - 1), ads, x, y0)
        assert np.array_equal(y_one, y_split)


# ---------------------------------------------------------------- P8
def test_p8_linearity_and_scale_and_duplicates():
    H_in, H_out, ip, ids, ads, x, _ = _rand_problem(500, p_none=0.0)
    z = np.zeros((x.shape[0], H_out))
    d1 = O.delta(H_in, H_out, ip, ids, ads, x, z)
    for k in (-3, 1, 5):
        dk = O.delta(H_in, H_out, ip, ids, ads, x * 2.0 ** k, z)
        assert np.array_equal(dk, d1 * 2.0 ** k)
    # (A, B, s) == (A, s*B, 1)
    folded = [(a, r, 1.0, A, s * B) for (a, r, s, A, B) in ads]
    d2 = O.delta(H_in, H_out, ip, ids, folded, x, z)
    assert np.linalg.norm(d2 - d1) <= 1e-12 * np.linalg.norm(d1)
    # scale enters linearly: doubling s doubles the delta (exact)
    dbl = [(a, r, 2 * s, A, B) for (a, r, s, A, B) in ads]
    assert np.array_equal(O.delta(H_in, H_out, ip, ids, dbl, x, z), 2 * d1)
    # duplicate ids across segments are fine and equal to separate-segment results
    ip_d = [0, 1, 2]
    dd = O.delta(H_in, H_out, ip_d, [0, 0], ads, x[:2], z[:2])
    assert np.array_equal(dd[0], O.delta(H_in, H_out, [0, 1], [0], ads, x[:1], z[:1])[0])


def test_unknown_adapter_and_bad_csr_raise():
    H_in, H_out, ip, ids, ads, x, y0 = _rand_problem(600, p_none=0.0)
    with pytest.raises(KeyError):
        O.delta(H_in, H_out, ip, np.full_like(ids, 99), ads, x, y0)
    bad = ip.copy(); bad[0] = 1
    with pytest.raises(ValueError):
        O.delta(H_in, H_out, bad, ids, ads, x, y0)


def test_no_adapter_rows_untouched():
    H_in, H_out, ip, ids, ads, x, y0 = _rand_problem(601, p_none=0.5)
    y = O.delta(H_in, H_out, ip, ids, ads, x, y0)
    for i in range(len(ids)):
        if ids[i] < 0:
            assert np.array_equal(y[ip[i]:ip[i + 1]], y0[ip[i]:ip[i + 1]])


# ---------------------------------------------------------------- P9
def test_p9_randomized_sweep_spec_acceptance3():
    """SPEC acceptance 3: 1000 random batches (H <= 32, |S| <= 16, r in 1..16);
    the oracle matches an independent numpy per-request loop (einsum order) within 1e-12."""
    rng = np.random.default_rng(12345)
    for trial in range(1000):
        H_in, H_out = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        S = int(rng.integers(1, 17))
        lens = rng.integers(0, 4, size=S)
        ip = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        n_ad = int(rng.integers(1, 5))
        ads = [(a, int(rng.integers(1, 17)), 1.0, None, None) for a in range(n_ad)]
        ads = [(a, r, s, rng.uniform(-0.1, 0.1, (r, H_in)), rng.uniform(-0.1, 0.1, (r, H_out))) for a, r, s, _, _ in ads]
        ids = rng.integers(-1, n_ad, size=S).astype(np.int32)
        T = int(ip[-1])
        x = rng.uniform(-0.1, 0.1, (T, H_in)); y0 = rng.uniform(-0.1, 0.1, (T, H_out))
        y = O.delta(H_in, H_out, ip, ids, ads, x, y0)
        for i in range(S):
            sl = slice(ip[i], ip[i + 1])
            if ids[i] < 0:
                assert np.array_equal(y[sl], y0[sl]); continue
            _, r, s, A, B = ads[ids[i]]
            ref = y0[sl] + s * np.einsum("tj,jn->tn", np.einsum("tk,jk->tj", x[sl], A), B)
            assert np.allclose(y[sl], ref, rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- P10
def test_p10_toy_example_features():
    lines = [l.split() for l in open(os.path.join(GOLDEN, "p10_toy_features.txt"))
             if l.strip() and not l.startswith("#")]
    for parts in lines:
        if parts[0] == "work":
            _, name, ranks, H, bg, mb = parts
            ranks = [int(r) for r in ranks.split(",")]
            assert O.work_units("bgmv", ranks, int(H)) == int(bg)
            assert O.work_units("mbgmv", ranks, int(H)) == int(mb)
            continue
        name, spec, nsm, srs = parts
        ranks = []
        for item in spec.split(","):
            r, n = item.split("x")
            ranks += [int(r)] * int(n)
        # one decode request per segment, each on its own adapter
        table = {i: (r, 1.0, list(range(i * 64, i * 64 + r))) for i, r in enumerate(ranks)}
        md = O.canonical_metadata(list(range(len(ranks) + 1)), list(range(len(ranks))), table, L_tc=64)
        assert md["nseg_x_maxrank"] == int(nsm), name
        assert md["sum_rank_seg"] == int(srs), name


# ---------------------------------------------------------------- P11
def test_p11_adapter_bytes_closed_form():
    g = _kv(os.path.join(GOLDEN, "p11_adapter_bytes.txt"))
    r, H, L, P, b = (int(g[k]) for k in ("rank", "hidden", "layers", "projections", "elem_bytes"))
    total = P * L * O.adapter_bytes(r, H, H, b)
    assert total == int(g["adapter_bytes_total"]) == 96 * 2 ** 20
    kv = 200 * 2 * L * H * b
    assert kv == int(g["kv_cache_200_tokens"]) == 100 * 2 ** 20


# ---------------------------------------------------------------- P14
def test_p14_openmp_bitwise_equals_serial_and_repeatable():
    b = gen.config_c1(y_zero=False)
    y1 = O.delta_for_batch(b, n_threads=1)
    y2 = O.delta_for_batch(b, n_threads=4)
    y3 = O.delta_for_batch(b, n_threads=1)
    assert np.array_equal(y1, y2) and np.array_equal(y1, y3)
    H_in, H_out, ip, ids, ads, x, y0 = _rand_problem(700, H_in=128, H_out=96, S=12, max_len=20, max_rank=40)
    assert np.array_equal(O.delta(H_in, H_out, ip, ids, ads, x, y0, n_threads=1),
                          O.delta(H_in, H_out, ip, ids, ads, x, y0, n_threads=8))


def test_token_mask_and_v_out():
    H_in, H_out, ip, ids, ads, x, y0 = _rand_problem(800, p_none=0.0)
    y, v = O.delta(H_in, H_out, ip, ids, ads, x, y0, want_v=True)
    T = x.shape[0]
    mask = np.zeros(T, np.uint8); mask[::2] = 1
    ym = O.delta(H_in, H_out, ip, ids, ads, x, y0, token_mask=mask)
    assert np.array_equal(ym[::2], y[::2]) and np.all(np.isnan(ym[1::2]))
    # v_t = s * x_t A  (paper A = A_st^T): check against BLAS per token
    tab = {a[0]: a for a in ads}
    for i in range(len(ids)):
        _, r, s, A, B = tab[int(ids[i])]
        for t in range(ip[i], ip[i + 1]):
            assert np.allclose(v[t, :r], s * (A @ x[t]), rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- metadata / allocator
def test_canonical_metadata_brute_force_definitions():
    ip = [0, 1, 1, 4, 5, 9, 10]
    ids = [3, 1, 3, -1, 1, 2]
    table = {1: (2, 0.5, [7, 2]), 2: (1, 4.0, [9]), 3: (3, 1.0, [0, 1, 5])}
    md = O.canonical_metadata(ip, ids, table, L_tc=4)
    assert md["tok_seg"].tolist() == [0, 2, 2, 2, 3, 4, 4, 4, 4, 5]
    # segment 1 (id 1) is empty; id 1 still owns tokens via segment 4 -> group exists
    assert md["group_id"].tolist() == [1, 2, 3]
    assert md["group_ntok"].tolist() == [4, 1, 4]
    assert md["group_tokens"].tolist() == [5, 6, 7, 8, 9, 0, 1, 2, 3]
    assert md["group_tok_off"].tolist() == [0, 4, 5]
    assert md["pages"].tolist() == [7, 2, 9, 0, 1, 5]
    assert md["group_page_off"].tolist() == [0, 2, 3]
    assert md["group_scale"].tolist() == [0.5, 4.0, 1.0]
    assert md["seg_kind"].tolist() == [O.KIND_DECODE, O.KIND_NONE, O.KIND_DECODE, O.KIND_NONE,
                                       O.KIND_PREFILL, O.KIND_DECODE]
    assert md["n_seg"] == 4 and md["max_rank"] == 3 and md["nseg_x_maxrank"] == 12
    assert md["sum_rank_seg"] == 3 + 3 + 2 + 1
    assert md["sum_rank_groups"] == 6
    assert md["sum_rank_tokens"] == 3 * 1 + 3 * 3 + 2 * 4 + 1 * 1


def test_allocator_replay_lowest_free_first():
    a = O.PageAllocatorReplay(n_pages=10, max_adapters=2)
    assert a.load(10, 3) == [0, 1, 2]
    assert a.load(11, 2) == [3, 4]
    a.unload(10)
    assert a.load(12, 4) == [0, 1, 2, 5]
    with pytest.raises(O.PoolFull):
        a.load(13, 1)          # slots exhausted (2 resident)
    a.unload(11)
    with pytest.raises(O.PoolFull):
        a.load(13, 7)          # only 6 free pages: 3,4,6,7,8,9
    assert a.load(13, 6) == [3, 4, 6, 7, 8, 9]
    with pytest.raises(KeyError):
        a.load(13, 1)


def test_generator_is_deterministic_and_bf16_rounding():
    b1, b2 = gen.config_c2(), gen.config_c2()
    assert np.array_equal(b1.x, b2.x) and np.array_equal(b1.adapter_ids, b2.adapter_ids)
    assert sorted(np.bincount(b1.adapter_ids).tolist()) == [2] * 32
    assert sum(a.rank for a in b1.adapters) == 960
    # RNE: 1 + 2^-8 (exact tie) rounds to even (1.0); 1 + 3*2^-9 rounds up
    v = np.array([1 + 2 ** -8, 1 + 3 * 2 ** -9, -2.5], np.float32)
    assert gen.bf16_bits_to_f32(gen.f32_to_bf16_bits(v)).tolist() == [1.0, 1.0078125, -2.5]
