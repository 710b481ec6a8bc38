"""GPU parity of the experimental cluster-span decode kernel (N1c, csrc/span_kernel.cu; selected
with LORA_OPT_DECODE_PATH = 1) against the fp64 oracle and the default kernel pair, via the C ABI.

Covers: the c2 / c5 decode shapes (spans of 2..16 CTAs, ring streaming of slices larger than
the ring), Zipf batches (several 8-token chunks of one adapter), ragged hidden sizes whose last
k/n slice is not a multiple of 16, ranks 1..256, empty / no-adapter segments, lora_apply_multi
(jobs of different shapes in one grid), CUDA graph replay, and bitwise batch-order independence.
"""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

from gpu_util import TOL, make_pool, rel_l2, run_gpu, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2401_11240_b200 as L
    return L


def _span_pool(b, L, **kw):
    from paper_2401_11240_b200 import binding as B
    pool = make_pool(b, L, **kw)
    pool.set_option(B.LORA_OPT_DECODE_PATH, 1)
    return pool


def _both_paths(L, b):
    """outs[0] = cluster-span kernel (LORA_OPT_DECODE_PATH 1), outs[1] = kernel pair (default)."""
    from paper_2401_11240_b200 import binding as B
    outs = {}
    for path in (1, 0):
        pool = make_pool(b, L, L_tc=1 << 30)
        pool.set_option(B.LORA_OPT_DECODE_PATH, path)
        outs[1 - path], md = run_gpu(b, L, pool=pool)
        pool.close()
    return outs


CASES = {
    "c2_runA": lambda: gen.config_c2(y_zero=True),
    "c2_runB": lambda: gen.config_c2(y_zero=False),
    "c2_zipf": lambda: gen.config_c2(zipf=True, y_zero=False, tag=5),
    "c5_q": lambda: gen.config_c5("q", y_zero=False),
    "c5_k": lambda: gen.config_c5("k", y_zero=False),
    "c5_down": lambda: gen.config_c5("down", y_zero=False),
    "c5_up": lambda: gen.config_c5("up", y_zero=False) if "up" in gen.C5_SHAPES else gen.config_c5("q"),
}


@pytest.mark.parametrize("name", list(CASES))
def test_span_matches_oracle_and_pair(L, name):
    b = CASES[name]()
    ref = O.delta_for_batch(b, n_threads=16)
    outs = _both_paths(L, b)
    e_span = rel_l2(outs[0], ref, "bf16")
    e_pair = rel_l2(outs[1], ref, "bf16")
    assert e_span <= TOL["bf16"], (name, e_span)
    assert e_pair <= TOL["bf16"], (name, e_pair)


@pytest.mark.parametrize("seed", range(12))
def test_span_ragged_shapes_and_ranks(L, seed):
    """H multiples of 8 but not 16 (ragged last slices), ranks up to 256, empty and id<0 segments."""
    rng = np.random.default_rng(900 + seed)
    H_in = int(rng.integers(2, 80)) * 8 + (8 if seed % 2 else 0)
    H_out = int(rng.integers(2, 80)) * 8 + (8 if seed % 3 else 0)
    max_rank = min(256, H_in, H_out)
    b = gen.random_batch(5000 + seed, "bf16", H_in, H_out, max_seg=48, max_rank=max_rank, max_len=12,
                         n_adapters=10, y_zero=bool(seed % 2))
    if b.T == 0:
        pytest.skip("empty batch")
    ref = O.delta_for_batch(b, n_threads=16)
    outs = _both_paths(L, b)
    assert rel_l2(outs[0], ref, "bf16") <= TOL["bf16"], (H_in, H_out)
    # rows of tokens without an adapter are bitwise untouched
    none = np.zeros(b.T, dtype=bool)
    for i, a in enumerate(b.adapter_ids):
        if a < 0:
            none[b.seg_indptr[i]:b.seg_indptr[i + 1]] = True
    y_in = b.y_in.reshape(b.T, -1)
    assert np.array_equal(outs[0].reshape(b.T, -1)[none], y_in[none])


def test_span_large_hidden_falls_back_or_matches(L):
    """28672 -> 8192 (c5 down): slices of 1792 columns; and a shape beyond the span limits
    (H = 40960 > 16 x 2048) that must take the kernel pair automatically."""
    for H_in, H_out in ((28672, 8192), (40960, 512)):
        b = gen.random_batch(77 + H_in, "bf16", H_in, H_out, max_seg=10, max_rank=64, max_len=3, n_adapters=4)
        ref = O.delta_for_batch(b, n_threads=16)
        pool = _span_pool(b, L, L_tc=1 << 30)
        y, _ = run_gpu(b, L, pool=pool)
        pool.close()
        assert rel_l2(y, ref, "bf16") <= TOL["bf16"], (H_in, H_out)


def test_span_batch_order_bitwise(L):
    """A token's result is a fixed function of (x_t, adapter): permuting the segments permutes
    the output rows bitwise (pin P6 on the span path)."""
    b = gen.config_c2(zipf=True, y_zero=False, tag=9)
    pool = _span_pool(b, L)
    y0, md = run_gpu(b, L, pool=pool)
    assert md["n_span_ctas"] > 0
    S = len(b.adapter_ids)
    perm = np.random.default_rng(3).permutation(S)
    lens = np.diff(b.seg_indptr)
    tok = [np.arange(b.seg_indptr[i], b.seg_indptr[i + 1]) for i in range(S)]
    order = np.concatenate([tok[i] for i in perm])
    bp = gen.Batch(**{**b.__dict__})
    bp.seg_indptr = gen.segments_to_indptr([int(lens[i]) for i in perm])
    bp.adapter_ids = np.asarray(b.adapter_ids)[perm].astype(np.int32)
    bp.x = b.x.reshape(b.T, -1)[order].copy()
    bp.y_in = b.y_in.reshape(b.T, -1)[order].copy()
    y1, _ = run_gpu(bp, L, pool=pool)
    pool.close()
    assert np.array_equal(y1.reshape(b.T, -1), y0.reshape(b.T, -1)[order])


def test_span_apply_multi_mixed_shapes(L):
    """lora_apply_multi over pools of different shapes (q 8192x8192 and k 8192x1024 of c5) on the
    span path matches the oracle (the fused batch may exceed the span parameter blob and take the
    pair, so only tolerance, not bitwise equality with separate applies, is required)."""
    import torch
    bq, bk = gen.config_c5("q", y_zero=False), gen.config_c5("k", y_zero=False)
    # one batch layout for both pools (lora_apply_multi shares seg_indptr / adapter_ids / x)
    bk = gen.Batch(**{**bk.__dict__, "seg_indptr": bq.seg_indptr, "adapter_ids": bq.adapter_ids, "x": bq.x})
    pq, pk = _span_pool(bq, L, L_tc=1 << 30), _span_pool(bk, L, L_tc=1 << 30)
    x = to_torch(bq.x, "cuda")
    ys = [to_torch(bq.y_in, "cuda"), to_torch(bk.y_in, "cuda")]
    L.apply_multi([pq, pk], [x, x], ys, bq.seg_indptr, bq.adapter_ids)
    torch.cuda.synchronize()
    sep = [to_torch(bq.y_in, "cuda"), to_torch(bk.y_in, "cuda")]
    pq.apply(x, sep[0], bq.seg_indptr, bq.adapter_ids)
    pk.apply(x, sep[1], bq.seg_indptr, bq.adapter_ids)
    torch.cuda.synchronize()
    for b, y in ((bq, ys[0]), (bk, ys[1]), (bq, sep[0]), (bk, sep[1])):
        ref = O.delta_for_batch(b, n_threads=16)
        got = y.cpu().numpy().view(np.uint16)
        assert rel_l2(got, ref, "bf16") <= TOL["bf16"]
    pq.close()
    pk.close()


def test_span_graph_replay_accumulates(L):
    """Graph capture of span applies (kernel parameters captured by value): 5 replays add the
    delta 5 times, identical to 5 eager applies."""
    import torch
    b = gen.config_c2(y_zero=False, tag=2)
    pool = _span_pool(b, L)
    x = to_torch(b.x, "cuda")
    y_e = to_torch(b.y_in, "cuda")
    for _ in range(5):
        pool.apply(x, y_e, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    y_g = to_torch(b.y_in, "cuda")
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        pool.apply(x, y_g, b.seg_indptr, b.adapter_ids, stream=st)
    y_g.copy_(to_torch(b.y_in, "cuda"))
    with torch.cuda.stream(st):
        for _ in range(5):
            g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_e, y_g)
    pool.close()
