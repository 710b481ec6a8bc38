"""GPU parity: the CUDA path through the C ABI versus the fp64 oracle on the same seeded
inputs (SURVEY.md §8(c) "GPU parity test matrix").  Tolerances are BASELINE.json's:
rel-L2 <= 5e-3 (bf16 inputs, fp32 accumulation), <= 1e-5 (fp32); metadata bit-exact."""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

from gpu_util import TOL, from_torch, make_pool, rel_l2, run_gpu, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2401_11240_b200 as lib
    return lib


def _md_ref(batch, L_tc=64):
    table = {}
    alloc = O.PageAllocatorReplay(sum(a.rank for a in batch.adapters) + 1, len(batch.adapters) + 4)
    for a in batch.adapters:
        alloc.load(a.id, a.rank, a.scale)
    return O.canonical_metadata(batch.seg_indptr, batch.adapter_ids, alloc.table, L_tc)


def _check_md(md, ref):
    for k in ("tok_seg", "group_id", "group_rank", "group_ntok", "group_page_off", "group_tok_off", "group_tokens",
              "pages", "seg_kind"):
        assert np.array_equal(md[k], ref[k]), k
    assert np.array_equal(md["group_scale"].view(np.uint32), ref["group_scale"].view(np.uint32))
    for k in ("n_seg", "max_rank", "nseg_x_maxrank", "sum_rank_seg", "sum_rank_groups", "sum_rank_tokens"):
        assert md[k] == ref[k], k


@pytest.mark.parametrize("y_zero", [True, False], ids=["runA_delta", "runB_accumulate"])
def test_c1_tiny_fp32(L, y_zero):
    b = gen.config_c1(y_zero=y_zero)
    y, md = run_gpu(b, L)
    ref = O.delta_for_batch(b)
    assert rel_l2(y, ref, "f32") <= TOL["f32"]
    _check_md(md, _md_ref(b))


@pytest.mark.parametrize("y_zero", [True, False], ids=["runA_delta", "runB_accumulate"])
def test_c2_decode_bf16(L, y_zero):
    b = gen.config_c2(y_zero=y_zero)
    y, md = run_gpu(b, L)
    ref = O.delta_for_batch(b, n_threads=8)
    err = rel_l2(y, ref, "bf16")
    assert err <= TOL["bf16"], err
    _check_md(md, _md_ref(b))


def test_c2_zipf_bf16(L):
    b = gen.config_c2(zipf=True)
    y, md = run_gpu(b, L)
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
    _check_md(md, _md_ref(b))


def test_prefill_tiles_bf16_and_fp32(L):
    for dtype in ("bf16", "f32"):
        for y_zero in (True, False):
            b = gen.config_c1_prefill_tiles(y_zero=y_zero, dtype=dtype)
            y, md = run_gpu(b, L)
            ref = O.delta_for_batch(b, n_threads=8)
            assert rel_l2(y, ref, dtype) <= TOL[dtype], (dtype, y_zero)
            _check_md(md, _md_ref(b))
            if dtype == "bf16":
                # segments >= L_tc with rank <= 128 ran on the tcgen05 kernel: 63->0 (decode), 64, 127,
                # 128, 129, 300 tokens -> 1+1+1+2+3 tiles, minus the rank-128 segment routing rule (all <= 128)
                assert md["n_prefill_tiles"] == 1 + 1 + 1 + 2 + 3, md["n_prefill_tiles"]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tcgen05_prefill_vs_simt_path_and_oracle(L, seed):
    """The same prefill batch through the tcgen05 kernel (L_tc = 16) and through the decode
    kernels only (L_tc huge): both within tolerance of the oracle, ragged tiles, all ranks 1..128."""
    rng = np.random.default_rng(seed)
    lens = [int(v) for v in rng.integers(16, 400, size=6)]
    ranks = {i: int(r) for i, r in enumerate(rng.choice([1, 3, 8, 16, 24, 40, 64, 100, 128], size=6))}
    ids = list(range(6))
    H_in, H_out = [(256, 384), (512, 128), (1024, 1024)][seed]
    b = gen.build_batch("tcp%d" % seed, 777 + seed, "bf16", H_in, H_out, lens, ids, ranks, y_zero=bool(seed % 2))
    ref = O.delta_for_batch(b, n_threads=8)
    y_tc, md_tc = run_gpu(b, L, L_tc=16)
    y_simt, md_simt = run_gpu(b, L, L_tc=1 << 30)
    assert md_tc["n_prefill_tiles"] == sum((n + 127) // 128 for n in lens)
    assert md_simt["n_prefill_tiles"] == 0
    assert rel_l2(y_tc, ref, "bf16") <= TOL["bf16"]
    assert rel_l2(y_simt, ref, "bf16") <= TOL["bf16"]


def test_c3_prefill_reduced(L):
    """config 3 shape (4096, ranks 8..128) with 8 x 512-token segments, all tokens checked."""
    b = gen.config_c3(n_seg=8)
    y, md = run_gpu(b, L)
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
    _check_md(md, _md_ref(b))


def test_c3_full_size_every_token(L):
    """config 3 at full size (32 x 512 tokens = 128 token tiles, the bench's launch configuration):
    every one of the 16,384 tokens against the oracle (OpenMP over tokens), global and per-token
    rel-L2 (gpu_util.rel_l2), run A (delta alone) and run B (accumulate)."""
    import os
    for y_zero in (True, False):
        b = gen.config_c3(y_zero=y_zero)
        y, md = run_gpu(b, L)
        assert md["n_prefill_tiles"] == 128
        ref = O.delta_for_batch(b, n_threads=len(os.sched_getaffinity(0)))
        assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
        _check_md(md, _md_ref(b))


@pytest.mark.parametrize("proj", ["k", "q", "down"])
def test_c5_70b_shapes_decode(L, proj):
    b = gen.config_c5(proj, y_zero=False)
    y, md = run_gpu(b, L)
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]


def test_page_readback_p12(L):
    for b in (gen.config_c1(), gen.config_c2()):
        pool = make_pool(b, L)
        for a in b.adapters:
            A, B = pool.read_pages(a.id, a.rank)
            assert np.array_equal(A, a.A) and np.array_equal(B, a.B)
        pool.close()


def test_no_adapter_rows_bitwise_untouched(L):
    b = gen.config_c2(y_zero=False)
    ids = b.adapter_ids.copy()
    ids[::4] = -1
    y, _ = run_gpu(b, L, adapter_ids=ids)
    T = b.T
    y = y.reshape(T, -1)
    ref = O.delta(b.H_in, b.H_out, b.seg_indptr, ids,
                  [(a.id, a.rank, a.scale, gen.storage_to_f64(a.A, "bf16"), gen.storage_to_f64(a.B, "bf16"))
                   for a in b.adapters], gen.storage_to_f64(b.x, "bf16"), gen.storage_to_f64(b.y_in, "bf16"))
    for i in range(len(ids)):
        rows = slice(b.seg_indptr[i], b.seg_indptr[i + 1])
        if ids[i] < 0:
            assert np.array_equal(y[rows], b.y_in[rows])
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]


@pytest.mark.parametrize("which", ["A", "B"])
def test_zero_adapter_p5(L, which):
    for dtype_batch in (gen.config_c1(y_zero=False), gen.config_c2(y_zero=False)):
        b = dtype_batch
        for a in b.adapters:
            if which == "A":
                a.A = np.zeros_like(a.A)
            else:
                a.B = np.zeros_like(a.B)
        y, _ = run_gpu(b, L)
        yv = gen.storage_to_f64(y, b.dtype)
        assert np.array_equal(yv, gen.storage_to_f64(b.y_in, b.dtype))


def test_zero_padded_rank_p4(L):
    """An adapter zero-padded from r to 2r gives the same delta within tolerance."""
    b = gen.config_c2()
    y1, _ = run_gpu(b, L)
    for a in b.adapters:
        a.A = np.concatenate([a.A, np.zeros_like(a.A)])
        a.B = np.concatenate([a.B, np.zeros_like(a.B)])
        a.rank *= 2
    y2, _ = run_gpu(b, L)
    ref = O.delta_for_batch(gen.config_c2(), n_threads=8)
    assert rel_l2(y2, ref, "bf16") <= TOL["bf16"]
    assert rel_l2(y2, gen.storage_to_f64(y1, "bf16").reshape(ref.shape), "bf16") <= TOL["bf16"]


def test_segment_permutation_bitwise_p6(L):
    b = gen.config_c2()
    y, _ = run_gpu(b, L)
    y = y.reshape(b.T, -1)
    rng = np.random.default_rng(5)
    perm = rng.permutation(b.S)
    b2 = gen.config_c2()
    b2.adapter_ids = b.adapter_ids[perm].copy()
    b2.x = b.x[perm].copy()           # one-token segments: token index = segment index
    b2.y_in = b.y_in[perm].copy()
    y2, _ = run_gpu(b2, L)
    assert np.array_equal(y2.reshape(b.T, -1), y[perm])


def test_segment_split_merge_p7(L):
    b = gen.config_c1_prefill_tiles()
    ref = O.delta_for_batch(b, n_threads=8)
    lens = np.diff(b.seg_indptr)
    new_lens, new_ids = [], []
    for ln, aid in zip(lens, b.adapter_ids):
        if ln > 2:
            new_lens += [1, ln - 1]
            new_ids += [aid, aid]
        else:
            new_lens.append(ln)
            new_ids.append(aid)
    ip = gen.segments_to_indptr(new_lens)
    y, _ = run_gpu(b, L, seg_indptr=ip, adapter_ids=np.array(new_ids, np.int32))
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]


def test_determinism_repeat(L):
    b = gen.config_c2(y_zero=False)
    outs = [run_gpu(b, L)[0] for _ in range(3)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_randomized_sweep_p9(L):
    rng = np.random.default_rng(77)
    for trial in range(120):
        dtype = "bf16" if trial % 3 else "f32"
        vec = 8 if dtype == "bf16" else 4
        H_in = int(rng.integers(1, 33)) * vec
        H_out = int(rng.integers(1, 33)) * vec
        b = gen.random_batch(1000 + trial, dtype, H_in, H_out, max_seg=64, max_rank=min(128, H_in, H_out),
                             max_len=int(rng.choice([1, 4, 40, 300])), n_adapters=8, y_zero=bool(trial % 2))
        if b.T == 0:
            continue
        y, md = run_gpu(b, L)
        ref = O.delta_for_batch(b, n_threads=8)
        assert rel_l2(y, ref, dtype) <= TOL[dtype], (trial, dtype, H_in, H_out)
        _check_md(md, _md_ref(b))


def test_empty_batches_are_noops(L):
    import torch
    b = gen.config_c1(y_zero=False)
    pool = make_pool(b, L)
    x = to_torch(b.x, "cuda")
    y = to_torch(b.y_in, "cuda")
    pool.apply(x, y, [0], [])
    pool.apply(x, y, [0, 0, 0], [0, 1])
    pool.apply(x, y, [0, 4], [-1])
    torch.cuda.synchronize()
    assert np.array_equal(from_torch(y, "f32"), b.y_in)
    pool.close()


def test_cuda_graph_capture_replay(L):
    import torch
    b = gen.config_c2()
    pool = make_pool(b, L)
    x = to_torch(b.x, "cuda")
    y = torch.zeros((b.T, b.H_out), dtype=torch.int16, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=s)    # warm-up (scratch sizing)
    torch.cuda.synchronize()
    y.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=s)
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(from_torch(y, "bf16"), ref, "bf16") <= TOL["bf16"]
    pool.close()


def test_graph_capture_scratch_growth(L):
    """Scratch growth and CUDA graphs: an apply that would have to grow the pool's scratch inside a
    capture is refused (LORA_ERR_UNSUPPORTED, nothing allocated or synchronised, so the caller's
    capture stays valid); a graph captured before an eager apply grew the scratch still replays
    exactly (outgrown buffers are retired, not freed)."""
    import torch
    big = gen.config_c2(T=256, y_zero=False)
    small = gen.config_c2(T=16, y_zero=False, tag=3)
    used = set(int(a) for a in small.adapter_ids)
    small.adapters = [a for a in big.adapters if a.id in used]   # the pool holds big's adapters
    pool = make_pool(big, L)
    s = torch.cuda.Stream()
    xs, ys = to_torch(small.x, "cuda"), to_torch(small.y_in, "cuda")
    xb, yb = to_torch(big.x, "cuda"), to_torch(big.y_in, "cuda")
    y0s, y0b = ys.clone(), yb.clone()
    with torch.cuda.stream(s):
        pool.apply(xs, ys, small.seg_indptr, small.adapter_ids, stream=s)   # sizes scratch for 16 tokens
    torch.cuda.synchronize()
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=s):
        pool.apply(xs, ys, small.seg_indptr, small.adapter_ids, stream=s)
    g2 = torch.cuda.CUDAGraph()
    with pytest.raises(L.LoraError) as ei:
        with torch.cuda.graph(g2, stream=s):
            pool.apply(xb, yb, big.seg_indptr, big.adapter_ids, stream=s)
    assert ei.value.name == "LORA_ERR_UNSUPPORTED" and "capture" in str(ei.value)
    torch.cuda.synchronize()
    yb.copy_(y0b)
    with torch.cuda.stream(s):
        pool.apply(xb, yb, big.seg_indptr, big.adapter_ids, stream=s)       # grows the scratch
    torch.cuda.synchronize()
    assert rel_l2(from_torch(yb, "bf16"), O.delta_for_batch(big, n_threads=8), "bf16") <= TOL["bf16"]
    ys.copy_(y0s)
    with torch.cuda.stream(s):
        g1.replay()                                                            # captured before the growth
    torch.cuda.synchronize()
    assert rel_l2(from_torch(ys, "bf16"), O.delta_for_batch(small, n_threads=8), "bf16") <= TOL["bf16"]
    pool.close()


def test_async_load_then_apply_orders_on_event(L):
    """lora_load_adapter returns before the copy lands; an apply issued right after must see
    the adapter (the stream waits on the load's ready event)."""
    import torch
    b = gen.config_c2()
    pool = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=2048)
    keep = []
    for a in b.adapters:
        A, B = to_torch(a.A, pin=True), to_torch(a.B, pin=True)
        keep.append((A, B))
        pool.load_adapter(a.id, a.rank, A, B, a.scale)
    x = to_torch(b.x, "cuda")
    y = torch.zeros((b.T, b.H_out), dtype=torch.int16, device="cuda")
    s = torch.cuda.Stream()
    pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=s)
    s.synchronize()
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(from_torch(y, "bf16"), ref, "bf16") <= TOL["bf16"]
    assert all(pool.adapter_ready(a.id) for a in b.adapters)
    # unload half, load new adapters into the freed pages, apply again
    for a in b.adapters[::2]:
        pool.unload_adapter(a.id)
    b2 = gen.config_c2(tag=7)
    for a in b2.adapters[::2]:
        A, B = to_torch(a.A, pin=True), to_torch(a.B, pin=True)
        keep.append((A, B))
        pool.load_adapter(a.id, a.rank, A, B, a.scale)
    y.zero_()
    pool.apply(to_torch(b2.x, "cuda"), y, b2.seg_indptr, b2.adapter_ids, stream=s)
    s.synchronize()
    mixed = gen.config_c2(tag=7)
    mixed.adapters = [b2.adapters[i] if i % 2 == 0 else b.adapters[i] for i in range(32)]
    ref2 = O.delta_for_batch(mixed, n_threads=8)
    assert rel_l2(from_torch(y, "bf16"), ref2, "bf16") <= TOL["bf16"]
    pool.close()


def test_unknown_adapter_on_apply_has_no_side_effect(L):
    import torch
    b = gen.config_c1(y_zero=False)
    pool = make_pool(b, L, extra_pages=8)
    x = to_torch(b.x, "cuda")
    y = to_torch(b.y_in, "cuda")
    with pytest.raises(L.LoraError) as ei:
        pool.apply(x, y, [0, 1, 2], [0, 42])
    assert ei.value.name == "LORA_ERR_UNKNOWN_ADAPTER"
    torch.cuda.synchronize()
    assert np.array_equal(from_torch(y, "f32"), b.y_in)
    with pytest.raises(L.LoraError) as ei:
        pool.load_adapter(9, 2, np.zeros((2, 64), np.float32), np.zeros((2, 64), np.float32), 1.0)
    assert ei.value.name == "LORA_ERR_NOT_PINNED"
    pool.close()


def test_misaligned_pointers_rejected_without_side_effects(L):
    """x / y not 16-B aligned and a TP v buffer not 4-B aligned are refused (LORA_ERR_ALIGN) before
    any launch: y is unchanged, no CUDA error is left pending, and the next valid apply is exact."""
    import torch
    b = gen.config_c2(y_zero=False)
    pool = make_pool(b, L)
    x = to_torch(b.x, "cuda")
    y = to_torch(b.y_in, "cuda")
    v = torch.zeros(1 << 20, dtype=torch.float32, device="cuda")
    cases = [
        lambda: pool.apply(x.data_ptr() + 2, y, b.seg_indptr, b.adapter_ids),
        lambda: pool.apply(x, y.data_ptr() + 8, b.seg_indptr, b.adapter_ids),
        lambda: pool.apply_shrink(x, b.seg_indptr, b.adapter_ids, v.data_ptr() + 2),
    ]
    for fn in cases:
        with pytest.raises(L.LoraError) as ei:
            fn()
        assert ei.value.name == "LORA_ERR_ALIGN", str(ei.value)
    torch.cuda.synchronize()
    assert np.array_equal(from_torch(y, "bf16"), b.y_in)
    pool.apply(x, y, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(from_torch(y, "bf16"), ref, "bf16") <= TOL["bf16"]
    pool.close()


def test_apply_multi_qkv_fused_equals_separate(L):
    """lora_apply_multi over 3 pools (q, k, v of one layer; k/v with GQA-like narrower output) in
    one launch pair == three separate lora_apply calls, bit for bit, and within tolerance of the oracle."""
    import torch
    shapes = [(512, 512), (512, 128), (512, 128)]
    batches = []
    for i, (hin, hout) in enumerate(shapes):
        b = gen.build_batch("m%d" % i, 900 + i, "bf16", hin, hout, [1] * 24 + [3, 70], list(range(24)) + [2, 5],
                            {a: [8, 16, 32, 64][a % 4] for a in range(24)}, y_zero=False)
        batches.append(b)
    batches[1].x = batches[0].x.copy()
    batches[2].x = batches[0].x.copy()
    pools = [make_pool(b, L) for b in batches]
    xs = [to_torch(b.x, "cuda") for b in batches]
    y_sep = [to_torch(b.y_in, "cuda") for b in batches]
    y_fus = [to_torch(b.y_in, "cuda") for b in batches]
    for p, x, y, b in zip(pools, xs, y_sep, batches):
        p.apply(x, y, b.seg_indptr, b.adapter_ids)
    L.apply_multi(pools, xs, y_fus, batches[0].seg_indptr, batches[0].adapter_ids)
    torch.cuda.synchronize()
    for b, ys_, yf in zip(batches, y_sep, y_fus):
        assert torch.equal(ys_, yf)
        ref = O.delta_for_batch(b, n_threads=8)
        assert rel_l2(from_torch(yf, "bf16"), ref, "bf16") <= TOL["bf16"]
    for p in pools:
        p.close()


def test_box_path_never_reads_neighbour_pages(L):
    """Tenant isolation on the TMA-box path (prefill and fused base GEMM): an adapter of rank 24
    (not a multiple of 16) whose page run is followed by another adapter whose A and B hold Inf /
    NaN.  Rows past the rank must come from the zero page: y stays finite and matches the oracle."""
    import torch
    rng = np.random.default_rng(11)
    b = gen.build_batch("iso", 2424, "bf16", 256, 512, [300, 129], [0, 2], {0: 24, 2: 8}, y_zero=False)
    pool = L.LoraPool(b.H_in, b.H_out, 8, "bf16", max_total_rank=64)
    pool.set_option(L.binding.LORA_OPT_TC_THRESHOLD, 16)
    by_id = {a.id: a for a in b.adapters}
    a0 = by_id[0]
    pool.load_adapter(0, a0.rank, to_torch(a0.A, pin=True), to_torch(a0.B, pin=True), a0.scale)
    # neighbour: pages right after adapter 0's run, full of Inf / NaN
    bad_A = np.full((16, b.H_in), 0x7F80, np.uint16)   # +Inf
    bad_B = np.full((16, b.H_out), 0x7FC0, np.uint16)  # NaN
    bad_A[::2] = 0x7FC0
    pool.load_adapter(1, 16, to_torch(bad_A, pin=True), to_torch(bad_B, pin=True), 1.0)
    a2 = by_id[2]
    pool.load_adapter(2, a2.rank, to_torch(a2.A, pin=True), to_torch(a2.B, pin=True), a2.scale)
    assert pool.adapter_pages(0) == list(range(24)) and pool.adapter_pages(1)[0] == 24
    ref = O.delta_for_batch(b, n_threads=8)
    y, md = run_gpu(b, L, pool=pool)
    assert md["n_prefill_tiles"] == 3 + 2
    yf = gen.storage_to_f64(y, "bf16")
    assert np.isfinite(yf).all()
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
    # fused base GEMM: y = x·W + delta, the same pool
    w = rng.standard_normal((b.H_in, b.H_out)).astype(np.float32) / np.sqrt(b.H_in)
    W = gen.f32_to_storage(w, "bf16")
    yb = torch.zeros((b.T, b.H_out), dtype=torch.int16, device="cuda")
    pool.apply_fused_base(to_torch(b.x, "cuda"), to_torch(W, "cuda"), yb, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    got = gen.storage_to_f64(from_torch(yb, "bf16"), "bf16").reshape(b.T, b.H_out)
    base = gen.storage_to_f64(b.x, "bf16").reshape(b.T, b.H_in) @ gen.storage_to_f64(W, "bf16").reshape(b.H_in, b.H_out)
    want = base + (ref.reshape(b.T, b.H_out) - gen.storage_to_f64(b.y_in, "bf16").reshape(b.T, b.H_out))
    assert np.isfinite(got).all()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= TOL["bf16"]
    pool.close()


@pytest.mark.parametrize("name", ["c2", "c2_zipf", "c1"])
def test_pad_max_rank_bgmv_mode(L, name):
    """LORA_OPT_PAD_MAX_RANK (padded BGMV) computes the same delta: zero rank rows add
    exact zeros, so the bf16 tensor-core path is bitwise equal to MBGMV; fp32 within tolerance."""
    from paper_2401_11240_b200 import binding as B
    b = {"c2": lambda: gen.config_c2(y_zero=False), "c2_zipf": lambda: gen.config_c2(zipf=True, y_zero=False, tag=4),
         "c1": lambda: gen.config_c1(y_zero=False)}[name]()
    outs = []
    for pad in (0, 1):
        pool = make_pool(b, L, L_tc=1 << 30)
        pool.set_option(B.LORA_OPT_PAD_MAX_RANK, pad)
        y, _ = run_gpu(b, L, pool=pool)
        outs.append(y)
        pool.close()
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(outs[1], ref, b.dtype) <= TOL[b.dtype]
    if b.dtype == "bf16":
        assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("kernel", [1, 0], ids=["gather_kernel", "memcpy"])
def test_load_paths_land_exact_bytes(L, kernel):
    """LORA_OPT_LOAD_KERNEL 1 (zero-copy gather kernel) and 0 (cudaMemcpyAsync, default) land the
    adapter bytes in its pages bitwise (read back, pin P12), including fragmented page runs, and the
    apply matches the oracle."""
    import torch
    from paper_2401_11240_b200 import binding as B
    b = gen.config_c2(y_zero=False)
    pool = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=sum(a.rank for a in b.adapters) + 64)
    pool.set_option(B.LORA_OPT_LOAD_KERNEL, kernel)
    # fragment the free list: load and unload a filler between adapters
    keep = []
    for i, a in enumerate(b.adapters):
        pool.load_adapter(a.id, a.rank, to_torch(a.A, pin=True), to_torch(a.B, pin=True), a.scale)
        if i == 3:
            filler = gen.make_adapter(1, 2, 999, 24, b.H_in, b.H_out, "bf16")
            pool.load_adapter(999, 24, to_torch(filler.A, pin=True), to_torch(filler.B, pin=True), 1.0)
            keep.append(filler)
        if i == 6:
            pool.unload_adapter(999)
    torch.cuda.synchronize()
    for a in b.adapters:
        A, Bm = pool.read_pages(a.id, a.rank)
        assert np.array_equal(A, a.A) and np.array_equal(Bm, a.B), a.id
    y, _ = run_gpu(b, L, pool=pool)
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
    pool.close()


def test_huge_decode_batch_metadata_upload_path(L):
    """A decode batch whose metadata (600 adapters, 4,000 one-token segments: ~12 K words even with
    1-word unit records) exceeds the kernel-parameter blob: the planner's blob goes to device memory
    through the PDL-chained upload kernel.  Result vs the oracle, eagerly and in a graph replay."""
    import torch
    rng = np.random.default_rng(0)
    H, n_ad, T = 256, 600, 4000
    ranks = {a: int(rng.choice([8, 16, 32, 64])) for a in range(n_ad)}
    ids = rng.integers(0, n_ad, size=T).astype(np.int32)
    b = gen.build_batch("huge", 31337, "bf16", H, H, [1] * T, ids, ranks, y_zero=False)
    pool = make_pool(b, L)
    y, md = run_gpu(b, L, pool=pool)
    assert md["G"] == len(set(ids.tolist()))
    ref = O.delta_for_batch(b, n_threads=16)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
    x = to_torch(b.x, "cuda")
    yg = to_torch(b.y_in, "cuda")
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        pool.apply(x, yg, b.seg_indptr, b.adapter_ids, stream=st)
    yg.copy_(to_torch(b.y_in, "cuda"))
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(from_torch(yg, "bf16"), y)
    pool.close()


def test_two_pools_on_two_streams_concurrently(L):
    """Distinct pools applied concurrently on two streams (own scratch each) give the same bits as
    serial applies."""
    import torch
    b1, b2 = gen.config_c2(y_zero=False, tag=1), gen.config_c2(y_zero=False, tag=2)
    p1, p2 = make_pool(b1, L), make_pool(b2, L)
    x1, x2 = to_torch(b1.x, "cuda"), to_torch(b2.x, "cuda")
    ys = [to_torch(b1.y_in, "cuda"), to_torch(b2.y_in, "cuda")]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(5):
        p1.apply(x1, ys[0], b1.seg_indptr, b1.adapter_ids, stream=s1)
        p2.apply(x2, ys[1], b2.seg_indptr, b2.adapter_ids, stream=s2)
    torch.cuda.synchronize()
    ser = [to_torch(b1.y_in, "cuda"), to_torch(b2.y_in, "cuda")]
    for _ in range(5):
        p1.apply(x1, ser[0], b1.seg_indptr, b1.adapter_ids)
        p2.apply(x2, ser[1], b2.seg_indptr, b2.adapter_ids)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ser[0]) and torch.equal(ys[1], ser[1])
    p1.close()
    p2.close()


@pytest.mark.parametrize("proj", ["q", "down"])
def test_c5_prefill_column_split(L, proj):
    """c5 prefill (8 x 512 tokens, 70B shapes): only 32 token tiles, so the planner gives every tile
    a split-K cluster of 4 CTAs (shrink K and expand columns split); full output vs the oracle, and
    the tcgen05 path is really taken."""
    b = gen.config_c5(proj, prefill=True, y_zero=False)
    y, md = run_gpu(b, L)
    assert md["n_prefill_tiles"] == 32
    assert md["prefill_cluster"] > 1 and md["n_prefill_ctas"] == 32 * md["prefill_cluster"]
    ref = O.delta_for_batch(b, n_threads=16)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]


def test_prefill_rank_129_to_256_on_tcgen05(L):
    """Prefill-length segments of rank 129..256 run on the tcgen05 kernel too (D1 up to 256 TMEM
    columns, the V operand in 64 KB, each column tile's B rows in two ring stages), next to rank
    <= 128 segments, in one apply; ragged lengths, odd ranks (zero-page padding), the oracle."""
    b = gen.build_batch("r200", 4711, "bf16", 512, 512, [300, 150, 1, 1], [0, 1, 0, 1], {0: 200, 1: 96},
                        y_zero=False)
    y, md = run_gpu(b, L)
    assert md["n_prefill_tiles"] == 3 + 2
    ref = O.delta_for_batch(b, n_threads=8)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_prefill_wide_ranks_vs_simt_and_oracle(L, seed):
    """Ranks 129..256 (incl. 129, 136, 255, 256) mixed with small ranks: the tcgen05 path (L_tc = 16)
    and the decode kernels alone both match the oracle; contiguous page runs (TMA boxes across the
    rank-128 boundary) and, for odd seeds, a fragmented free list (gather4 rows in both halves)."""
    rng = np.random.default_rng(100 + seed)
    lens = [int(v) for v in rng.integers(40, 420, size=5)]
    pick = [129, 136, 160, 200, 255, 256, 8, 64, 128]
    ranks = {i: int(r) for i, r in enumerate(rng.choice(pick, size=5, replace=False))}
    ranks[0] = [256, 129, 255, 200][seed]
    H_in, H_out = [(512, 512), (1024, 384), (256, 1024), (768, 256)][seed]
    b = gen.build_batch("wide%d" % seed, 5150 + seed, "bf16", H_in, H_out, lens, list(range(5)), ranks,
                        y_zero=bool(seed % 2))
    ref = O.delta_for_batch(b, n_threads=8)
    import torch
    pool = L.LoraPool(b.H_in, b.H_out, 16, "bf16", max_total_rank=sum(ranks.values()) + 64)
    pool.set_option(L.binding.LORA_OPT_TC_THRESHOLD, 16)
    if seed % 2:   # a 24-page hole at the front of the pool: adapter 0 (wide) straddles it and a spacer
        filler = gen.make_adapter(1, 2, 999, 24, b.H_in, b.H_out, "bf16")
        spacer = gen.make_adapter(1, 3, 997, 8, b.H_in, b.H_out, "bf16")
        pool.load_adapter(999, 24, to_torch(filler.A, pin=True), to_torch(filler.B, pin=True), 1.0)
        pool.load_adapter(997, 8, to_torch(spacer.A, pin=True), to_torch(spacer.B, pin=True), 1.0)
        pool.unload_adapter(999)
    for a in b.adapters:
        pool.load_adapter(a.id, a.rank, to_torch(a.A, pin=True), to_torch(a.B, pin=True), a.scale)
    if seed % 2:
        pg = pool.adapter_pages(0)
        assert pg[:24] == list(range(24)) and pg[24] == 32, pg[:30]
    torch.cuda.synchronize()
    y_tc, md = run_gpu(b, L, pool=pool)
    assert md["n_prefill_tiles"] == sum((n + 127) // 128 for n in lens)
    assert rel_l2(y_tc, ref, "bf16") <= TOL["bf16"]
    pool.close()
    y_simt, md_s = run_gpu(b, L, L_tc=1 << 30)
    assert md_s["n_prefill_tiles"] == 0
    assert rel_l2(y_simt, ref, "bf16") <= TOL["bf16"]


@pytest.mark.parametrize("H_in,H_out,n_tiles", [(4096, 1024, 2), (1024, 1024, 24), (1024, 4096, 3)])
def test_prefill_wide_rank_few_tiles(L, H_in, H_out, n_tiles):
    """Rank 256 / 200 / 144 on the few-tile paths: split-K clusters (partials of up to 256 columns
    in the L2 scratch, v rows over DSMEM) and the column split with shrink recompute."""
    rng = np.random.default_rng(n_tiles)
    lens = [128 * n_tiles - 37, 1, 1]
    ranks = {0: 256, 1: 200, 2: 144}
    b = gen.build_batch("wft%d" % n_tiles, 6000 + n_tiles, "bf16", H_in, H_out, lens, [0, 1, 2], ranks,
                        y_zero=False)
    y, md = run_gpu(b, L)
    assert md["n_prefill_tiles"] == n_tiles
    ref = O.delta_for_batch(b, n_threads=16)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
    del rng


def _few_tile_batch(name, seed, H_in, H_out, n_tiles):
    """Prefill segments (ragged lengths 65..400, ranks incl. 1 / 24 / 128) totalling exactly n_tiles
    128-token tiles, plus three decode tokens."""
    rng = np.random.default_rng(seed)
    lens, tiles = [], 0
    while tiles < n_tiles:
        ln = int(rng.integers(65, 401))
        t = -(-ln // 128)
        if tiles + t > n_tiles:
            ln = int(rng.integers(65, 129)) + 128 * (n_tiles - tiles - 1)
            t = n_tiles - tiles
        lens.append(ln)
        tiles += t
    ranks_cycle = (1, 8, 24, 128, 16, 64)
    n_ad = min(len(lens), 6)
    ids = [i % n_ad for i in range(len(lens))] + [0, 1 % n_ad, 0]
    lens = lens + [1, 1, 1]
    ranks = {a: ranks_cycle[a] for a in range(n_ad)}
    return gen.build_batch(name, seed, "bf16", H_in, H_out, lens, ids, ranks, y_zero=False)


@pytest.mark.parametrize("H_in,H_out,n_tiles", [
    (1024, 1024, 3), (1024, 1024, 20), (1024, 1024, 24), (1024, 1024, 27), (1024, 1024, 30),
    (1024, 1024, 40), (1024, 1024, 60), (1024, 4096, 2), (4096, 1024, 2)])
def test_prefill_few_tile_splits(L, H_in, H_out, n_tiles):
    """Few token tiles: the planner gives each tile `split` CTAs (N2 few-tile rule):
    split = min(H_out/128, SMs // tiles). For split <= 8, or when H_in > H_out, the tile's CTAs form a
    split-K cluster, capped at min(8, H_in/64); partial D1 tiles are summed in rank order. Otherwise
    every CTA recomputes the shrink for its share of the columns. Each case hits a different cluster
    size (8, 7, 6, 5, 4, 3, 2 on 148 SMs) or the recompute path. Full output vs the oracle."""
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    b = _few_tile_batch("few%d_%d_%d" % (H_in, H_out, n_tiles), 100 + n_tiles, H_in, H_out, n_tiles)
    y, md = run_gpu(b, L)
    assert md["n_prefill_tiles"] == n_tiles
    split = max(1, min(H_out // 128, sms // n_tiles))
    splitk = split <= 8 or H_in > H_out
    if splitk:
        split = min(split, 8, H_in // 64)
    assert md["n_prefill_ctas"] == n_tiles * split
    assert md["prefill_cluster"] == (split if splitk else 1)
    ref = O.delta_for_batch(b, n_threads=16)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]



@pytest.mark.gpu
def test_expand_unit_widths_multi_and_large_single(L):
    """Decode expand units of both sizing rules (DESIGN.md §6 N1): a q/k/v-style lora_apply_multi
    (widest <= 56 KB units, non-power-of-two widths, H_out = 1000 so the last unit of each gc is
    ragged) with chunks of 1..8 tokens (one and two token groups per MMA) == separate lora_apply
    calls bit for bit and within tolerance of the oracle; and a single-pool batch large enough to
    leave the power-of-two rule (256 adapters x 2 tokens) against the oracle."""
    import torch
    rng = np.random.default_rng(5150)
    lens = [int(v) for v in rng.integers(1, 9, size=40)]
    ids = [int(v) for v in rng.integers(0, 24, size=40)]
    ranks = {a: int(v) for a, v in enumerate(rng.choice([1, 8, 13, 16, 24, 32, 64, 100, 128], size=24))}
    shapes = [(1024, 1000), (1024, 256), (1024, 256)]
    batches = [gen.build_batch("wm%d" % i, 5150 + i, "bf16", hin, hout, lens, ids, ranks, y_zero=False)
               for i, (hin, hout) in enumerate(shapes)]
    batches[1].x = batches[0].x.copy()
    batches[2].x = batches[0].x.copy()
    pools = [make_pool(b, L) for b in batches]
    xs = [to_torch(b.x, "cuda") for b in batches]
    y_sep = [to_torch(b.y_in, "cuda") for b in batches]
    y_fus = [to_torch(b.y_in, "cuda") for b in batches]
    for p, x, y, b in zip(pools, xs, y_sep, batches):
        p.apply(x, y, b.seg_indptr, b.adapter_ids)
    L.apply_multi(pools, xs, y_fus, batches[0].seg_indptr, batches[0].adapter_ids)
    torch.cuda.synchronize()
    for b, ys_, yf in zip(batches, y_sep, y_fus):
        assert torch.equal(ys_, yf)
        ref = O.delta_for_batch(b, n_threads=8)
        assert rel_l2(from_torch(yf, "bf16"), ref, "bf16") <= TOL["bf16"]
    for p in pools:
        p.close()

    n_ad = 256
    big = gen.build_batch("wide", 5160, "bf16", 1024, 1000, [2] * n_ad, list(range(n_ad)),
                          {a: [8, 16, 32, 64][a % 4] for a in range(n_ad)}, y_zero=False)
    y, md = run_gpu(big, L)
    assert md["n_expand_units"] < sum(-(-1000 // c) for c in
                                      [1024 if r <= 16 else 32768 // (2 * r) for r in [8, 16, 32, 64] * 64])
    assert rel_l2(y, O.delta_for_batch(big, n_threads=8), "bf16") <= TOL["bf16"]


@pytest.mark.gpu
def test_plan_cache_follows_batch_and_table_changes(L):
    """The pool reuses its plan while (batch, adapter table, planner settings) are unchanged
    (pool.cpp plan_cached).  Alternating batches, a reload of an adapter id with another rank and
    pages, an option change and a multi-pool apply between single applies must all give the oracle's
    result (a stale plan would read wrong pages / ranks)."""
    import torch
    ba = gen.build_batch("pcA", 7100, "bf16", 512, 512, [1] * 12, list(range(12)),
                         {a: [8, 16, 24, 64][a % 4] for a in range(12)}, y_zero=False)
    bb = gen.build_batch("pcB", 7101, "bf16", 512, 512, [2, 1, 3], [3, 0, 7],
                         {a: [8, 16, 24, 64][a % 4] for a in range(12)}, y_zero=False)
    bb.adapters = ba.adapters   # one adapter set (the pool's), two batches over it
    pool = make_pool(ba, L, extra_pages=256)
    x_a, x_b = to_torch(ba.x, "cuda"), to_torch(bb.x, "cuda")

    def check(b, x):
        y = to_torch(b.y_in, "cuda")
        pool.apply(x, y, b.seg_indptr, b.adapter_ids)
        torch.cuda.synchronize()
        assert rel_l2(from_torch(y, "bf16"), O.delta_for_batch(b, n_threads=8), "bf16") <= TOL["bf16"]

    for b, x in ((ba, x_a), (ba, x_a), (bb, x_b), (ba, x_a), (bb, x_b)):
        check(b, x)
    # reload id 3 with another rank: same batch arrays, new table
    new3 = gen.make_adapter(gen.BASE_SEED + 9, 7103, 3, 40, 512, 512, "bf16")
    pool.unload_adapter(3)
    pool.load_adapter(3, new3.rank, to_torch(new3.A, pin=True), to_torch(new3.B, pin=True), new3.scale)
    ba.adapters = bb.adapters = [new3 if a.id == 3 else a for a in ba.adapters]
    check(ba, x_a)
    check(bb, x_b)
    # planner option change, then a multi-pool apply led by this pool, then a single apply again
    pool.set_option(L.binding.LORA_OPT_TC_THRESHOLD, 2)
    check(bb, x_b)
    other = make_pool(ba, L)
    ys = [to_torch(ba.y_in, "cuda"), to_torch(ba.y_in, "cuda")]
    L.apply_multi([pool, other], [x_a, x_a], ys, ba.seg_indptr, ba.adapter_ids)
    torch.cuda.synchronize()
    assert rel_l2(from_torch(ys[0], "bf16"), O.delta_for_batch(ba, n_threads=8), "bf16") <= TOL["bf16"]
    check(ba, x_a)
    pool.close()
    other.close()


@pytest.mark.gpu
def test_randomized_multi_sweep(L):
    """lora_apply_multi over 2..4 pools of random shapes sharing one random batch (decode and prefill
    segments, ranks 1..128, ids < 0): bitwise equal to separate lora_apply calls and within tolerance of
    the oracle.  Covers the multi-launch unit sizing (<= 56 KB expand units), 1-word and 3-word unit
    records and chunks of 1..8 tokens."""
    import torch
    rng = np.random.default_rng(4242)
    for trial in range(24):
        n_pools = int(rng.integers(2, 5))
        H_in = int(rng.integers(8, 97)) * 16
        lengths = [int(v) for v in rng.choice([1, 1, 2, 3, 5, 8, 9, 70], size=int(rng.integers(4, 60)))]
        n_ad = int(rng.integers(2, 40))
        ids = [int(rng.integers(0, n_ad)) if rng.random() > 0.1 else -1 for _ in lengths]
        H_outs = [int(rng.integers(1, 97)) * 16 for _ in range(n_pools)]
        rmax = min(128, H_in, min(H_outs))
        ranks = {a: int(rng.integers(1, rmax + 1)) for a in range(n_ad)}
        batches = []
        for p in range(n_pools):
            H_out = H_outs[p]
            b = gen.build_batch("ms%d_%d" % (trial, p), 9000 + 10 * trial + p, "bf16", H_in, H_out, lengths, ids, ranks,
                                y_zero=bool(p % 2))
            if p:
                b.x = batches[0].x.copy()
            batches.append(b)
        if batches[0].T == 0:
            continue
        pools = [make_pool(b, L) for b in batches]
        xs = [to_torch(b.x, "cuda") for b in batches]
        y_sep = [to_torch(b.y_in, "cuda") for b in batches]
        y_fus = [to_torch(b.y_in, "cuda") for b in batches]
        for p, x, y, b in zip(pools, xs, y_sep, batches):
            p.apply(x, y, b.seg_indptr, b.adapter_ids)
        L.apply_multi(pools, xs, y_fus, batches[0].seg_indptr, batches[0].adapter_ids)
        torch.cuda.synchronize()
        for b, ys_, yf in zip(batches, y_sep, y_fus):
            assert torch.equal(ys_, yf), (trial, b.H_in, b.H_out)
            ref = O.delta_for_batch(b, n_threads=8)
            assert rel_l2(from_torch(yf, "bf16"), ref, "bf16") <= TOL["bf16"], (trial, b.H_in, b.H_out)
        for p in pools:
            p.close()
