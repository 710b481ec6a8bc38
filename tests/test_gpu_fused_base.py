"""NEXT f2 on the GPU: lora_apply_fused_base, y = x·W + s·(x·A)·B in one tcgen05 kernel, against the
fp64 oracle's delta plus x·W in fp64 (numpy on the same bf16 values).  PAPER.md Eq. 1,
§4.1 P:548-550.  The delta is checked on its own as well (y − x·W vs the oracle delta), so a large
base term cannot hide a wrong adapter contribution."""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

from gpu_util import TOL, from_torch, make_pool, rel_l2, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2401_11240_b200 as lib
    return lib


def _weight(seed, H_in, H_out):
    w = gen.storage_to_f64(gen.make_rows(seed, 77, 0, H_in, H_out, "bf16"), "bf16") / np.sqrt(H_in)
    return gen.f32_to_storage(w.astype(np.float32), "bf16")


def _fragmented_pool(b, L):
    """Adapters whose pages are NOT one run (the kernel's gather4 path): a rank-4 filler is loaded
    first and unloaded after the first adapter, so the next adapter's pages wrap around it."""
    pool = L.LoraPool(b.H_in, b.H_out, len(b.adapters) + 4, b.dtype,
                      max_total_rank=sum(a.rank for a in b.adapters) + 8)
    filler = np.zeros((4, b.H_in), np.uint16), np.zeros((4, b.H_out), np.uint16)
    pool.load_adapter(999, 4, to_torch(filler[0], pin=True), to_torch(filler[1], pin=True), 1.0)
    for i, a in enumerate(b.adapters):
        pool.load_adapter(a.id, a.rank, to_torch(a.A, pin=True), to_torch(a.B, pin=True), a.scale)
        if i == 0:
            pool.unload_adapter(999)
    return pool


def _check(L, b, W, fragmented=False):
    import torch
    pool = _fragmented_pool(b, L) if fragmented else make_pool(b, L)
    x = to_torch(b.x, "cuda")
    Wd = to_torch(W, "cuda")
    y = torch.full((b.T, b.H_out), 0x7fc0, dtype=torch.int16, device="cuda")   # NaN: every row must be written
    pool.apply_fused_base(x, Wd, y, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    got = gen.storage_to_f64(from_torch(y, "bf16"), "bf16").reshape(b.T, b.H_out)
    base = gen.storage_to_f64(b.x, "bf16").reshape(b.T, b.H_in) @ gen.storage_to_f64(W, "bf16").reshape(b.H_in, b.H_out)
    delta = O.delta_for_batch(b, n_threads=16).reshape(b.T, b.H_out)   # y_in = 0: the delta alone
    assert np.isfinite(got).all()
    full = np.linalg.norm(got - (base + delta)) / np.linalg.norm(base + delta)
    assert full <= TOL["bf16"], full
    # the delta alone: bf16 rounding of y (~2^-9 |y|) is the floor here, so the bound is looser
    d_err = np.linalg.norm((got - base) - delta) / np.linalg.norm(delta)
    assert d_err <= 2e-2, d_err
    # tokens without an adapter get exactly the base product (up to its one rounding)
    ids = np.repeat(b.adapter_ids, np.diff(b.seg_indptr))
    if (ids < 0).any():
        m = ids < 0
        assert np.linalg.norm(got[m] - base[m]) / np.linalg.norm(base[m]) <= TOL["bf16"]
    pool.close()
    return full, d_err


@pytest.mark.parametrize("fragmented", [False, True], ids=["box_loads", "gather4_loads"])
@pytest.mark.parametrize("H_out", [256, 768], ids=["one_ctile", "three_ctiles"])
def test_fused_base_ragged_small(L, fragmented, H_out):
    """Ragged segments (1..300 tokens, tails inside a tile; odd tile counts, so some 128-token tiles
    run without a pair partner), ranks 1 / 8 / 128, an id < 0 segment, an adapter used by two
    segments; one or three 256-column tiles; adapters in one page run (2D box loads in the shrink
    pass) or fragmented (gather4 loads)."""
    b = gen.build_batch("fb_small", 811, "bf16", 256, H_out, [300, 1, 128, 50, 129], [0, -1, 1, 2, 0],
                        {0: 8, 1: 128, 2: 1}, y_zero=True)
    W = _weight(5, 256, H_out)
    _check(L, b, W, fragmented)


def test_fused_base_prefill_mix(L):
    """8 prompts of 512 tokens at H = 1024 -> 2048 (16 column tiles), ranks 8..128."""
    ranks = {i: (8, 16, 32, 64, 128)[i % 5] for i in range(8)}
    b = gen.build_batch("fb_mix", 812, "bf16", 1024, 2048, [512] * 8, list(range(8)), ranks, y_zero=True)
    W = _weight(6, 1024, 2048)
    _check(L, b, W)


def test_fused_base_base_only_batch(L):
    """Every segment id < 0: no shrink pass, y = x·W (K loop without extension)."""
    b = gen.build_batch("fb_base", 816, "bf16", 512, 512, [130, 300], [-1, -1], {0: 8}, y_zero=True)
    import torch
    pool = make_pool(b, L)
    x = to_torch(b.x, "cuda")
    W = _weight(9, 512, 512)
    y = torch.full((b.T, b.H_out), 0x7fc0, dtype=torch.int16, device="cuda")
    pool.apply_fused_base(x, to_torch(W, "cuda"), y, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    got = gen.storage_to_f64(from_torch(y, "bf16"), "bf16").reshape(b.T, b.H_out)
    base = gen.storage_to_f64(b.x, "bf16").reshape(b.T, b.H_in) @ gen.storage_to_f64(W, "bf16").reshape(b.H_in, b.H_out)
    assert np.isfinite(got).all()
    assert np.linalg.norm(got - base) / np.linalg.norm(base) <= TOL["bf16"]
    pool.close()


def test_fused_base_rejects_unsupported(L):
    import torch
    b = gen.build_batch("fb_r200", 813, "bf16", 256, 256, [200], [0], {0: 200}, y_zero=True)
    pool = make_pool(b, L)
    x = to_torch(b.x, "cuda")
    y = torch.zeros((b.T, b.H_out), dtype=torch.int16, device="cuda")
    W = to_torch(_weight(7, 256, 256), "cuda")
    with pytest.raises(L.LoraError) as ei:
        pool.apply_fused_base(x, W, y, b.seg_indptr, b.adapter_ids)
    assert ei.value.name == "LORA_ERR_UNSUPPORTED"
    with pytest.raises(L.LoraError) as ei:
        pool.apply_fused_base(x, W, x, b.seg_indptr, b.adapter_ids)   # y overlaps x
    assert ei.value.name == "LORA_ERR_ARG"
    pool.close()
    b2 = gen.build_batch("fb_n384", 814, "bf16", 256, 384, [64], [0], {0: 8}, y_zero=True)   # hidden_out % 256
    pool = make_pool(b2, L)
    with pytest.raises(L.LoraError) as ei:
        pool.apply_fused_base(to_torch(b2.x, "cuda"), to_torch(_weight(7, 256, 384), "cuda"),
                              torch.zeros((b2.T, 384), dtype=torch.int16, device="cuda"), b2.seg_indptr, b2.adapter_ids)
    assert ei.value.name == "LORA_ERR_UNSUPPORTED"
    pool.close()


def test_fused_base_graph_capture_matches_eager(L):
    """The fused path allocates nothing and queries no event on a captured stream: a graph of it
    replays bitwise-equal to the eager call."""
    import torch
    b = gen.build_batch("fb_graph", 815, "bf16", 256, 512, [200, 64, 1], [0, 1, -1], {0: 16, 1: 64}, y_zero=True)
    pool = make_pool(b, L)
    x = to_torch(b.x, "cuda")
    W = to_torch(_weight(8, 256, 512), "cuda")
    y_eager = torch.zeros((b.T, b.H_out), dtype=torch.int16, device="cuda")
    y_graph = torch.zeros_like(y_eager)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pool.apply_fused_base(x, W, y_eager, b.seg_indptr, b.adapter_ids, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        pool.apply_fused_base(x, W, y_graph, b.seg_indptr, b.adapter_ids, stream=s)
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_eager, y_graph)
    pool.close()


def test_fused_base_rejects_fp32_pool(L):
    import torch
    pool = L.LoraPool(256, 256, 2, "f32", max_total_rank=8)
    x = torch.zeros((4, 256), dtype=torch.float32, device="cuda")
    with pytest.raises(L.LoraError) as ei:
        pool.apply_fused_base(x, x, torch.zeros_like(x), [0, 4], [-1])
    assert ei.value.name == "LORA_ERR_UNSUPPORTED"
    pool.close()


def test_fused_base_graph_replays_and_epochs(L):
    """The V items publish V behind per-tile flags holding the launch's epoch (advanced by every
    launch, never reset).  A graph of two fused calls (two batches, the second reusing the first's
    V tiles) replayed three times with new x each time, interleaved with eager calls, must match the
    eager results every time -- a stale flag from an earlier launch would let a column tile read an
    old V."""
    import torch
    b1 = gen.build_batch("fb_ep1", 817, "bf16", 512, 768, [300, 260], [0, 1], {0: 16, 1: 128}, y_zero=True)
    b2 = gen.build_batch("fb_ep2", 818, "bf16", 512, 768, [200, 356], [1, 0], {0: 16, 1: 128}, y_zero=True)
    b2.adapters = b1.adapters
    pool = make_pool(b1, L)
    W = to_torch(_weight(10, 512, 768), "cuda")
    x1 = to_torch(b1.x, "cuda")
    x2 = to_torch(b2.x, "cuda")
    yg1 = torch.zeros((b1.T, 768), dtype=torch.int16, device="cuda")
    yg2 = torch.zeros((b2.T, 768), dtype=torch.int16, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):   # warm-up outside the capture (scratch sizing)
        pool.apply_fused_base(x1, W, yg1, b1.seg_indptr, b1.adapter_ids, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        pool.apply_fused_base(x1, W, yg1, b1.seg_indptr, b1.adapter_ids, stream=s)
        pool.apply_fused_base(x2, W, yg2, b2.seg_indptr, b2.adapter_ids, stream=s)
    for rep in range(3):
        x1.copy_(torch.roll(x1, 1, 0))
        x2.copy_(torch.roll(x2, 3, 0))
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        ye1 = torch.zeros_like(yg1)
        ye2 = torch.zeros_like(yg2)
        pool.apply_fused_base(x2, W, ye2, b2.seg_indptr, b2.adapter_ids)
        pool.apply_fused_base(x1, W, ye1, b1.seg_indptr, b1.adapter_ids)
        torch.cuda.synchronize()
        assert torch.equal(yg1, ye1) and torch.equal(yg2, ye2), rep
    pool.close()
