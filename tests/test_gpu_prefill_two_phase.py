"""GPU parity of the two-phase prefill path (LORA_OPT_PREFILL_TWO_PHASE): V = bf16(s·x·A) per 128-token
tile by the N2 kernel in V-out mode (split-K clusters when there are few tiles), then the persistent
2-CTA GEMM in delta mode adds V·B to y.  Same V and the same K-step order as the one-phase N2 kernel, so
the result is checked bitwise against it, and against the fp64 oracle within BASELINE.json's bf16
tolerance (SURVEY.md §8(c) GPU parity matrix): c1p tiles (ragged, ranks 1..128, H = 256), c3-shaped
(reduced), the 70B prefill shapes (split-K V pass), decode tokens and id < 0 segments in the same
batch, a fragmented pool, the fused q/k/v call and graph replay."""
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


def _apply(L, pool, b, two):
    import torch
    from paper_2401_11240_b200 import binding as B
    pool.set_option(B.LORA_OPT_PREFILL_TWO_PHASE, two)
    x = to_torch(b.x, "cuda")
    y = to_torch(b.y_in, "cuda")
    pool.apply(x, y, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    return from_torch(y, "bf16")


def _check(L, b, pool=None, oracle=True):
    own = pool is None
    pool = make_pool(b, L) if own else pool
    y1 = _apply(L, pool, b, 0)
    y2 = _apply(L, pool, b, 1)
    assert np.array_equal(y1, y2)
    if oracle:
        ref = O.delta_for_batch(b, n_threads=16)
        assert rel_l2(y2, ref, "bf16") <= TOL["bf16"]
    if own:
        pool.close()


@pytest.mark.parametrize("y_zero", [True, False], ids=["runA_delta", "runB_accumulate"])
def test_two_phase_prefill_tiles(L, y_zero):
    _check(L, gen.config_c1_prefill_tiles(y_zero=y_zero))


def test_two_phase_c3_reduced(L):
    _check(L, gen.config_c3(y_zero=False, n_seg=10, seg_len=384, H=1024))


@pytest.mark.parametrize("proj", ["q", "down", "k"])
def test_two_phase_c5_prefill_shapes(L, proj):
    _check(L, gen.config_c5(proj, y_zero=False, prefill=True), oracle=proj != "down")


def test_two_phase_mixed_decode_and_none(L):
    ranks = {0: 8, 1: 64, 2: 128, 3: 24}
    lengths = [1, 300, 5, 64, 129, 1, 700, 2, 255]
    ids = [0, 1, 2, -1, 3, 1, 0, -1, 2]
    b = gen.build_batch("tp_mix", 2201, "bf16", 512, 768, lengths, ids, ranks, y_zero=False)
    _check(L, b)


def test_two_phase_fragmented_pool(L):
    b = gen.build_batch("tp_frag", 2202, "bf16", 512, 512, [200, 300], [0, 1], {0: 40, 1: 72}, y_zero=False)
    pool = L.LoraPool(b.H_in, b.H_out, 8, "bf16", max_total_rank=200)
    filler = np.zeros((4, b.H_in), np.uint16), np.zeros((4, b.H_out), np.uint16)
    pool.load_adapter(99, 4, to_torch(filler[0], pin=True), to_torch(filler[1], pin=True), 1.0)
    for i, a in enumerate(b.adapters):
        pool.load_adapter(a.id, a.rank, to_torch(a.A, pin=True), to_torch(a.B, pin=True), a.scale)
        if i == 0:
            pool.unload_adapter(99)
    _check(L, b, pool=pool)
    pool.close()


def test_two_phase_multi_and_graph(L):
    import torch
    from paper_2401_11240_b200 import binding as B
    shapes = [(512, 512), (512, 256), (512, 256)]
    lengths, ids = [300, 1, 200], [0, 1, 2]
    bs = [gen.build_batch("tpm%d" % i, 2210 + i, "bf16", hi, ho, lengths, ids, {0: 16, 1: 8, 2: 96}, y_zero=False)
          for i, (hi, ho) in enumerate(shapes)]
    for b in bs[1:]:
        b.x = bs[0].x.copy()
    pools = [make_pool(b, L) for b in bs]
    xs = [to_torch(b.x, "cuda") for b in bs]
    outs = {}
    for two in (0, 1):
        for p in pools:
            p.set_option(B.LORA_OPT_PREFILL_TWO_PHASE, two)
        ys = [to_torch(b.y_in, "cuda") for b in bs]
        L.apply_multi(pools, xs, ys, bs[0].seg_indptr, bs[0].adapter_ids)
        torch.cuda.synchronize()
        outs[two] = [y.clone() for y in ys]
        if two == 1:   # graph replay of the two-phase call
            yg = [to_torch(b.y_in, "cuda") for b in bs]
            st = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                L.apply_multi(pools, xs, yg, bs[0].seg_indptr, bs[0].adapter_ids, stream=st)
            for y, b in zip(yg, bs):
                y.copy_(to_torch(b.y_in, "cuda"))
            with torch.cuda.stream(st):
                g.replay()
            torch.cuda.synchronize()
            for a_, b_ in zip(yg, outs[1]):
                assert torch.equal(a_, b_)
    for b, y0, y1 in zip(bs, outs[0], outs[1]):
        assert torch.equal(y0, y1)
        assert rel_l2(from_torch(y1, "bf16"), O.delta_for_batch(b, n_threads=8), "bf16") <= TOL["bf16"]
    for p in pools:
        p.close()
