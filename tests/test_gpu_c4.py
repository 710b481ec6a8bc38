"""Config 4 on the GPU: a Zipf-skewed adapter stream over a paged pool holding 20% of the
adapters' ranks, LRU eviction, cold-start loads overlapped with applies (no host sync between
steps).  Every step's result is checked against the oracle -- page reuse after unload must be
stream-ordered behind the applies that read the pages (pins P12/M4 under churn)."""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

from gpu_util import TOL, from_torch, rel_l2, to_torch

pytestmark = pytest.mark.gpu


def test_c4_churn_small(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2401_11240_b200 as L
    from paper_2401_11240_b200.serving import AdapterCache, HostRepository
    H, n_ad = 256, 60
    ads = {a: gen.make_adapter(gen.BASE_SEED + 3, 7, a, gen.c4_rank(a), H, H, "bf16") for a in range(n_ad)}
    repo = HostRepository()
    for a, ad in ads.items():
        repo.add(a, ad.rank, ad.scale, to_torch(ad.A, pin=True), to_torch(ad.B, pin=True))
    budget = sum(ad.rank for ad in ads.values()) * 2 // 5   # >= any step's working set
    pool = L.LoraPool(H, H, n_ad, "bf16", max_total_rank=budget)
    cache = AdapterCache(pool, repo, budget, n_ad)
    st = torch.cuda.Stream()
    outs = []
    for step in range(12):
        d = gen.config_c4_draw(step, n_decode=16, prefill_len=100, n_adapters=n_ad)
        ids = list(d["decode_ids"]) + [int(d["prefill_id"][0])]
        lens = [1] * 16 + [100]
        b = gen.build_batch("c4s%d" % step, 4242 + step, "bf16", H, H, lens, ids, {}, y_zero=False)
        b.adapters = [ads[a] for a in sorted(set(ids))]
        cache.ensure(ids)
        x = to_torch(b.x, "cuda")
        y = to_torch(b.y_in, "cuda")
        with torch.cuda.stream(st):
            pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
        outs.append((b, x, y))
    torch.cuda.synchronize()
    assert cache.evictions > 0 and cache.misses > 0
    for b, x, y in outs:
        ref = O.delta_for_batch(b, n_threads=8)
        assert rel_l2(from_torch(y, "bf16"), ref, "bf16") <= TOL["bf16"], b.name
    pool.close()


def test_c4_full_size_steps():
    """Config 4 at full size: Llama-2-13B 5120 -> 5120, 1000 adapters (ranks 8..128) in pinned host
    memory, a pool of 20% of their ranks, Zipf(1.0) draws of 64 decode tokens + one 512-token prefill
    segment per step (the prefill takes the tcgen05 kernel), LRU loads on the cache's side stream
    overlapping the applies; every step's full output vs the fp64 oracle."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2401_11240_b200 as L
    from paper_2401_11240_b200.serving import AdapterCache, HostRepository
    H, n_ad = 5120, 1000
    ads = {}
    repo = HostRepository()

    def adapter(a):
        if a not in ads:
            ads[a] = gen.c4_adapter(a, H)
            repo.add(a, ads[a].rank, ads[a].scale, to_torch(ads[a].A, pin=True), to_torch(ads[a].B, pin=True))
        return ads[a]

    budget = sum(gen.c4_rank(a) for a in range(n_ad)) // 5
    pool = L.LoraPool(H, H, n_ad, "bf16", max_total_rank=budget)
    cache = AdapterCache(pool, repo, budget, n_ad)
    st = torch.cuda.Stream()
    outs = []
    for step in range(5):
        d = gen.config_c4_draw(step)
        ids = [int(a) for a in d["decode_ids"]] + [int(d["prefill_id"][0])]
        for a in ids:
            adapter(a)
        lens = [1] * 64 + [512]
        b = gen.build_batch("c4full%d" % step, 9000 + step, "bf16", H, H, lens, ids, {}, y_zero=False)
        b.adapters = [ads[a] for a in sorted(set(ids))]
        cache.ensure(ids)
        x = to_torch(b.x, "cuda")
        y = to_torch(b.y_in, "cuda")
        with torch.cuda.stream(st):
            pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
        outs.append((b, x, y))   # x stays alive until the side-stream applies are done
    torch.cuda.synchronize()
    assert pool.metadata()["n_prefill_tiles"] == 4   # the 512-token segment ran on the tcgen05 kernel
    for b, _, y in outs:
        ref = O.delta_for_batch(b, n_threads=16)
        assert rel_l2(from_torch(y, "bf16"), ref, "bf16") <= TOL["bf16"], b.name
    pool.close()
