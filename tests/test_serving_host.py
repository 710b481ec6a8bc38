"""CPU tests of the config-4 serving host logic (LRU adapter residency over a paged pool and
request placement), on host-only pools (no CUDA), checked against the oracle allocator replay."""
import numpy as np

from oracle import oracle as O
from workloads import gen

import paper_2401_11240_b200 as L
from paper_2401_11240_b200.serving import AdapterCache, HostRepository, home_gpu, serves


def _repo(n, ranks):
    repo = HostRepository()
    for a in range(n):
        r = ranks[a % len(ranks)]
        repo.add(a, r, 16.0 / r, np.zeros((r, 32), np.float32), np.zeros((r, 32), np.float32))
    return repo


def test_lru_cache_matches_allocator_replay():
    n_pages, max_ad = 60, 10
    pool = L.LoraPool(32, 32, max_ad, "f32", max_total_rank=n_pages, host_only=True)
    repo = _repo(30, [4, 8, 16])
    cache = AdapterCache(pool, repo, page_budget=n_pages, max_adapters=max_ad)
    ref = O.PageAllocatorReplay(n_pages, max_ad)
    lru = []
    rng = np.random.default_rng(0)
    for step in range(200):
        ids = sorted(set(int(v) for v in rng.integers(0, 30, size=int(rng.integers(1, 4)))))
        # reference LRU policy
        for a in ids:
            if a in lru:
                continue
            r = repo.items[a][0]
            while sum(ref.table[b][0] for b in lru) + r > n_pages or len(lru) >= max_ad:
                victim = next(b for b in lru if b not in ids)
                lru.remove(victim)
                ref.unload(victim)
            ref.load(a, r, repo.items[a][1])
            lru.append(a)
        for a in ids:
            lru.remove(a)
            lru.append(a)
        cache.ensure(ids)
        assert list(cache.lru) == lru
        for a in lru:
            assert pool.adapter_pages(a) == ref.pages_of(a)
        assert pool.info()["free_pages"] == sum(ref.free)
    assert cache.hits + cache.misses > 0 and cache.evictions > 0
    pool.close()


def test_placement_partitions_every_request_once():
    reqs = gen.config_c4_draw(step=1, n_decode=256)["decode_ids"]
    hot = list(range(16))
    for world in (1, 2, 4, 8):
        owners = [[r for r in range(world) if serves(int(a), r, world, hot)] for a in reqs]
        for a, o in zip(reqs, owners):
            if int(a) in hot:
                assert o == list(range(world))       # replicated
            else:
                assert o == [home_gpu(int(a), world, hot)]


def test_zipf_popularity_matches_survey_figures():
    """Zipf(1.0) over 1000 ids: top-1 ~13.4%, top-16 ~45.2%, top-200 ~78.5% of draws."""
    k = np.arange(1, 1001, dtype=np.float64)
    p = 1 / k
    p /= p.sum()
    assert abs(p[:1].sum() - 0.134) < 0.002 and abs(p[:16].sum() - 0.452) < 0.002
    assert abs(p[:200].sum() - 0.785) < 0.002
