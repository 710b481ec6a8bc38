"""Adapter residency management for serving (config 4): an LRU cache of adapters over one paged
pool, fed from a host-memory adapter repository.

PAPER.md §2.3 C1: adapters live in host memory and are fetched to the GPU on demand;
the fetch (cold start) takes "a few to tens of milliseconds" and is 10-20% of serving time.  Here a
miss enqueues lora_load_adapter (pinned host -> HBM pages on the pool's side stream, returns
immediately); the next lora_apply on a compute stream waits on the load's ready event only if it
is still in flight, so loads overlap the applies of other adapters.  Eviction is least-recently-
used with ties broken by the lower id, and frees pages at call time; the
library orders their physical reuse after the applies already enqueued.

Request placement across GPUs: adapter home GPU = id mod N, the hottest
adapters replicated on every GPU; a request goes to one of the GPUs hosting its adapter, chosen by
the paper's rank-aware Algorithm 1 (scheduler.rank_aware_pick with the cost model fitted
to this library's decode kernel) -- route_requests.  Each GPU then serves its requests alone: there
is no data-path collective.
"""
from __future__ import annotations

import collections
from typing import Dict, Iterable, List, Optional, Tuple

import numpy as np

from .binding import LoraError, LoraPool
from . import scheduler as S


class HostRepository:
    """Adapters in (pinned) host memory: id -> (rank, scale, A [r][H_in], B [r][H_out])."""

    def __init__(self):
        self.items: Dict[int, Tuple[int, float, object, object]] = {}

    def add(self, aid: int, rank: int, scale: float, A, B) -> None:
        self.items[int(aid)] = (int(rank), float(scale), A, B)

    def __contains__(self, aid) -> bool:
        return int(aid) in self.items

    def bytes_of(self, aid: int, elem_bytes: int) -> int:
        r, _, A, B = self.items[int(aid)]
        return r * (A.shape[1] + B.shape[1]) * elem_bytes


def home_gpu(aid: int, world: int, replicated: Iterable[int] = ()) -> Optional[int]:
    """Placement rule: None = replicated everywhere, else the home rank."""
    if aid in set(replicated):
        return None
    return int(aid) % world


def serves(aid: int, rank: int, world: int, replicated: Iterable[int] = ()) -> bool:
    h = home_gpu(aid, world, replicated)
    return h is None or h == rank


def route_requests(decode_ids, prefill_ids, prefill_len: int, world: int, replicated: Iterable[int],
                   model: "S.PerfModel", rank_of, avg_resp_len: float = 128.0, slo_us: float = float("inf"),
                   penalty: float = 1e9) -> Tuple[List[int], List[int]]:
    """Algorithm 1 over one step's requests, in arrival order (decode requests, then the
    prompts): each goes to the candidate GPU -- those hosting its adapter (home_gpu) -- with the
    minimum total cost = CalcCost x (running + queued requests), CalcCost from the fitted DecPerf /
    PrePerf models (scheduler.calc_cost); ties go to the lower GPU.  Deterministic: every rank runs
    it on the same global request list and keeps its own share.  Returns the GPU of every decode
    request and of every prompt."""
    servers = [S.Server(g) for g in range(world)]
    rep = set(int(a) for a in replicated)

    def cands(aid):
        h = home_gpu(aid, world, rep)
        return servers if h is None else [servers[h]]

    dec_to, pre_to = [], []
    for i, a in enumerate(decode_ids):
        a = int(a)
        req = S.Request(i, a, int(rank_of(a)), prompt_len=0)
        s = S.rank_aware_pick(req, cands(a), model, avg_resp_len=avg_resp_len, slo_us=slo_us, penalty=penalty)
        s.running.append(req)
        dec_to.append(s.sid)
    for i, a in enumerate(prefill_ids):
        a = int(a)
        req = S.Request(len(dec_to) + i, a, int(rank_of(a)), prompt_len=int(prefill_len))
        s = S.rank_aware_pick(req, cands(a), model, avg_resp_len=avg_resp_len, slo_us=slo_us, penalty=penalty)
        s.queue.append(req)
        pre_to.append(s.sid)
    return dec_to, pre_to


class AdapterCache:
    """LRU residency of adapters in one LoraPool."""

    def __init__(self, pool: LoraPool, repo: HostRepository, page_budget: int, max_adapters: int):
        self.pool = pool
        self.repo = repo
        self.page_budget = int(page_budget)
        self.max_adapters = int(max_adapters)
        self.lru: "collections.OrderedDict[int, int]" = collections.OrderedDict()   # id -> rank, LRU first
        self.pages_used = 0
        self.hits = 0
        self.misses = 0
        self.loaded_bytes = 0
        self.evictions = 0

    def _evict_one(self, protect) -> None:
        # least recently used; among entries of equal recency the lower id (OrderedDict order is
        # exact recency, ties only arise within one ensure() call -> resolved by ascending id)
        for aid in self.lru:
            if aid not in protect:
                r = self.lru.pop(aid)
                self.pool.unload_adapter(aid)
                self.pages_used -= r
                self.evictions += 1
                return
        raise LoraError(6, "cannot make room: every resident adapter is needed by this batch")

    def ensure(self, ids: Iterable[int]) -> List[int]:
        """Make every id in `ids` resident (loading misses); returns the ids loaded now."""
        need = sorted(set(int(a) for a in ids if int(a) >= 0))
        protect = set(need)
        loaded = []
        for aid in need:
            if aid in self.lru:
                self.hits += 1
                self.lru.move_to_end(aid)
                continue
            self.misses += 1
            r, s, A, B = self.repo.items[aid]
            while self.pages_used + r > self.page_budget or len(self.lru) >= self.max_adapters:
                self._evict_one(protect)
            self.pool.load_adapter(aid, r, A, B, s)
            self.lru[aid] = r
            self.pages_used += r
            self.loaded_bytes += self.repo.bytes_of(aid, 2 if self.pool.dtype == "bf16" else 4)
            loaded.append(aid)
        # recency of this batch: ascending id among the batch's adapters
        for aid in need:
            self.lru.move_to_end(aid)
        return loaded

    @property
    def hit_rate(self) -> float:
        n = self.hits + self.misses
        return self.hits / n if n else 0.0
