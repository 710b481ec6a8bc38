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
adapters replicated on every GPU; each GPU serves only requests for adapters it hosts, so there is
no data-path collective.
"""
from __future__ import annotations

import collections
from typing import Dict, Iterable, List, Optional, Tuple

import numpy as np

from .binding import LoraError, LoraPool


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
