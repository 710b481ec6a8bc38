"""Rank-aware request scheduling across inference servers.

PAPER.md §4.3: per-batch LoRA kernel latency is linear in a rank feature of the batch --
    Perf_BGMV(S)  = alpha_B * |S| * max_{i in S} rank(i) + beta_B      (padded kernel)
    Perf_MBGMV(S) = alpha_M * sum_{i in S} rank(i) + beta_M              (padding-free)
-- fitted by profiling (R^2 = 0.96 in the paper).  Algorithm 1 routes each arriving
request to the candidate server with the minimum total cost, where
    cost  = (PrePerf(queue + req) - PrePerf(queue)) / avg_resp_len
          + (DecPerf(exists + req) - DecPerf(exists))          [+ penalty if DecPerf(exists + req) > SLO]
    total = cost * (len(running_batch) + len(queue)).

Here the models are fitted to this library's measured kernels (scripts/cost_model.py ->
profiles/r1_cost_model.json: MBGMV time vs sum over (adapter, 8-token chunk) of r, R^2 0.957; padded
BGMV vs G * max r, R^2 0.98).  Pure host logic (no CUDA); the hot path it schedules is lora_apply.
serving.route_requests applies Algorithm 1 to a decode step's requests across the GPUs of a node
(bench.py config 4); the cluster simulation against the paper's baseline policies is evaluation,
not product (scripts/schedule_sim.py).
"""
from __future__ import annotations

import dataclasses
import json
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np


@dataclasses.dataclass
class LinearModel:
    """t = alpha * feature + beta (microseconds per kernel invocation)."""
    alpha: float
    beta: float
    r2: float = float("nan")

    @staticmethod
    def fit(features: Sequence[float], times: Sequence[float]) -> "LinearModel":
        x = np.asarray(features, dtype=np.float64)
        y = np.asarray(times, dtype=np.float64)
        A = np.stack([x, np.ones_like(x)], axis=1)
        (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
        pred = A @ np.array([a, b])
        ss = float(((y - y.mean()) ** 2).sum())
        r2 = 1.0 - float(((y - pred) ** 2).sum()) / ss if ss > 0 else 1.0
        return LinearModel(float(a), float(b), r2)

    def __call__(self, feature: float) -> float:
        return self.alpha * feature + self.beta


CHUNK = 8   # decode tokens per (adapter group, token chunk) unit of the kernel (kTokChunkMma)


def feature_mbgmv(ranks: Sequence[int], adapters: Optional[Sequence[int]] = None) -> float:
    """The padding-free kernel's rank feature (P:753-757 sums the ranks of the batch's requests).
    The model is fitted (profiles/r1_cost_model.json, "mbgmv_time_vs_sum_rank_gc", R^2 0.957) on what
    this library's decode kernel reads: every DISTINCT adapter's rank rows once per 8-token chunk,
    sum over adapters of r * ceil(tokens / 8).  With `adapters` (the adapter id of each request,
    parallel to `ranks`) that is what is computed; without, every request is its own adapter (the
    paper's setting, where the two coincide)."""
    if adapters is None:
        return float(sum(ranks))
    count: Dict[int, int] = {}
    rank_of: Dict[int, int] = {}
    for a, r in zip(adapters, ranks):
        count[a] = count.get(a, 0) + 1
        rank_of[a] = r
    return float(sum(rank_of[a] * -(-n // CHUNK) for a, n in count.items()))


def feature_bgmv(ranks: Sequence[int]) -> float:
    """|S| * max rank."""
    return float(len(ranks) * max(ranks)) if ranks else 0.0


@dataclasses.dataclass
class PerfModel:
    """DecPerf / PrePerf of Algorithm 1.  kind: "mbgmv" or "bgmv" (the decode kernel in use).
    DecPerf(S) = n_layers_proj * kernel(S): a decode iteration invokes the delta once per adapted
    projection (32 invocations for Llama-2-7B W_Q/W_K/W_V ... P:133); the base model's own time is
    a constant offset folded into beta_total.  PrePerf(queue) = alpha_p * prompt tokens + beta_p."""
    decode: LinearModel
    kind: str = "mbgmv"
    invocations: int = 128            # 32 layers x q/k/v/o
    base_decode_us: float = 0.0       # base-model time per decode iteration (constant)
    prefill: LinearModel = dataclasses.field(default_factory=lambda: LinearModel(0.0, 0.0))

    def dec_perf(self, ranks: Sequence[int], adapters: Optional[Sequence[int]] = None) -> float:
        """adapters: the adapter id of each request (MBGMV: distinct adapters per 8-token chunk)."""
        if not ranks:
            return 0.0
        f = feature_mbgmv(ranks, adapters) if self.kind == "mbgmv" else feature_bgmv(ranks)
        return self.base_decode_us + self.invocations * self.decode(f)

    def pre_perf(self, prompts: Sequence[int]) -> float:
        if not prompts:
            return 0.0
        return self.prefill(float(sum(prompts)))

    @staticmethod
    def from_cost_model(path: str, kind: str = "mbgmv", **kw) -> "PerfModel":
        """The fit of scripts/cost_model.py (profiles/r1_cost_model.json), per-apply microseconds."""
        d = json.load(open(path))
        key = "mbgmv_time_vs_sum_rank_gc" if kind == "mbgmv" else "bgmv_time_vs_G_x_maxrank"
        f = d[key]
        return PerfModel(LinearModel(f["alpha_us_per_unit"], f["beta_us"], f["r2"]), kind=kind, **kw)


def measured_model(kind: str = "mbgmv", invocations: int = 128) -> PerfModel:
    """The models fitted to this library's kernels on B200 (scripts/cost_model.py ->
    profiles/r1_cost_model.json: MBGMV us per apply = 0.0037362 * sum_gc r + 5.4006, R^2 0.957;
    padded BGMV = 0.0084753 * G * max r + 3.5120, R^2 0.977) and the tcgen05 prefill apply (bench
    config 3: 88 us for 16,384 tokens, i.e. 5.37 ns per token per apply), per decode iteration of
    `invocations` applies."""
    dec = LinearModel(0.0037362, 5.4006, 0.957) if kind == "mbgmv" else LinearModel(0.0084753, 3.5120, 0.977)
    pre = LinearModel(invocations * 88.0 / 16384, invocations * 5.0)
    return PerfModel(dec, kind=kind, invocations=invocations, prefill=pre)


@dataclasses.dataclass
class Request:
    rid: int
    adapter: int
    rank: int
    prompt_len: int = 128


@dataclasses.dataclass
class Server:
    """What Algorithm 1's GetStats() returns, plus the adapters the server can serve."""
    sid: int
    running: List[Request] = dataclasses.field(default_factory=list)   # decoding
    queue: List[Request] = dataclasses.field(default_factory=list)     # waiting for prefill
    adapters: Optional[set] = None    # None = can serve any adapter (loads on demand)

    def can_serve(self, req: Request) -> bool:
        return self.adapters is None or req.adapter in self.adapters


def calc_cost(req: Request, server: Server, model: PerfModel, avg_resp_len: float, slo_us: float,
              penalty: float) -> float:
    """Algorithm 1, CalcCost."""
    exists = server.running + server.queue
    d_prefill = model.pre_perf([q.prompt_len for q in server.queue] + [req.prompt_len]) - \
        model.pre_perf([q.prompt_len for q in server.queue])
    ranks = [e.rank for e in exists]
    ads = [e.adapter for e in exists]
    dec_new = model.dec_perf(ranks + [req.rank], ads + [req.adapter])
    d_decode = dec_new - model.dec_perf(ranks, ads)
    cost = d_prefill / avg_resp_len + d_decode
    if dec_new > slo_us:
        cost += penalty
    return cost


def rank_aware_pick(req: Request, servers: Sequence[Server], model: PerfModel, avg_resp_len: float = 128.0,
                    slo_us: float = 36_000.0, penalty: float = 1e9) -> Server:
    """Algorithm 1 main loop body: candidates = servers able to serve the request;
    total_cost = CalcCost * (len(running) + len(queue)); the minimum wins (ties -> lower sid)."""
    cands = [s for s in servers if s.can_serve(req)]
    if not cands:
        raise ValueError("no server can serve adapter %d" % req.adapter)
    best, best_cost = None, None
    for s in cands:
        n = len(s.running) + len(s.queue)
        total = calc_cost(req, s, model, avg_resp_len, slo_us, penalty) * n
        if best is None or total < best_cost:
            best, best_cost = s, total
    return best
