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
profiles/r1_cost_model.json: MBGMV time vs sum_G r, R^2 0.92; padded BGMV vs G * max r, R^2 0.98).
Pure host logic (no CUDA); the hot path it schedules is lora_apply.
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


def feature_mbgmv(ranks: Sequence[int]) -> float:
    """sum of the batch's LoRA ranks.  Our kernel reads each distinct adapter once per
    8-token chunk; a request batch of distinct adapters is the paper's setting."""
    return float(sum(ranks))


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

    def dec_perf(self, ranks: Sequence[int]) -> float:
        if not ranks:
            return 0.0
        f = feature_mbgmv(ranks) if self.kind == "mbgmv" else feature_bgmv(ranks)
        return self.base_decode_us + self.invocations * self.decode(f)

    def pre_perf(self, prompts: Sequence[int]) -> float:
        if not prompts:
            return 0.0
        return self.prefill(float(sum(prompts)))

    @staticmethod
    def from_cost_model(path: str, kind: str = "mbgmv", **kw) -> "PerfModel":
        """The fit of scripts/cost_model.py (profiles/r1_cost_model.json), per-apply microseconds."""
        d = json.load(open(path))
        key = "mbgmv_time_vs_sum_rank_groups" if kind == "mbgmv" else "bgmv_time_vs_G_x_maxrank"
        f = d[key]
        return PerfModel(LinearModel(f["alpha_us_per_unit"], f["beta_us"], f["r2"]), kind=kind, **kw)


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
    dec_new = model.dec_perf(ranks + [req.rank])
    d_decode = dec_new - model.dec_perf(ranks)
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


# ---- baseline policies of the paper's scheduler evaluation
def pick_random(req, servers, rng: np.random.Generator) -> Server:
    c = [s for s in servers if s.can_serve(req)]
    return c[int(rng.integers(0, len(c)))]


def pick_most_idle(req, servers) -> Server:
    c = [s for s in servers if s.can_serve(req)]
    return min(c, key=lambda s: (len(s.running) + len(s.queue), s.sid))


def pick_first_fit(req, servers, model: PerfModel, slo_us: float) -> Server:
    c = [s for s in servers if s.can_serve(req)]
    for s in c:
        if model.dec_perf([e.rank for e in s.running + s.queue] + [req.rank]) <= slo_us:
            return s
    return c[0]


def simulate(policy: str, model: PerfModel, n_servers: int, requests: Sequence[Request], resp_len: int,
             arrival_gap_iters: float, slo_us: float, seed: int = 0) -> Dict[str, float]:
    """Discrete decode-iteration simulation of a cluster: requests arrive every arrival_gap_iters
    iterations, join the chosen server, prefill in the next iteration, then decode resp_len tokens;
    every iteration a server's per-token latency is DecPerf(running batch).  Returns the SLO
    attainment (fraction of decode iterations of requests whose per-token latency met the SLO) and
    the mean per-token latency."""
    rng = np.random.default_rng(seed)
    servers = [Server(i) for i in range(n_servers)]
    left: Dict[int, int] = {}
    met = total = 0
    lat_sum = 0.0
    pending = list(requests)
    t = 0.0
    next_arrival = 0.0
    while pending or any(s.running or s.queue for s in servers):
        while pending and next_arrival <= t:
            req = pending.pop(0)
            if policy == "rank_aware":
                s = rank_aware_pick(req, servers, model, avg_resp_len=resp_len, slo_us=slo_us)
            elif policy == "random":
                s = pick_random(req, servers, rng)
            elif policy == "most_idle":
                s = pick_most_idle(req, servers)
            elif policy == "first_fit":
                s = pick_first_fit(req, servers, model, slo_us)
            else:
                raise ValueError(policy)
            s.queue.append(req)
            left[req.rid] = resp_len
            next_arrival += arrival_gap_iters
        for s in servers:
            s.running += s.queue     # prefill this iteration, decode from the next
            s.queue = []
            if not s.running:
                continue
            lat = model.dec_perf([r.rank for r in s.running])
            for r in s.running:
                total += 1
                met += lat <= slo_us
                lat_sum += lat
                left[r.rid] -= 1
            s.running = [r for r in s.running if left[r.rid] > 0]
        t += 1.0
    return {"slo_attainment": met / max(1, total), "mean_token_latency_us": lat_sum / max(1, total)}
