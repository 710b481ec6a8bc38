"""Rank-aware scheduling (Algorithm 1) vs the paper's baselines (Random, MostIdle,
FirstFit) in a seeded cluster simulation driven by the performance models fitted to
this library's decode kernels (profiles/r1_cost_model.json).  8 servers, 600 requests, ranks
8..128 (30/25/20/15/10 %), 64 decode tokens each, one arrival per 0.6 decode iterations.
usage: python scripts/schedule_sim.py [out.json]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_11240_b200 import scheduler as S  # noqa: E402
from paper_2401_11240_b200.scheduler import PerfModel, Request, Server, rank_aware_pick  # noqa: E402,F401
from typing import Dict, Sequence  # noqa: E402

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



rng = np.random.default_rng(1)
reqs = [S.Request(i, int(rng.integers(0, 200)), int(rng.choice([8, 16, 32, 64, 128], p=[.3, .25, .2, .15, .1])))
        for i in range(600)]
out = {"setup": __doc__.split("\n")[3:6], "results": []}
for kind, slos in (("mbgmv", (950, 1000, 1050, 1100)), ("bgmv", (1200, 1400, 1600, 2000))):
    m = S.PerfModel.from_cost_model(os.path.join(ROOT, "profiles", "r1_cost_model.json"), kind=kind)
    for slo in slos:
        row = {"kernel_model": kind, "slo_us_per_token": slo}
        for p in ("rank_aware", "random", "most_idle", "first_fit"):
            row[p] = round(simulate(p, m, 8, reqs, resp_len=64, arrival_gap_iters=0.6, slo_us=slo, seed=3)
                           ["slo_attainment"], 4)
        out["results"].append(row)
        print(row)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
