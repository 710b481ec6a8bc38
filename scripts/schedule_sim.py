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

rng = np.random.default_rng(1)
reqs = [S.Request(i, int(rng.integers(0, 200)), int(rng.choice([8, 16, 32, 64, 128], p=[.3, .25, .2, .15, .1])))
        for i in range(600)]
out = {"setup": __doc__.split("\n")[3:6], "results": []}
for kind, slos in (("mbgmv", (950, 1000, 1050, 1100)), ("bgmv", (1200, 1400, 1600, 2000))):
    m = S.PerfModel.from_cost_model(os.path.join(ROOT, "profiles", "r1_cost_model.json"), kind=kind)
    for slo in slos:
        row = {"kernel_model": kind, "slo_us_per_token": slo}
        for p in ("rank_aware", "random", "most_idle", "first_fit"):
            row[p] = round(S.simulate(p, m, 8, reqs, resp_len=64, arrival_gap_iters=0.6, slo_us=slo, seed=3)
                           ["slo_attainment"], 4)
        out["results"].append(row)
        print(row)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
