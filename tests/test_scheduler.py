"""CPU tests of the rank-aware scheduler (paper_2401_11240_b200/scheduler.py; §4.3,
Algorithm 1): linear performance models, CalcCost, the selection rule, and a seeded
cluster simulation against the paper's baseline policies."""
import os

import numpy as np
import pytest

from paper_2401_11240_b200 import scheduler as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_linear_model_fit_recovers_exact_line():
    x = np.array([8, 40, 100, 960, 3000], dtype=float)
    m = S.LinearModel.fit(x, 0.0125 * x + 3.5)
    assert abs(m.alpha - 0.0125) < 1e-12 and abs(m.beta - 3.5) < 1e-9 and abs(m.r2 - 1.0) < 1e-12


def test_features_follow_the_paper():
    # BGMV: |S| * max rank; MBGMV: sum of ranks
    assert S.feature_bgmv([8, 64, 16]) == 3 * 64
    assert S.feature_mbgmv([8, 64, 16]) == 88
    assert S.feature_bgmv([]) == 0.0


def _model(kind="mbgmv", alpha=0.01, beta=5.0, inv=10, pre=(0.02, 1.0)):
    return S.PerfModel(S.LinearModel(alpha, beta), kind=kind, invocations=inv,
                       prefill=S.LinearModel(*pre))


def test_calc_cost_by_hand():
    m = _model()
    srv = S.Server(0, running=[S.Request(1, 1, 16)], queue=[S.Request(2, 2, 32, prompt_len=100)])
    req = S.Request(3, 3, 64, prompt_len=50)
    # prefill: PrePerf(queue + req) - PrePerf(queue) = 0.02 * 50; per token: / avg_resp_len 10
    # decode: 10 * 0.01 * 64 (MBGMV delta is the added rank)
    exp = 0.02 * 50 / 10 + 10 * 0.01 * 64
    assert abs(S.calc_cost(req, srv, m, avg_resp_len=10, slo_us=1e9, penalty=1e6) - exp) < 1e-9
    # SLO violation adds the penalty: DecPerf(exists + req) = 10 * (0.01 * 112 + 5) = 61.2 > 60
    assert S.calc_cost(req, srv, m, avg_resp_len=10, slo_us=60.0, penalty=1e6) > 1e6


def test_idle_server_wins_and_ties_go_to_lower_id():
    m = _model()
    busy = S.Server(0, running=[S.Request(1, 1, 8)])
    idle1, idle2 = S.Server(1), S.Server(2)
    assert S.rank_aware_pick(S.Request(9, 9, 64), [busy, idle1, idle2], m).sid == 1


def test_slo_penalty_steers_away():
    m = _model(inv=100)
    a = S.Server(0, running=[S.Request(i, i, 128) for i in range(3)])      # sum r 384
    b = S.Server(1, running=[S.Request(10 + i, i, 8) for i in range(3)])   # sum r 24
    req = S.Request(99, 5, 128)
    # DecPerf(a + req) = 100 * (0.01 * 512 + 5) = 1012 > 1000; b: 100 * (0.01 * 152 + 5) = 652
    assert S.rank_aware_pick(req, [a, b], m, slo_us=1000.0).sid == 1


def test_bgmv_model_groups_similar_ranks():
    """Under the padded kernel the added cost depends on the batch's max rank: a rank-64 request is
    cheaper on a server already padding to 128 (delta = 128 alpha) than on one at rank 8
    (delta = 3*64 - 2*8 = 176 alpha) -- the rank-aware behaviour the paper motivates."""
    m = _model(kind="bgmv")
    hi = S.Server(0, running=[S.Request(1, 1, 128), S.Request(2, 2, 128)])
    lo = S.Server(1, running=[S.Request(3, 3, 8), S.Request(4, 4, 8)])
    assert S.rank_aware_pick(S.Request(5, 5, 64), [lo, hi], m).sid == 0


def test_candidates_respect_adapter_placement():
    m = _model()
    a = S.Server(0, adapters={1, 2})
    b = S.Server(1, running=[S.Request(7, 3, 8)], adapters={3})
    assert S.rank_aware_pick(S.Request(8, 3, 16), [a, b], m).sid == 1
    with pytest.raises(ValueError):
        S.rank_aware_pick(S.Request(9, 4, 16), [a, b], m)


@pytest.mark.parametrize("kind,slo", [("mbgmv", 1000.0), ("bgmv", 1400.0)])
def test_simulation_rank_aware_beats_random_and_most_idle(kind, slo):
    """Seeded cluster simulation (8 servers, 600 requests, ranks 8..128) with the models fitted to
    this library's kernels (profiles/r1_cost_model.json): rank-aware SLO attainment exceeds the
    Random and MostIdle baselines (the paper: 99% SLO)."""
    m = S.PerfModel.from_cost_model(os.path.join(ROOT, "profiles", "r1_cost_model.json"), kind=kind)
    rng = np.random.default_rng(1)
    reqs = [S.Request(i, int(rng.integers(0, 200)), int(rng.choice([8, 16, 32, 64, 128], p=[.3, .25, .2, .15, .1])))
            for i in range(600)]
    res = {p: S.simulate(p, m, 8, reqs, resp_len=64, arrival_gap_iters=0.6, slo_us=slo, seed=3)["slo_attainment"]
           for p in ("rank_aware", "random", "most_idle")}
    assert res["rank_aware"] > res["random"] + 0.1 and res["rank_aware"] > res["most_idle"] + 0.1, res
