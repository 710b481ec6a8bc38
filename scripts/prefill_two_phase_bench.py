"""c3 and c5 prefill shapes: one-phase N2 kernel vs the two-phase path (LORA_OPT_PREFILL_TWO_PHASE),
µs per apply from CUDA graphs of NP applies on distinct pools (x/y >> L2), median of reps.
usage: python scripts/prefill_two_phase_bench.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from paper_2401_11240_b200 import binding as B  # noqa: E402
from workloads import gen  # noqa: E402

peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
NP = 4


def bench(b, name):
    pools = []
    for _ in range(NP):
        p = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
        for a in b.adapters:
            p.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                           torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
        pools.append(p)
    xs = [torch.from_numpy(b.x.view(np.int16)).cuda() for _ in range(NP)]
    ys = [torch.zeros(b.T, b.H_out, dtype=torch.int16, device="cuda") for _ in range(NP)]
    st = torch.cuda.Stream()
    sum_r = sum(a.rank for a in b.adapters)
    byts = 2 * (sum_r * (b.H_in + b.H_out) + b.T * b.H_in + 2 * b.T * b.H_out)
    out = {"shape": [b.H_in, b.H_out], "T": b.T}
    for two in (0, 1):
        for p in pools:
            p.set_option(B.LORA_OPT_PREFILL_TWO_PHASE, two)
        def run():
            for p, x, y in zip(pools, xs, ys):
                p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
        with torch.cuda.stream(st):
            run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            run()
        ts = []
        for _ in range(9):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st):
                g.replay()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / NP)
        us = float(np.median(ts))
        out["two_phase" if two else "one_phase"] = {"us": round(us, 1),
                                                    "roofline_frac": round(byts / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 3)}
    for p in pools:
        p.close()
    print(name, json.dumps(out), flush=True)


bench(gen.config_c3(y_zero=False), "c3")
for proj in ("q", "gate", "down", "k"):
    bench(gen.config_c5(proj, y_zero=False, prefill=True), "c5_" + proj)
