"""c5 prefill: Llama-2-70B shapes, 8 segments x 512 tokens over 8 adapters (ranks
16..128), one apply per pool on the tcgen05 kernel; device time per apply and HBM roofline fraction.
usage: python scripts/c5_prefill.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for proj in ("q", "gate", "down"):
    b = gen.config_c5(proj, prefill=True)
    NP = 3
    pools = []
    for _ in range(NP):
        pool = L.LoraPool(b.H_in, b.H_out, 16, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
        for a in b.adapters:
            pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                              torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
        pools.append(pool)
    torch.cuda.synchronize()
    x = torch.from_numpy(b.x.view(np.int16)).cuda()
    ys = [torch.zeros(b.T, b.H_out, dtype=torch.int16, device="cuda") for _ in pools]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for p, y in zip(pools, ys):
            p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
    torch.cuda.synchronize()
    md = pools[0].metadata()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for p, y in zip(pools, ys):
            p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / NP)
    us = float(np.median(ts))
    sum_r = sum(a.rank for a in b.adapters)
    byts = 2 * (sum_r * (b.H_in + b.H_out) + b.T * b.H_in + 2 * b.T * b.H_out)
    print("c5 prefill %-5s %5d->%5d T=%d tiles=%d: %.1f us/apply, %.0f GB/s = %.1f%% of HBM roofline"
          % (proj, b.H_in, b.H_out, b.T, md["n_prefill_tiles"], us, byts / (us * 1e-6) / 1e9,
             100 * byts / (us * 1e-6) / 1e9 / peak))
    for p in pools:
        p.close()
