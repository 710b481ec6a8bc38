"""Is the c3 prefill bound per SM or chip-wide?  c3-shaped batches (512-token segments, ranks
[8,16,32,64,128][i mod 5], 4096 -> 4096) with 16..37 segments = 64..148 token tiles, one CTA per
tile: per-SM bound -> time flat in the tile count up to 148; chip-bound -> time grows with bytes.
usage: python scripts/prefill_tiles_scaling.py"""
import json
import os
import sys

import numpy as np
import torch

os.environ.setdefault("LORA_EXP_PF_SPLIT", "1")   # one CTA per tile at every tile count
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
st = torch.cuda.Stream()
for n_seg in (16, 24, 32, 37):
    b = gen.config_c3(n_seg=n_seg)
    NP = 3
    pools = []
    for _ in range(NP):
        pool = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
        for a in b.adapters:
            pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                              torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
        pools.append(pool)
    x = torch.from_numpy(b.x.view(np.int16)).cuda()
    ys = [torch.zeros(b.T, b.H_out, dtype=torch.int16, device="cuda") for _ in pools]
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
    for _ in range(7):
        flush.zero_()
        torch.cuda.synchronize()
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
    print("c3-shaped n_seg=%d tiles=%d ctas=%d: %.1f us/apply, %.0f GB/s = %.1f%%"
          % (n_seg, md["n_prefill_tiles"], md["n_prefill_ctas"], us, byts / (us * 1e-6) / 1e9,
             100 * byts / (us * 1e-6) / 1e9 / peak), flush=True)
    del g
    for p in pools:
        p.close()
