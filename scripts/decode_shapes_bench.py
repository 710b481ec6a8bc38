"""Per-apply time of the default decode pair over several decode batch shapes (4096 -> 4096 bf16,
CUDA graph of N pools' applies, L2 flushed before each replay).  Used for A/B comparisons of a
decode-kernel change: run once per build, compare the lines.
  uniform : c2 (64 tokens over 32 adapters, ~2 tokens per adapter)
  zipf    : c2 with Zipf(1.0) adapter draws (a few adapters own full 8-token chunks)
  one64   : 64 tokens of one rank-64 adapter (8 full chunks)
  t256    : 256 tokens over 32 adapters (8 tokens per adapter)
usage: python scripts/decode_shapes_bench.py [n_pools]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

NP = int(sys.argv[1]) if len(sys.argv) > 1 else 48


def tt(a, pin=False):
    t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a)
    return t.pin_memory() if pin else t


def shapes():
    yield "uniform", gen.config_c2()
    yield "zipf", gen.config_c2(zipf=True)
    yield "one64", gen.build_batch("one64", gen.BASE_SEED + 1, "bf16", 4096, 4096, [1] * 64, [0] * 64,
                                   {0: 64}, y_zero=True)
    yield "t256", gen.config_c2(T=256)


st = torch.cuda.Stream()
flush = torch.empty(512 * 2 ** 20, dtype=torch.int8, device="cuda")
out = {}
for name, b in shapes():
    pools = []
    for i in range(NP):
        pool = L.LoraPool(b.H_in, b.H_out, 64, b.dtype, max_total_rank=sum(a.rank for a in b.adapters))
        for a in b.adapters:
            pool.load_adapter(a.id, a.rank, tt(a.A, True), tt(a.B, True), a.scale)
        pools.append(pool)
    x = tt(b.x).cuda()
    ys = [tt(b.y_in).cuda() for _ in pools]
    with torch.cuda.stream(st):
        for p, y in zip(pools, ys):
            p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
    torch.cuda.synchronize()
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
    out[name] = float(np.median(ts))
    del g
    for p in pools:
        p.close()
print("decode us/apply: " + "  ".join("%s %.2f" % kv for kv in out.items()))
