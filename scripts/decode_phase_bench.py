"""Steady-state cost of each decode kernel in isolation: CUDA graphs of N back-to-back
full applies, shrink-only applies (lora_apply_shrink) and expand-only applies
(lora_apply_expand), c2 workload, distinct adapter weights per pool (inputs > L2).
usage: python scripts/decode_phase_bench.py [n_pools]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

NP = int(sys.argv[1]) if len(sys.argv) > 1 else 64


def tt(a, pin=False):
    t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a)
    return t.pin_memory() if pin else t


pools = []
b = gen.config_c2(tag=0)
for i in range(NP):
    bb = gen.config_c2(tag=i) if i < 4 else b
    pool = L.LoraPool(b.H_in, b.H_out, 64, b.dtype, max_total_rank=sum(a.rank for a in b.adapters))
    for a in bb.adapters:
        pool.load_adapter(a.id, a.rank, tt(a.A, True), tt(a.B, True), a.scale)
    pools.append(pool)
x = tt(b.x).cuda()
ys = [tt(b.y_in).cuda() for _ in pools]
vs = [torch.zeros(1 << 20, dtype=torch.float32, device="cuda") for _ in pools]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for p, y, v in zip(pools, ys, vs):
        p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
        p.apply_shrink(x, b.seg_indptr, b.adapter_ids, v, stream=st)
        p.apply_expand(y, v, stream=st)
torch.cuda.synchronize()
flush = torch.empty(512 * 2 ** 20, dtype=torch.int8, device="cuda")


def run(body, reps=5):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        body()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / NP)
    return float(np.median(ts))


full = run(lambda: [p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st) for p, y in zip(pools, ys)])
shr = run(lambda: [p.apply_shrink(x, b.seg_indptr, b.adapter_ids, v, stream=st) for p, v in zip(pools, vs)])
exp = run(lambda: [p.apply_expand(y, v, stream=st) for p, y, v in zip(pools, ys, vs)])
split = run(lambda: [(p.apply_shrink(x, b.seg_indptr, b.adapter_ids, v, stream=st), p.apply_expand(y, v, stream=st))
                     for p, y, v in zip(pools, ys, vs)])
md = pools[0].metadata()
print("c2 x %d pools: us/apply  full %.2f | shrink-only %.2f | expand-only %.2f | split pair %.2f  (units S %d E %d)"
      % (NP, full, shr, exp, split, md["n_shrink_units"], md["n_decode_units"] - md["n_shrink_units"]))

# the shrink/expand kernel pair, and its one-grid variant (per-gc counters)
for p in pools:
    p.set_option(L.binding.LORA_OPT_DECODE_PATH, 1)
span = run(lambda: [p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st) for p, y in zip(pools, ys)])
for p in pools:
    p.set_option(L.binding.LORA_OPT_DECODE_PATH, 0)
print("c2 x %d pools: us/apply  kernel pair (default) %.2f | cluster span %.2f" % (NP, full, span))
for p in pools:
    p.set_option(L.binding.LORA_OPT_DECODE_FUSED, 1)
with torch.cuda.stream(st):
    for p, y in zip(pools, ys):
        p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
torch.cuda.synchronize()
fused = run(lambda: [p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st) for p, y in zip(pools, ys)])
for p in pools:
    p.set_option(L.binding.LORA_OPT_DECODE_FUSED, 2)
with torch.cuda.stream(st):
    for p, y in zip(pools, ys):
        p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
torch.cuda.synchronize()
flagc = run(lambda: [p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st) for p, y in zip(pools, ys)])
print("c2 x %d pools: us/apply  flag-chained pair %.2f" % (NP, flagc))
for p in pools:
    p.set_option(L.binding.LORA_OPT_DECODE_FUSED, 0)
# q/k/v style: 3 pools per lora_apply_multi launch pair
trip = [(pools[i:i + 3], ys[i:i + 3]) for i in range(0, NP - 2, 3)]
with torch.cuda.stream(st):
    for ps, yy in trip:
        L.apply_multi(ps, [x] * 3, yy, b.seg_indptr, b.adapter_ids, stream=st)
torch.cuda.synchronize()
multi = run(lambda: [L.apply_multi(ps, [x] * 3, yy, b.seg_indptr, b.adapter_ids, stream=st) for ps, yy in trip]) \
    * NP / (3 * len(trip))
print("c2 x %d pools: us/apply  fused-grid %.2f | multi(3) %.2f" % (NP, fused, multi))
