"""Per-CTA timeline of cluster-span decode applies (csrc/span_kernel.cu) replayed from a CUDA
graph, as in bench.py: N pools (distinct adapter weights), one graph of N back-to-back applies.
Trace slots: 1 start, 7 ring issued, 2 griddepcontrol.wait passed, 3 x/y + first chunk ready,
6 first cluster barrier passed, 5 done, 4 rank, 0 SM.
usage: python scripts/trace_span.py [c2|c5q|c5down] [n_pools]"""
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
NP = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mk = {"c2": lambda tag: gen.config_c2(tag=tag), "c5q": lambda tag: gen.config_c5("q"),
      "c5down": lambda tag: gen.config_c5("down")}[which]


def tt(a, pin=False):
    t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a)
    return t.pin_memory() if pin else t


pools, batches = [], []
for i in range(NP):
    b = mk(i)
    pool = L.LoraPool(b.H_in, b.H_out, 64, b.dtype, max_total_rank=sum(a.rank for a in b.adapters))
    for a in b.adapters:
        pool.load_adapter(a.id, a.rank, tt(a.A, True), tt(a.B, True), a.scale)
    pool.set_option(L.binding.LORA_OPT_DECODE_PATH, 1)
    pools.append(pool)
    batches.append(b)
b = batches[0]
x = tt(b.x).cuda()
ys = [tt(bb.y_in).cuda() for bb in batches]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for p, y in zip(pools, ys):
        p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
torch.cuda.synchronize()
md = pools[0].metadata()
n = md["n_span_ctas"]
assert n > 0, "span path not taken"
bufs = [torch.zeros(16 * n + 64, dtype=torch.int64, device="cuda") for _ in pools]
for p, bf in zip(pools, bufs):
    p.set_trace(bf)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for p, y in zip(pools, ys):
        p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
flush = torch.empty(512 * 2 ** 20, dtype=torch.int8, device="cuda")
times = []
for rep in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) * 1e3)
print("graph of %d applies: %.2f us per replay (%.2f us / apply), CTAs/apply %d, cluster %d" %
      (NP, min(times), min(times) / NP, n, md["span_cluster"]))
Us = [bf.cpu().numpy()[:16 * n].reshape(n, 16) for bf in bufs]
t0 = min(U[:, 1].min() for U in Us)
act = lambda U: U[U[:, 4] > 0]  # noqa
for i, U in enumerate(Us):
    A = act(U)
    r = lambda col: (A[:, col] - t0) / 1e3  # noqa
    print("apply %d: start %6.2f..%6.2f issued ..%6.2f wait-ok %6.2f..%6.2f data %6.2f..%6.2f cl1 %6.2f..%6.2f done %6.2f..%6.2f"
          % (i, r(1).min(), r(1).max(), r(7).max(), r(2).min(), r(2).max(), r(3).min(), r(3).max(), r(6).min(),
             r(6).max(), r(5).min(), r(5).max()))
A = np.concatenate([act(U) for U in Us])
for lab, a_, b_ in (("start->rec", 1, 14), ("rec->meta", 14, 15), ("meta->issued", 15, 7), ("start->issued", 1, 7), ("issued->wait", 7, 2), ("wait->data", 2, 3), ("data->lastA", 3, 8),
                    ("lastA->vpart", 8, 9), ("vpart->cl1", 9, 6), ("cl1->vdone", 6, 13), ("vdone->B0", 13, 10),
                    ("B0->Blast", 10, 11), ("Blast->ystage", 11, 12), ("ystage->done", 12, 5),
                    ("start->done", 1, 5), ("start->B0", 1, 10), ("start->lastA", 1, 8)):
    d = (A[:, b_] - A[:, a_]) / 1e3
    print("   %-14s med %.2f p90 %.2f max %.2f" % (lab, np.median(d), np.percentile(d, 90), d.max()))
prev = None
for i, U in enumerate(Us):
    A = act(U)
    w, dn = A[:, 2].min(), A[:, 5].max()
    print("apply %d: prev.done->wait %6.2f  wait->done %5.2f" % (i, (w - prev) / 1e3 if prev is not None else float("nan"),
                                                            (dn - w) / 1e3))
    prev = dn
per_sm = defaultdict(list)
for i, U in enumerate(Us):
    for row in U:
        per_sm[int(row[0])].append((row[1], row[5], i))
hist = defaultdict(int)
for sm, L_ in per_sm.items():
    for e in L_:
        hist[sum(1 for f in L_ if f[0] <= e[0] < f[1])] += 1
print("   resident CTAs on the SM at CTA start:", dict(sorted(hist.items())), " SMs used:", len(per_sm))
