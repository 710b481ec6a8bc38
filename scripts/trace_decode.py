"""Per-CTA timeline of decode applies replayed from a CUDA graph (lora_debug_set_trace).
Builds N pools of one config (distinct adapter weights), captures a graph of N back-to-back
applies (as in bench.py), replays it after an L2 flush and prints, per apply and kernel,
when CTAs started, passed griddepcontrol.wait, had their data, and finished.
usage: python scripts/trace_decode.py [c2|c5q|c5down] [n_pools]"""
import os
import sys

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
    if os.environ.get("LORA_TRACE_FUSED"):   # hand-off variant (LORA_OPT_DECODE_FUSED 1 or 2)
        pool.set_option(L.binding.LORA_OPT_DECODE_FUSED, int(os.environ["LORA_TRACE_FUSED"]))
    for a in b.adapters:
        pool.load_adapter(a.id, a.rank, tt(a.A, True), tt(a.B, True), a.scale)
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
n_units = md["n_decode_units"]
n_shrink = md["n_shrink_units"]
bufs = [torch.zeros(8 * n_units + 64, dtype=torch.int64, device="cuda") for _ in pools]
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
print("graph of %d applies: %.2f us per replay (%.2f us / apply), units/apply %d (shrink %d)" %
      (NP, min(times), min(times) / NP, n_units, n_shrink))
Us = [bf.cpu().numpy()[:8 * n_units].reshape(n_units, 8) for bf in bufs]
t0 = min(U[:, 1].min() for U in Us)
for i, U in enumerate(Us):
    for name, S in (("S", U[:n_shrink]), ("E", U[n_shrink:])):
        r = lambda col: (S[:, col] - t0) / 1e3  # noqa
        print("apply %d %s: start %6.2f..%6.2f  wait-ok %6.2f..%6.2f  data %6.2f..%6.2f  done %6.2f..%6.2f"
              % (i, name, r(1).min(), r(1).max(), r(2).min(), r(2).max(), r(3).min(), r(3).max(), r(5).min(),
                 r(5).max()))
U = np.concatenate([U[:n_shrink] for U in Us])
for lab, a_, b_ in (("S start->wait", 1, 2), ("S wait->data", 2, 3), ("S data->done", 3, 5)):
    d = (U[:, b_] - U[:, a_]) / 1e3
    print("   %-14s med %.2f p90 %.2f max %.2f" % (lab, np.median(d), np.percentile(d, 90), d.max()))
U = np.concatenate([U[n_shrink:] for U in Us])
for lab, a_, b_ in (("E start->wait", 1, 2), ("E wait->data", 2, 3), ("E data->done", 3, 5)):
    d = (U[:, b_] - U[:, a_]) / 1e3
    print("   %-14s med %.2f p90 %.2f max %.2f" % (lab, np.median(d), np.percentile(d, 90), d.max()))
# per-rank breakdown (slot 4 = unit rank) and per-apply critical path
for name, sl in (("S", slice(0, n_shrink)), ("E", slice(n_shrink, n_units))):
    U = np.concatenate([u[sl] for u in Us])
    for r in sorted(set(U[:, 4].tolist())):
        V = U[U[:, 4] == r]
        print("   %s r=%3d n=%4d  start->wait %.2f  wait->data %.2f  data->done %.2f  start->done %.2f (med us)" % (
            name, r, len(V), np.median((V[:, 2] - V[:, 1]) / 1e3), np.median((V[:, 3] - V[:, 2]) / 1e3),
            np.median((V[:, 5] - V[:, 3]) / 1e3), np.median((V[:, 5] - V[:, 1]) / 1e3)))
prev_done = None
for i, U in enumerate(Us):
    S, E = U[:n_shrink], U[n_shrink:]
    s_wait, s_done = S[:, 2].min(), S[:, 5].max()
    e_wait, e_done = E[:, 2].min(), E[:, 5].max()
    print("apply %d: prevE.done->S.wait %6.2f  S wait->done %5.2f  S.done->E.wait %5.2f  E wait->done %5.2f" % (
        i, (s_wait - prev_done) / 1e3 if prev_done is not None else float("nan"), (s_done - s_wait) / 1e3,
        (e_wait - s_done) / 1e3, (e_done - e_wait) / 1e3))
    prev_done = e_done
# finer phases (slots 6/7): S 6 = loads issued; E 7 = MMAs done, E 6 = y tile arrived
U = np.concatenate([u[:n_shrink] for u in Us])
print("   S start->issued med %.2f p90 %.2f" % (np.median((U[:, 6] - U[:, 1]) / 1e3), np.percentile((U[:, 6] - U[:, 1]) / 1e3, 90)))
U = np.concatenate([u[n_shrink:] for u in Us])
for lab, a_, b_ in (("E data->mma", 3, 7), ("E mma->y", 7, 6), ("E y->done", 6, 5), ("E wait->y", 2, 6)):
    d = (U[:, b_] - U[:, a_]) / 1e3
    print("   %-14s med %.2f p90 %.2f max %.2f" % (lab, np.median(d), np.percentile(d, 90), d.max()))
# co-residency: per SM, max number of simultaneously resident CTAs of each kind
ev = []
for i, u in enumerate(Us):
    for k, sl in (("S", slice(0, n_shrink)), ("E", slice(n_shrink, n_units))):
        for row in u[sl]:
            ev.append((int(row[0]), row[1], row[5], k, i))
from collections import defaultdict
per_sm = defaultdict(list)
for e in ev:
    per_sm[e[0]].append(e)
mx = defaultdict(int)
hist = defaultdict(int)
for sm, L_ in per_sm.items():
    for e in L_:
        t = e[1]
        live = [f for f in L_ if f[1] <= t < f[2]]
        key = "S%dE%d" % (sum(f[3] == "S" for f in live), sum(f[3] == "E" for f in live))
        hist[key] += 1
print("   residency at CTA start (S count, E count incl. itself):", dict(sorted(hist.items())))
print("   SMs used:", len(per_sm))
U = np.concatenate([u[:n_shrink] for u in Us])
print("   S start->meta-decoded med %.2f p90 %.2f; meta->issued med %.2f" % (
    np.median((U[:, 7] - U[:, 1]) / 1e3), np.percentile((U[:, 7] - U[:, 1]) / 1e3, 90), np.median((U[:, 6] - U[:, 7]) / 1e3)))
