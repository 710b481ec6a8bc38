"""Per-CTA timeline of the bench's decode layer (one q/k/v lora_apply_multi + one o lora_apply,
c2 batch, 4096 -> 4096 bf16) replayed from a CUDA graph of NL layers (lora_debug_set_trace).
Prints per layer and kernel: first start, first/last wait-passed, last done; per-kernel phase
medians; and the per-SM residency.  usage: python scripts/trace_layer.py [NL] [warm]"""
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 6
WARM = len(sys.argv) > 2 and sys.argv[2] == "warm"
H = 4096
b = gen.config_c2()
ip, ids = b.seg_indptr, b.adapter_ids


def tt(a, pin=False):
    t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a)
    return t.pin_memory() if pin else t


pools = []
for l in range(NL):
    row = []
    for p in range(4):
        ads = [gen.make_adapter(gen.BASE_SEED + 1, 1 + l * 4 + p, a, gen.C2_RANKS[a % 4], H, H, "bf16") for a in range(32)]
        pool = L.LoraPool(H, H, 32, "bf16", max_total_rank=sum(a.rank for a in ads))
        for a in ads:
            pool.load_adapter(a.id, a.rank, tt(a.A, True), tt(a.B, True), a.scale)
        row.append(pool)
    pools.append(row)
torch.cuda.synchronize()
x = torch.randn(NL, 2, 64, H, device="cuda").to(torch.bfloat16)
ys = torch.zeros(NL, 4, 64, H, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.Stream()


def step():
    for l in range(NL):
        L.apply_multi(pools[l][:3], [x[l, 0]] * 3, [ys[l, 0], ys[l, 1], ys[l, 2]], ip, ids, stream=st)
        pools[l][3].apply(x[l, 1], ys[l, 3], ip, ids, stream=st)


with torch.cuda.stream(st):
    step()
torch.cuda.synchronize()
# unit counts per launch: the q/k/v pools' plans come from lora_apply_multi (its unit sizing), the o
# pool's from its single lora_apply
mq, mo = pools[0][0].metadata(), pools[0][3].metadata()
counts = {"qkv": (3 * mq["n_shrink_units"], 3 * mq["n_expand_units"]), "o": (mo["n_shrink_units"], mo["n_expand_units"])}
bufs = {}
for l in range(NL):
    for k, p in (("qkv", pools[l][0]), ("o", pools[l][3])):
        ns, ne = counts[k]
        bufs[(l, k)] = torch.zeros(8 * (ns + ne) + 4 * (ns + ne) + 64, dtype=torch.int64, device="cuda")
        p.set_trace(bufs[(l, k)])
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    step()
flush = torch.empty(512 * 2 ** 20, dtype=torch.int8, device="cuda")
for rep in range(3):
    if not WARM:
        flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    print("replay %d: %.2f us per layer" % (rep, e0.elapsed_time(e1) * 1e3 / NL))
U = {}
for key, bf in bufs.items():
    ns, ne = counts[key[1]]
    a = bf.cpu().numpy()[:8 * (ns + ne)].reshape(ns + ne, 8)
    U[key] = (a[:ns], a[ns:])
t0 = min(min(S[:, 1].min(), E[:, 1].min()) for S, E in U.values())
us = lambda v: (v - t0) / 1e3  # noqa
print("per layer (us from the first CTA start; S = shrink grid, E = expand grid)")
prev = None
for l in range(NL):
    for k in ("qkv", "o"):
        S, E = U[(l, k)]
        print("L%d %-3s S start %7.2f wait %7.2f..%7.2f done %7.2f | E start %7.2f wait %7.2f..%7.2f done %7.2f | "
              "S.done->E.wait %.2f" % (l, k, us(S[:, 1].min()), us(S[:, 2].min()), us(S[:, 2].max()), us(S[:, 5].max()),
                                     us(E[:, 1].min()), us(E[:, 2].min()), us(E[:, 2].max()), us(E[:, 5].max()),
                                     (E[:, 2].min() - S[:, 5].max()) / 1e3))
for k in ("qkv", "o"):
    S = np.concatenate([U[(l, k)][0] for l in range(1, NL)])
    E = np.concatenate([U[(l, k)][1] for l in range(1, NL)])
    for lab, A, c0, c1 in (("S start->wait", S, 1, 2), ("S wait->data", S, 2, 3), ("S data->done", S, 3, 5),
                           ("E start->wait", E, 1, 2), ("E wait->data", E, 2, 3), ("E data->mma", E, 3, 7),
                           ("E mma->y", E, 7, 6), ("E y->done", E, 6, 5), ("E wait->done", E, 2, 5)):
        d = (A[:, c1] - A[:, c0]) / 1e3
        print("  %-3s %-14s med %.2f p10 %.2f p90 %.2f max %.2f" % (k, lab, np.median(d), np.percentile(d, 10),
                                                                 np.percentile(d, 90), d.max()))
    # how many CTAs passed their wait late (second wave): wait-passed more than 1 us after the first
    for nm, A in (("S", S), ("E", E)):
        late = 0
        for l in range(1, NL):
            X = U[(l, k)][0 if nm == "S" else 1]
            late += int(np.sum(X[:, 2] - X[:, 2].min() > 1000))
        print("  %-3s %s CTAs passing their wait > 1 us after the first: %.1f per layer of %d" % (
            k, nm, late / (NL - 1), len(U[(1, k)][0 if nm == "S" else 1])))
