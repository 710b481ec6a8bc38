"""Per-unit timeline of the persistent streaming decode kernel (N1s) on the bench's decode layer
(q/k/v lora_apply_multi + o lora_apply, c2 batch) replayed from a CUDA graph of NL layers.
Trace words per unit (16 per unit): 0 smid, 2 operands in the stage (consumer), 3 expand: v ready,
5 consumers done, 6 expand: gc acquired by the v loader, 7 producer issued the weights, 10 shrink:
publisher picked the partials, 11 shrink: published.  usage: python scripts/trace_stream.py [NL] [stages]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 4
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 2
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
        pool.set_option(L.binding.LORA_OPT_DECODE_STAGES, NS)
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
md = pools[0][3].metadata()
ns1, ne1 = md["n_shrink_units"], md["n_expand_units"]
print("o: %d shrink + %d expand units, grid %d, stages %d" % (ns1, ne1, md["decode_ctas"], md["decode_stages"]))
counts = {"qkv": (3 * ns1, 3 * ne1), "o": (ns1, ne1)}
bufs = {}
for l in range(NL):
    for k, p in (("qkv", pools[l][0]), ("o", pools[l][3])):
        n = sum(counts[k])
        bufs[(l, k)] = torch.zeros(16 * n + 64, dtype=torch.int64, device="cuda")
        p.set_trace(bufs[(l, k)])
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    step()
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    print("replay %d: %.2f us per layer (traced)" % (rep, e0.elapsed_time(e1) * 1e3 / NL))
U = {}
for key, bf in bufs.items():
    ns, ne = counts[key[1]]
    a = bf.cpu().numpy()[:16 * (ns + ne)].reshape(ns + ne, 16).astype(np.int64)
    U[key] = (a[:ns], a[ns:])
t0 = min(min(S[:, 7].min(), E[:, 7].min()) for S, E in U.values())
us = lambda v: (v - t0) / 1e3  # noqa
for l in range(NL):
    for k in ("qkv", "o"):
        S, E = U[(l, k)]
        print("L%d %-3s S issue %7.2f..%7.2f data %7.2f..%7.2f pub %7.2f..%7.2f | E issue %7.2f..%7.2f acq %7.2f..%7.2f "
              "data %7.2f..%7.2f done %7.2f..%7.2f" % (
                  l, k, us(S[:, 7].min()), us(S[:, 7].max()), us(S[:, 2].min()), us(S[:, 2].max()), us(S[:, 11].min()),
                  us(S[:, 11].max()), us(E[:, 7].min()), us(E[:, 7].max()), us(E[:, 6].min()), us(E[:, 6].max()),
                  us(E[:, 2].min()), us(E[:, 2].max()), us(E[:, 5].min()), us(E[:, 5].max())))
for k in ("qkv", "o"):
    S = np.concatenate([U[(l, k)][0] for l in range(1, NL)])
    E = np.concatenate([U[(l, k)][1] for l in range(1, NL)])
    for lab, A, c0, c1 in (("S issue->data", S, 7, 2), ("S data->done", S, 2, 5), ("S done->picked", S, 5, 10),
                           ("S picked->pub", S, 10, 11), ("E issue->data", E, 7, 2), ("E acq->v", E, 6, 3),
                           ("E v->data", E, 3, 2), ("E data->done", E, 2, 5)):
        d = (A[:, c1] - A[:, c0]) / 1e3
        print("  %-3s %-16s med %6.2f p10 %6.2f p90 %6.2f max %6.2f" % (k, lab, np.median(d), np.percentile(d, 10),
                                                                      np.percentile(d, 90), d.max()))
S, E = U[(1, "qkv")]
P = md["decode_ctas"]
for cta in (0, 77):
    print("CTA %d of L1 qkv:" % cta)
    for i in range(cta, len(S), P):
        r = S[i]
        print("  S u%-4d issue %7.2f data %7.2f done %7.2f picked %7.2f pub %7.2f" % (i, us(r[7]), us(r[2]), us(r[5]), us(r[10]), us(r[11])))
    for i in range(cta, len(E), P):
        r = E[i]
        print("  E u%-4d issue %7.2f acq %7.2f v %7.2f data %7.2f done %7.2f" % (i, us(r[7]), us(r[6]), us(r[3]), us(r[2]), us(r[5])))
