"""Per-CTA phase timeline of the tcgen05 prefill kernel (lora_debug_set_trace): config 3, or a c5
prefill shape (32 token tiles: split-K clusters).  usage: python scripts/trace_prefill.py [c3|c5q|c5down] [steady]
L2 is flushed by a READ pass (a writing flush leaves dirty lines whose write-backs the traced apply would
pay); `steady` instead traces an apply issued right behind an untraced one (its dirty y lines drain
during the traced apply, as in the back-to-back bench)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402


def tt(a, pin=False):
    t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a)
    return t.pin_memory() if pin else t


which = sys.argv[1] if len(sys.argv) > 1 else "c3"
b = {"c3": lambda: gen.config_c3(), "c5q": lambda: gen.config_c5("q", prefill=True),
     "c5down": lambda: gen.config_c5("down", prefill=True)}[which]()
pool = L.LoraPool(b.H_in, b.H_out, 64, b.dtype, max_total_rank=sum(a.rank for a in b.adapters))
for a in b.adapters:
    pool.load_adapter(a.id, a.rank, tt(a.A, True), tt(a.B, True), a.scale)
x = tt(b.x).cuda()
y = tt(b.y_in).cuda()
for _ in range(3):
    pool.apply(x, y, b.seg_indptr, b.adapter_ids)
torch.cuda.synchronize()
md = pool.metadata()
nt = md["n_prefill_ctas"]
buf = torch.zeros(4 * nt * 2 + 64, dtype=torch.int64, device="cuda")
pool.set_trace(buf)
steady = len(sys.argv) > 2 and sys.argv[2] == "steady"
flush = torch.zeros(512 * 2 ** 20 // 8, dtype=torch.int64, device="cuda")
flush.sum()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
if steady:
    pool.set_trace(None)
    pool.apply(x, y, b.seg_indptr, b.adapter_ids)
    pool.set_trace(buf)
e0.record()
pool.apply(x, y, b.seg_indptr, b.adapter_ids)
e1.record()
torch.cuda.synchronize()
pool.set_trace(None)
U = buf.cpu().numpy()[:4 * nt].reshape(nt, 4).astype(np.float64)
t0 = U[:, 0].min()
print("tiles %d, event %.1f us, first start -> last end %.1f us" % (nt, e0.elapsed_time(e1) * 1e3, (U[:, 1].max() - t0) / 1e3))
for lab, a_, b_ in (("start->shrink done", 0, 2), ("shrink done->V ready", 2, 3), ("V ready->end", 3, 1), ("total", 0, 1)):
    d = (U[:, b_] - U[:, a_]) / 1e3
    print("  %-22s med %.2f p10 %.2f p90 %.2f max %.2f us" % (lab, np.median(d), np.percentile(d, 10),
                                                              np.percentile(d, 90), d.max()))
print("  start spread %.2f us" % ((U[:, 0].max() - t0) / 1e3))
ranks = np.array([gen.C3_RANKS[(t // 4) % 5] for t in range(nt)]) if which == "c3" else np.zeros(nt, int)
for r in sorted(set(ranks.tolist())):
    m = ranks == r
    print("  rank %3d: shrink %.1f us, expand %.1f us, total %.1f us (%d tiles)" % (
        r, np.median((U[m, 2] - U[m, 0]) / 1e3), np.median((U[m, 1] - U[m, 3]) / 1e3),
        np.median((U[m, 1] - U[m, 0]) / 1e3), m.sum()))
