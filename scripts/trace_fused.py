"""Per-item timeline of the fused base GEMM (lora_apply_fused_base) on c3 shapes: for each CTA pair
(leader) and item: MMA start, mainloop end, epilogue start (tfull), epilogue end (lora_debug_set_trace).
usage: python scripts/trace_fused.py [no_adapters]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

b = gen.config_c3()
pool = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
for a in b.adapters:
    pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                      torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
x = torch.from_numpy(b.x.view(np.int16)).cuda().view(torch.bfloat16)
W = (torch.randn(b.H_in, b.H_out, device="cuda") / b.H_in ** 0.5).to(torch.bfloat16)
y = torch.empty(b.T, b.H_out, dtype=torch.bfloat16, device="cuda")
ids = b.adapter_ids if len(sys.argv) < 2 else np.full_like(b.adapter_ids, -1)
for _ in range(3):
    pool.apply_fused_base(x, W, y, b.seg_indptr, ids)
torch.cuda.synchronize()
tr = torch.zeros(74 * 64 * 4, dtype=torch.int64, device="cuda")
pool.set_trace(tr)
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
flush.zero_()
torch.cuda.synchronize()
pool.apply_fused_base(x, W, y, b.seg_indptr, ids)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(74, 64, 4).astype(np.uint64)
vit = (t[:, :, 2] >> np.uint64(63)).astype(bool)
t = (t & np.uint64((1 << 63) - 1)).astype(np.float64)
t0 = t[:, 0, 0][t[:, 0, 0] > 0].min()
rel = (t - t0) / 1e3
rel[t == 0] = np.nan
n_it = np.sum(t[:, :, 0] > 0, axis=1)
print("items per cluster: min %d max %d" % (n_it.min(), n_it.max()))
print("kernel span (first MMA start -> last epilogue end): %.1f us" % np.nanmax(rel[:, :, 3]))
for c in (0, 10, 40, 63, 64, 73):
    n = n_it[c]
    row = " ".join("%s%.1f/%.1f" % ("V" if vit[c, i] else "", rel[c, i, 0], rel[c, i, 1] - rel[c, i, 0]) for i in range(n))
    print("cluster %2d (%d items) start/mainloop: %s | end %.1f" % (c, n, row, np.nanmax(rel[c, :, 3])))
ml = rel[:, :, 1] - rel[:, :, 0]
live = t[:, :, 0] > 0
if vit.any():
    print("mainloop us: V items med %.2f max %.2f" % (np.nanmedian(ml[vit]), np.nanmax(ml[vit])))
print("mainloop us: other items med %.2f p90 %.2f" % (np.nanmedian(ml[~vit & live]), np.nanpercentile(ml[~vit & live], 90)))
ep = rel[:, :, 3] - rel[:, :, 2]
print("epilogue us (tfull -> drained) med %.2f p90 %.2f max %.2f" % (np.nanmedian(ep), np.nanpercentile(ep[~np.isnan(ep)], 90), np.nanmax(ep)))
lag = rel[:, :, 2] - rel[:, :, 1]
print("mainloop end -> epilogue start (rank chunks + commit) med %.2f p90 %.2f" % (np.nanmedian(lag), np.nanpercentile(lag[~np.isnan(lag)], 90)))
gap = rel[:, 1:, 0] - rel[:, :-1, 1]
print("item gap (prev mainloop end -> next MMA start) med %.2f p90 %.2f max %.2f" % (
    np.nanmedian(gap), np.nanpercentile(gap[~np.isnan(gap)], 90), np.nanmax(gap)))
