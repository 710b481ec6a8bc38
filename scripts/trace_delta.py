"""Two-phase prefill on c3: per-item timeline of the delta GEMM (lora_debug_set_trace: [cluster][item]
{MMA start, mainloop end, epilogue tfull, epilogue done}) and the V pass's span (prefill kernel's
per-tile stamps share the buffer's first words).  usage: python scripts/trace_delta.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from paper_2401_11240_b200 import binding as B  # noqa: E402
from workloads import gen  # noqa: E402

b = gen.config_c3(y_zero=False)
pool = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
for a in b.adapters:
    pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                      torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
pool.set_option(B.LORA_OPT_PREFILL_TWO_PHASE, 1)
x = torch.from_numpy(b.x.view(np.int16)).cuda()
y = torch.zeros(b.T, b.H_out, dtype=torch.int16, device="cuda")
for _ in range(3):
    pool.apply(x, y, b.seg_indptr, b.adapter_ids)
torch.cuda.synchronize()
tr = torch.zeros(74 * 64 * 4 + 4096, dtype=torch.int64, device="cuda")
pool.set_trace(tr)
pool.apply(x, y, b.seg_indptr, b.adapter_ids)
torch.cuda.synchronize()
t = tr.cpu().numpy()[:74 * 64 * 4].reshape(74, 64, 4).astype(np.float64)
live = t[:, :, 0] > 0
t0 = t[:, 0, 0][t[:, 0, 0] > 0].min()
rel = (t - t0) / 1e3
rel[t == 0] = np.nan
print("delta GEMM span: first MMA start -> last epilogue done %.1f us" % np.nanmax(rel[:, :, 3]))
for c in (0, 37, 73):
    n = int(live[c].sum())
    print("cluster %d: " % c + " ".join("[%.1f m%.1f e%.1f-%.1f]" % (rel[c, i, 0], rel[c, i, 1], rel[c, i, 2], rel[c, i, 3])
                                       for i in range(n)))
ep = rel[:, :, 3] - rel[:, :, 2]
print("epilogue per item med %.2f p90 %.2f us; MMA start->epi start med %.2f" % (
    np.nanmedian(ep), np.nanpercentile(ep[~np.isnan(ep)], 90), np.nanmedian(rel[:, :, 2] - rel[:, :, 0])))
