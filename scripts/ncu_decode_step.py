"""One decode layer step exactly as bench.py issues it (c2: q/k/v as one lora_apply_multi + o as one
lora_apply, 4096->4096 bf16, 64 tokens over 32 adapters), for ncu: the LAST 4 decode kernels of the
run are one step (multi pair, o pair).  usage (under ncu): python scripts/ncu_decode_step.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

H, T = 4096, 64
b = gen.config_c2(tag=0)
pools = []
for proj in range(4):
    pool = L.LoraPool(H, H, 32, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
    for a in range(32):
        ad = gen.make_adapter(gen.BASE_SEED + 1, 1 + proj, a, gen.C2_RANKS[a % 4], H, H, "bf16")
        pool.load_adapter(a, ad.rank, torch.from_numpy(ad.A.view(np.int16)).pin_memory(),
                          torch.from_numpy(ad.B.view(np.int16)).pin_memory(), ad.scale)
    pools.append(pool)
torch.cuda.synchronize()
xs = [torch.randn(T, H).to(torch.bfloat16).cuda() for _ in range(2)]
ys = [torch.zeros(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
for _ in range(3):
    L.apply_multi(pools[:3], [xs[0]] * 3, ys[:3], b.seg_indptr, b.adapter_ids)
    pools[3].apply(xs[1], ys[3], b.seg_indptr, b.adapter_ids)
torch.cuda.synchronize()
print("done: 3 steps x (multi pair + o pair)")
