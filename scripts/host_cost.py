"""Host-side cost per API call on the decode path (c2 batch, 4096 -> 4096 bf16): lora_plan alone,
lora_apply and lora_apply_multi (q/k/v) issue time without synchronisation, and the pure kernel
time per call for comparison.  usage: python scripts/host_cost.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

H = 4096
b = gen.config_c2()
pools = []
for p in range(4):
    pool = L.LoraPool(H, H, 32, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
    for a in b.adapters:
        pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                          torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
    pools.append(pool)
torch.cuda.synchronize()
x = torch.randn(64, H, device="cuda").to(torch.bfloat16)
ys = [torch.zeros(64, H, device="cuda", dtype=torch.bfloat16) for _ in range(4)]
st = torch.cuda.Stream()
ip, ids = np.ascontiguousarray(b.seg_indptr, np.int32), np.ascontiguousarray(b.adapter_ids, np.int32)


def timed(fn, n=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) / n * 1e6, (t2 - t0) / n * 1e6


with torch.cuda.stream(st):
    h, w = timed(lambda: pools[3].apply(x, ys[3], ip, ids, stream=st))
    print("lora_apply        host %.1f us/call  (host+drain %.1f)" % (h, w))
    h, w = timed(lambda: L.apply_multi(pools[:3], [x] * 3, ys[:3], ip, ids, stream=st))
    print("lora_apply_multi  host %.1f us/call  (host+drain %.1f)" % (h, w))
    h, w = timed(lambda: (L.apply_multi(pools[:3], [x] * 3, ys[:3], ip, ids, stream=st),
                          pools[3].apply(x, ys[3], ip, ids, stream=st)))
    print("one layer (multi + apply) host %.1f us  (host+drain %.1f)" % (h, w))
