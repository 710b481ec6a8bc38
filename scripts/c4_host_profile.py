"""Where config 4's step time goes: host time in AdapterCache.ensure (per lora_load_adapter call),
host time of lora_apply, and device time, over 40 Zipf steps (5120, 1000 adapters, 20% pool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from paper_2401_11240_b200.serving import AdapterCache, HostRepository  # noqa: E402
from workloads import gen  # noqa: E402

H, n_ad = 5120, 1000
repo = HostRepository()
for a in range(n_ad):
    ad = gen.c4_adapter(a, H)
    repo.add(a, ad.rank, ad.scale, torch.from_numpy(ad.A.view(np.int16)).pin_memory(),
             torch.from_numpy(ad.B.view(np.int16)).pin_memory())
budget = sum(gen.c4_rank(a) for a in range(n_ad)) // 5
pool = L.LoraPool(H, H, n_ad, "bf16", max_total_rank=budget)
if os.environ.get("LORA_LOAD_KERNEL"):
    pool.set_option(L.binding.LORA_OPT_LOAD_KERNEL, 1)
cache = AdapterCache(pool, repo, budget, n_ad)
st = torch.cuda.Stream()
x = torch.randn(576, H).to(torch.bfloat16).cuda()
y = torch.zeros(576, H, dtype=torch.bfloat16, device="cuda")
ip = gen.segments_to_indptr([1] * 64 + [512])
draws = []
for s in range(45):
    d = gen.config_c4_draw(s)
    draws.append(np.array([int(a) for a in d["decode_ids"]] + [int(d["prefill_id"][0])], np.int32))
for ids in draws[:5]:
    cache.ensure(ids.tolist())
    pool.apply(x, y, ip, ids, stream=st)
torch.cuda.synchronize()
t_ens = t_app = 0.0
n_load = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter()
e0.record(st)
for ids in draws[5:]:
    t = time.perf_counter()
    n_load += len(cache.ensure(ids.tolist()))
    t_ens += time.perf_counter() - t
    t = time.perf_counter()
    pool.apply(x, y, ip, ids, stream=st)
    t_app += time.perf_counter() - t
e1.record(st)
torch.cuda.synchronize()
wall = time.perf_counter() - w0
n = len(draws) - 5
print("per step: wall %.3f ms, device %.3f ms, ensure %.3f ms (%.1f loads, %.1f us/load), apply host %.3f ms"
      % (wall / n * 1e3, e0.elapsed_time(e1) / n, t_ens / n * 1e3, n_load / n, t_ens / max(1, n_load) * 1e6,
         t_app / n * 1e3))
