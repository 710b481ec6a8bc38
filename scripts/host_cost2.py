"""Host cost breakdown of one cached lora_apply (c2 batch): raw ctypes call vs the Python wrapper,
a trivial library call (ctypes floor), and a torch kernel launch for scale.  usage: python scripts/host_cost2.py"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from paper_2401_11240_b200 import binding as B  # noqa: E402
from workloads import gen  # noqa: E402

H = 4096
b = gen.config_c2()
pool = L.LoraPool(H, H, 32, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
for a in b.adapters:
    pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                      torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
torch.cuda.synchronize()
x = torch.randn(64, H, device="cuda").to(torch.bfloat16)
y = torch.zeros(64, H, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.Stream()
ip, ids = np.ascontiguousarray(b.seg_indptr, np.int32), np.ascontiguousarray(b.adapter_ids, np.int32)
h, xp, yp, pip, pid, n, sp = pool.handle, x.data_ptr(), y.data_ptr(), ip.ctypes.data, ids.ctypes.data, len(ids), st.cuda_stream
f = B.LIB.lora_apply
rdy = ctypes.c_int()


def t(fn, n=300):
    for _ in range(30):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return dt


print("ctypes trivial call (lora_adapter_ready) %.2f us" % t(lambda: B.LIB.lora_adapter_ready(h, 0, ctypes.byref(rdy))))
print("raw lora_apply (cached plan)           %.2f us" % t(lambda: f(h, xp, yp, pip, pid, n, sp)))
print("wrapper pool.apply                      %.2f us" % t(lambda: pool.apply(x, y, ip, ids, stream=st)))
z = torch.zeros(16, device="cuda")
with torch.cuda.stream(st):
    print("torch z.add_(1) launch                  %.2f us" % t(lambda: z.add_(1)))
md = pool.metadata()
print("blob words: shrink units %d expand units %d" % (md["n_shrink_units"], md["n_expand_units"]))
