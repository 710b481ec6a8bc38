"""NEXT f2 measurement: y = x·W + s·(x·A)·B on c3 shapes (32 x 512 tokens, 4096 -> 4096, ranks 8..128).
  fused   : lora_apply_fused_base (one tcgen05 kernel)
  unfused : torch.matmul(x, W) (cuBLAS) into y, then lora_apply (the delta pass: y read + write)
  base    : torch.matmul(x, W) alone (the floor the fused kernel competes with)
CUDA graphs of NP back-to-back calls, L2 flushed before each replay; prints µs per call and
TFLOP/s (2·T·H_in·H_out + delta flops) against MEASURED_PEAKS.json's bf16 peak.
usage: python scripts/fused_base_bench.py [n_seg]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_11240_b200 as L  # noqa: E402
from workloads import gen  # noqa: E402

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
n_seg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
b = gen.config_c3(n_seg=n_seg)
pool = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
for a in b.adapters:
    pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                      torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
x = torch.from_numpy(b.x.view(np.int16)).cuda().view(torch.bfloat16)
W = (torch.randn(b.H_in, b.H_out, device="cuda") / b.H_in ** 0.5).to(torch.bfloat16)
WT = W.t().contiguous()   # nn.Linear layout [H_out][H_in]
W_fused = WT if "-DFG_B_KMAJOR=1" in os.environ.get("LORA_BUILD_DEFS", "") else W
y = torch.empty(b.T, b.H_out, dtype=torch.bfloat16, device="cuda")
st = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
NP = 4


def fused():
    pool.apply_fused_base(x, W_fused, y, b.seg_indptr, b.adapter_ids, stream=st)


def unfused():
    torch.matmul(x, W, out=y)
    pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)


def base():
    torch.matmul(x, W, out=y)


no_ids = np.full_like(b.adapter_ids, -1)


def fused_gemm_only():   # every segment id < 0: no shrink pass, the GEMM without K extension
    pool.apply_fused_base(x, W_fused, y, b.seg_indptr, no_ids, stream=st)


def shrink_pass_only():   # the prefill kernel alone (expand included): an upper bound for the V pass
    pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)


def timed(fn):
    with torch.cuda.stream(st):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(NP):
            fn()
    ts = []
    for _ in range(7):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / NP)
    return float(np.median(ts))


sum_tr = sum(int(b.seg_indptr[i + 1] - b.seg_indptr[i]) * b.adapters[[a.id for a in b.adapters].index(int(b.adapter_ids[i]))].rank
             for i in range(len(b.adapter_ids)))
flops = 2.0 * b.T * b.H_in * b.H_out + 2.0 * sum_tr * (b.H_in + b.H_out)
out = {"T": b.T, "H": b.H_in, "tflop": round(flops / 1e12, 4)}
for name, fn in (("fused", fused), ("unfused", unfused), ("base", base), ("fused_gemm_only", fused_gemm_only),
                 ("prefill_delta", shrink_pass_only)):
    us = timed(fn)
    out[name] = {"us": round(us, 1), "tflops": round(flops / (us * 1e-6) / 1e12, 1),
                 "frac_bf16_peak": round(flops / (us * 1e-6) / 1e12 / peaks["bf16_tflops"], 3)}
print(json.dumps(out))
