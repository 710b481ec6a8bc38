"""scripts/trace_layer.py with every pool loaded by the zero-copy gather kernel (LORA_OPT_LOAD_KERNEL=LK,
env, default 1): for the bimodal steady-state investigation (DESIGN.md §6 cold start).
LK=dummy loads every pool by cudaMemcpyAsync after one throwaway pool loaded by the kernel;
LK=big loads by the kernel from ONE large pinned host buffer (every adapter's rows copied into it);
LK=alt loads the pools of even layers by cudaMemcpyAsync and of odd layers by the kernel (4 pools per
layer, in creation order).  usage: LK=1 python scripts/trace_layer_lk.py [NL]"""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_11240_b200 import binding as B  # noqa: E402

orig = B.LoraPool.__init__
count = [0]


def init(self, *a, **k):
    orig(self, *a, **k)
    lk = os.environ.get("LK", "1")
    self.set_option(B.LORA_OPT_LOAD_KERNEL, (count[0] // 4) % 2 if lk == "alt" else int(lk))
    count[0] += 1


B.LoraPool.__init__ = init
if os.environ.get("LK") == "big":
    import torch
    os.environ["LK"] = "1"
    BIG = torch.empty(2300 * 2 ** 20 // 2, dtype=torch.int16).pin_memory()
    off = [0]
    orig_load = B.LoraPool.load_adapter

    def load(self, aid, rank, A, Bm, scale):
        views = []
        for t in (A, Bm):
            n = t.numel()
            v = BIG[off[0]:off[0] + n].view(t.shape)
            v.copy_(t.view(torch.int16))
            off[0] += (n + 4095) // 4096 * 4096
            views.append(v)
        return orig_load(self, aid, rank, views[0], views[1], scale)
    B.LoraPool.load_adapter = load
if os.environ.get("LK") == "dummy":
    import numpy as np
    import torch
    os.environ["LK"] = "0"
    dp = B.LoraPool(4096, 4096, 2, "bf16", max_total_rank=64)
    dp.set_option(B.LORA_OPT_LOAD_KERNEL, 1)
    z = torch.zeros(64, 4096, dtype=torch.int16).pin_memory()
    dp.load_adapter(0, 64, z, z, 1.0)
    torch.cuda.synchronize()
    dp.close()
sys.argv = ["trace_layer.py"] + sys.argv[1:]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "trace_layer.py"), run_name="__main__")
