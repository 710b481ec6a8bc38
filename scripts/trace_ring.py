"""Per-CTA timeline of the c2 decode layer (q/k/v lora_apply_multi + o lora_apply) on the
persistent ring pair (LORA_OPT_DECODE_RING), replayed from a CUDA graph of NL layers.
Trace layout (ring_kernel.cu): per kernel [cta][64] u64: 0 start, 1 wait passed, 2+i tile i done,
62 smid, 63 end; the expand kernel's block follows the shrink's (num_sms * 64 words).
usage: python scripts/trace_ring.py [NL] [ring_cfg]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11240_b200 as L  # noqa: E402
from paper_2401_11240_b200 import binding as B  # noqa: E402
from workloads import gen  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 6
RING = int(sys.argv[2], 0) if len(sys.argv) > 2 else 1
H = 4096
SMS = torch.cuda.get_device_properties(0).multi_processor_count
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
        pool.set_option(B.LORA_OPT_DECODE_RING, RING)
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
g0 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g0, stream=st):
    step()
flush = torch.empty(512 * 2 ** 20, dtype=torch.int8, device="cuda")
for rep in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        g0.replay()
    e1.record(st)
    torch.cuda.synchronize()
    print("untraced replay %d: %.2f us per layer" % (rep, e0.elapsed_time(e1) * 1e3 / NL))
bufs = {}
for l in range(NL):
    for k, p in (("qkv", pools[l][0]), ("o", pools[l][3])):
        bufs[(l, k)] = torch.zeros(2 * SMS * 64, dtype=torch.int64, device="cuda")
        p.set_trace(bufs[(l, k)])
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    step()
for rep in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    print("traced replay %d: %.2f us per layer" % (rep, e0.elapsed_time(e1) * 1e3 / NL))
T = {k: v.cpu().numpy().reshape(2, SMS, 64).astype(np.float64) for k, v in bufs.items()}
t0 = min(a[0][a[0][:, 0] > 0, 0].min() for a in T.values())
print("per kernel (us from the first start): first start, wait first..last, end first..last, tiles/CTA max")
stats = {}
for l in range(NL):
    for k in ("qkv", "o"):
        a = T[(l, k)]
        for kk, name in ((0, "S"), (1, "E")):
            m = a[kk]
            live = m[:, 0] > 0
            m = m[live]
            ntile = (m[:, 2:62] > 0).sum(1)
            rel = (m - t0) / 1e3
            rel[m == 0] = np.nan
            print("L%d %-3s %s  start %7.2f  wait %7.2f..%7.2f  end %7.2f..%7.2f  tiles<=%d  SMs %d" % (
                l, k, name, np.nanmin(rel[:, 0]), np.nanmin(rel[:, 1]), np.nanmax(rel[:, 1]), np.nanmin(rel[:, 63]),
                np.nanmax(rel[:, 63]), ntile.max(), len(set(m[:, 62].astype(int)))))
            if l >= 1:
                d = stats.setdefault((k, name), {"start->wait": [], "wait->tile0": [], "tile gap": [], "last->end": []})
                d["start->wait"] += list((m[:, 1] - m[:, 0]) / 1e3)
                first = m[:, 2]
                d["wait->tile0"] += list((first - m[:, 1]) / 1e3)
                for row, n in zip(m, ntile):
                    if n > 1:
                        d["tile gap"] += list(np.diff(row[2:2 + n]) / 1e3)
                    d["last->end"].append((row[63] - row[1 + n]) / 1e3)
for (k, name), d in stats.items():
    print("%-3s %s " % (k, name) + "  ".join("%s med %.2f p90 %.2f" % (q, np.median(v), np.percentile(v, 90))
                                            for q, v in d.items() if v))
# CTA 0 of layer 1 qkv
a = T[(1, "qkv")]
for kk, name in ((0, "S"), (1, "E")):
    row = a[kk][0]
    n = int((row[2:62] > 0).sum())
    print("L1 qkv %s CTA0 sm %d: start %.2f wait %.2f tiles %s end %.2f" % (
        name, row[62], (row[0] - t0) / 1e3, (row[1] - t0) / 1e3,
        " ".join("%.2f" % ((v - t0) / 1e3) for v in row[2:2 + n]), (row[63] - t0) / 1e3))
