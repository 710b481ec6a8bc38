"""A/B of prebuilt liblora.so files on the prefill shapes (c3 and the c5 70B shapes), interleaved.
Each measurement: a CUDA graph of NP applies on distinct pools, replayed back to back (steady state:
the previous apply's dirty y lines drain during the next, as in bench.py's prefill object); device
time per apply and the HBM roofline fraction of the algorithmic bytes.
usage: python scripts/prefill_ab.py A.so B.so [reps] [cases]   (the in-tree library is restored afterwards)
cases: comma list of c3,c5q,c5gate,c5down (default) and c3w (c3 shapes with ranks 144/192/256)"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2401_11240_b200", "lib", "liblora.so")

CHILD = r'''
import json, os, sys
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2401_11240_b200 as L
from workloads import gen
peak = json.load(open(os.path.join(%r, "MEASURED_PEAKS.json")))["hbm_gbs"]
out = {}
want = "@CASES@".split(",")
mk = {"c3": lambda: gen.config_c3(), "c5q": lambda: gen.config_c5("q", prefill=True),
      "c5gate": lambda: gen.config_c5("gate", prefill=True), "c5down": lambda: gen.config_c5("down", prefill=True),
      "c3w": lambda: gen.build_batch("c3w", 31, "bf16", 4096, 4096, [512] * 32, list(range(32)),
                                     {i: (144, 192, 256)[i %% 3] for i in range(32)})}
NPS = {"c3": 8, "c5q": 6, "c5gate": 3, "c5down": 3, "c3w": 6}
for name in want:
    b, NP = mk[name](), NPS[name]
    pools = []
    for _ in range(NP):
        pool = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
        for a in b.adapters:
            pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                              torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
        pools.append(pool)
    x = torch.from_numpy(b.x.view(np.int16)).cuda()
    ys = [torch.zeros(b.T, b.H_out, dtype=torch.int16, device="cuda") for _ in pools]
    st = torch.cuda.Stream()
    def body():
        for p, y in zip(pools, ys):
            p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
    with torch.cuda.stream(st):
        body()
    torch.cuda.synchronize()
    md = pools[0].metadata()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        body()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    R = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        for _ in range(R):
            g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (R * NP)
    sum_r = sum(a.rank for a in b.adapters)
    byts = 2 * (sum_r * (b.H_in + b.H_out) + b.T * b.H_in + 2 * b.T * b.H_out)
    out[name] = [round(us, 2), round(byts / (us * 1e-6) / 1e9 / peak, 4), md["n_prefill_tiles"]]
    del g
    for p in pools:
        p.close()
print(json.dumps(out))
''' % (ROOT, ROOT)


def main():
    libs = sys.argv[1:3]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    cases = sys.argv[4] if len(sys.argv) > 4 else "c3,c5q,c5gate,c5down"
    keep = LIB + ".ab_keep"
    shutil.copy(LIB, keep)
    try:
        for rep in range(reps):
            for tag, so in zip("AB", libs):
                shutil.copy(so, LIB)
                r = subprocess.run([sys.executable, "-c", CHILD.replace("@CASES@", cases)], capture_output=True, text=True, cwd=ROOT, timeout=600)
                line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-800:]
                print("%s rep%d %s   (us/apply, HBM frac, tiles)" % (tag, rep, line), flush=True)
    finally:
        shutil.copy(keep, LIB)
        os.remove(keep)


if __name__ == "__main__":
    main()
