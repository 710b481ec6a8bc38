"""Prefill CTAs-per-tile sweep: c3 (and the c5 shapes) with LORA_EXP_PF_SPLIT=s forcing s CTAs per
128-token tile (split-K clusters for s <= 8), one subprocess per s (the override is read once per
process).  Prints device time per apply and HBM roofline fraction.
usage: python scripts/prefill_split_sweep.py [s ...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2401_11240_b200 as L
from workloads import gen
peak = json.load(open(os.path.join(%r, "MEASURED_PEAKS.json")))["hbm_gbs"]
out = {}
for name, b in (("c3", gen.config_c3()), ("c5q", gen.config_c5("q", prefill=True)),
                ("c5down", gen.config_c5("down", prefill=True))):
    NP = 3
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
    with torch.cuda.stream(st):
        for p, y in zip(pools, ys):
            p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
    torch.cuda.synchronize()
    md = pools[0].metadata()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for p, y in zip(pools, ys):
            p.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
    flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
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
    us = float(np.median(ts))
    sum_r = sum(a.rank for a in b.adapters)
    byts = 2 * (sum_r * (b.H_in + b.H_out) + b.T * b.H_in + 2 * b.T * b.H_out)
    out[name] = (round(us, 1), round(byts / (us * 1e-6) / 1e9 / peak, 3), md["n_prefill_tiles"])
    del g
    for p in pools:
        p.close()
print(json.dumps(out))
''' % (ROOT, ROOT)

splits = [int(s) for s in sys.argv[1:]] or [0, 2, 4]
for s in splits:
    env = dict(os.environ)
    env.pop("LORA_EXP_PF_SPLIT", None)
    if s:
        env["LORA_EXP_PF_SPLIT"] = str(s)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, cwd=ROOT)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-600:]
    print("split=%s  %s   (us/apply, HBM frac, tiles)" % (s or "default", line), flush=True)
