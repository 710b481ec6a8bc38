"""Small invocations of every kernel path through the C ABI, for compute-sanitizer
(scripts/sanitize.sh runs memcheck / racecheck / synccheck / initcheck over each case).
Each case also checks its result against the fp64 oracle, so a clean sanitizer run is a run of a
correct kernel.  usage: python scripts/sanitize_cases.py CASE   (CASE in CASES below)"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2401_11240_b200 as L  # noqa: E402
from gpu_util import TOL, from_torch, make_pool, rel_l2, to_torch  # noqa: E402
from oracle import oracle as O  # noqa: E402
from workloads import gen  # noqa: E402


def check(b, y):
    ref = O.delta_for_batch(b, n_threads=8)
    e = rel_l2(from_torch(y, b.dtype), ref, b.dtype)
    assert e <= TOL[b.dtype], e
    return e


def run_apply(b, L_tc=None, graph=False):
    pool = make_pool(b, L, L_tc=L_tc)
    x, y = to_torch(b.x, "cuda"), to_torch(b.y_in, "cuda")
    if graph:
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)   # sizes scratch
        torch.cuda.synchronize()
        y.copy_(to_torch(b.y_in, "cuda"))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)
        y.copy_(to_torch(b.y_in, "cuda"))
        with torch.cuda.stream(st):
            g.replay()
    else:
        pool.apply(x, y, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    md = pool.metadata()
    pool.close()
    return check(b, y), md


def case_c1():          # fp32 SIMT shrink/expand (decode and the two 8-token segments)
    return run_apply(gen.config_c1(y_zero=False))


def case_c1p():         # bf16 prefill tiles on tcgen05 (ragged 1..300 tokens, ranks 1..128) + decode pair
    return run_apply(gen.config_c1_prefill_tiles(y_zero=False))


def case_c2():          # bf16 decode pair (mma.sync), single apply, then a CUDA-graph replay
    run_apply(gen.config_c2(y_zero=False))
    return run_apply(gen.config_c2(zipf=True, y_zero=False, tag=5), graph=True)


def case_c2_multi():    # q/k/v in one lora_apply_multi launch pair
    b = gen.config_c2(y_zero=False)
    pools = [make_pool(b, L) for _ in range(3)]
    x = to_torch(b.x, "cuda")
    ys = [to_torch(b.y_in, "cuda") for _ in range(3)]
    L.apply_multi(pools, [x] * 3, ys, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    for p in pools:
        p.close()
    return [check(b, y) for y in ys]


def case_c5_splitk():   # few-tile prefill: split-K clusters exchanging partials through L2 (H_in > H_out)
    b = gen.build_batch("sk", 516, "bf16", 4096, 1024, [256, 200], [0, 1], {0: 128, 1: 24}, y_zero=False)
    e, md = run_apply(b)
    assert md["prefill_cluster"] > 1, md["prefill_cluster"]
    return e, md["prefill_cluster"]


def case_c5_colsplit():  # one 512-token segment: >8 CTAs per tile, column split with recomputed shrink
    b = gen.build_batch("cs", 515, "bf16", 1024, 4096, [512], [0], {0: 64}, y_zero=False)
    return run_apply(b)


def case_fused_base():  # NEXT f2: y = x·W + delta in one tcgen05 kernel (box and gather4 loads)
    b = gen.build_batch("f2", 814, "bf16", 256, 512, [300, 1, 129], [0, -1, 1], {0: 8, 1: 64}, y_zero=True)
    pool = make_pool(b, L)
    w = gen.storage_to_f64(gen.make_rows(814, 77, 0, b.H_in, b.H_out, "bf16"), "bf16") / np.sqrt(b.H_in)
    W = gen.f32_to_storage(w.astype(np.float32), "bf16")
    y = torch.zeros((b.T, b.H_out), dtype=torch.int16, device="cuda")
    pool.apply_fused_base(to_torch(b.x, "cuda"), to_torch(W, "cuda"), y, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    got = gen.storage_to_f64(from_torch(y, "bf16"), "bf16").reshape(b.T, b.H_out)
    ref = (gen.storage_to_f64(b.x, "bf16").reshape(b.T, b.H_in) @ gen.storage_to_f64(W, "bf16").reshape(b.H_in, b.H_out)
           + O.delta_for_batch(b, n_threads=8).reshape(b.T, b.H_out))
    e = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert e <= 5e-3, e
    pool.close()
    return e


def case_tp_split():    # TP shard: shrink + in-kernel k-reduce (counters) + expand of the compact v
    from paper_2401_11240_b200.tp import TPLoraLayer
    b = gen.config_c5("k", y_zero=False)
    full = {a.id: (to_torch(a.A, pin=True), to_torch(a.B, pin=True)) for a in b.adapters}
    lays = [TPLoraLayer(b.H_in, b.H_out, r, 2, 40, max_total_rank=sum(a.rank for a in b.adapters)) for r in range(2)]
    for lay in lays:
        for a in b.adapters:
            lay.load_adapter(a.id, a.rank, full[a.id][0], full[a.id][1], a.scale)
    vs = []
    for lay in lays:
        x = to_torch(np.ascontiguousarray(b.x[:, lay.in_lo:lay.in_hi]), "cuda")
        lay.pool.plan(b.seg_indptr, b.adapter_ids)
        v = torch.empty(lay.pool.metadata()["v_floats"], dtype=torch.float32, device="cuda")
        for _ in range(2):   # twice: the per-gc counters must re-arm
            lay.pool.apply_shrink(x, b.seg_indptr, b.adapter_ids, v)
        vs.append(v)
    vsum = vs[0] + vs[1]
    ys = [to_torch(np.ascontiguousarray(b.y_in[:, lay.out_lo:lay.out_hi]), "cuda") for lay in lays]
    for lay, y in zip(lays, ys):
        lay.pool.apply_expand(y, vsum)
    torch.cuda.synchronize()
    y = np.concatenate([from_torch(t, "bf16") for t in ys], axis=1)
    e = rel_l2(y, O.delta_for_batch(b, n_threads=8), "bf16")
    assert e <= TOL["bf16"], e
    for lay in lays:
        lay.close()
    return e


def case_load_kernel():  # zero-copy cold-start gather kernel (UVA reads of pinned rows)
    b = gen.config_c2()
    pool = L.LoraPool(b.H_in, b.H_out, 40, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
    pool.set_option(L.binding.LORA_OPT_LOAD_KERNEL, 1)
    for a in b.adapters:
        pool.load_adapter(a.id, a.rank, to_torch(a.A, pin=True), to_torch(a.B, pin=True), a.scale)
    torch.cuda.synchronize()
    for a in b.adapters[:4]:
        A, B = pool.read_pages(a.id, a.rank)
        assert np.array_equal(A, a.A) and np.array_equal(B, a.B)
    pool.close()
    return "bitwise"


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    name = sys.argv[1]
    print(name, CASES[name](), flush=True)
