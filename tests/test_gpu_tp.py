"""Tensor-parallel variant (pin P13): sharded results vs the UNSHARDED oracle.
On one GPU the tp ranks are emulated by tp pools on the same device (the SUM all-reduce of the
partial v is an elementwise add); a world-size-1 NCCL group exercises TPLoraLayer.apply's
collective path.  Multi-process coverage of the decomposition runs on CPU with gloo
(tests/test_tp_gloo.py)."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

from gpu_util import TOL, from_torch, rel_l2, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _pinned_full(b, torch):
    """every adapter's full A / B as pinned host tensors (the TP shard loads copy their columns)."""
    return {a.id: (to_torch(a.A, pin=True), to_torch(a.B, pin=True)) for a in b.adapters}


def _compact_v_ref(md, b, ref_v):
    """the oracle's v (s·x·A, fp64 [T][max r]) rearranged into the library's compact layout
    [gc][ntok][round_up(r, 4)] (groups ascending, each group's tokens in chunks of 8), unscaled."""
    scale = {a.id: a.scale for a in b.adapters}
    out = []
    for g in range(md["G"]):
        gid, r = int(md["group_id"][g]), int(md["group_rank"][g])
        toks = md["group_tokens"][md["group_tok_off"][g]: md["group_tok_off"][g] + md["group_ntok"][g]]
        rs = (r + 3) // 4 * 4
        for c0 in range(0, len(toks), 8):
            for t in toks[c0:c0 + 8]:
                row = np.zeros(rs)
                row[:r] = ref_v[t, :r] / scale[gid]
                out.append(row)
    return np.concatenate(out) if out else np.zeros(0)


@pytest.mark.parametrize("proj,tp", [("q", 2), ("k", 4), ("down", 8), ("gate", 2)])
def test_tp_emulated_matches_unsharded_oracle(torch_cuda, proj, tp):
    """tp shard pools on one GPU (loaded with lora_load_adapter_shard from the full pinned adapters);
    lora_apply_shrink's compact k-reduced v summed across the emulated ranks (the SUM all-reduce)
    equals the oracle's v (P13), and lora_apply_expand then gives the unsharded oracle's y."""
    torch = torch_cuda
    from paper_2401_11240_b200.tp import TPLoraLayer
    b = gen.config_c5(proj, y_zero=False)
    ref, ref_v = O.delta_for_batch(b, n_threads=8, want_v=True)
    full = _pinned_full(b, torch)
    layers = [TPLoraLayer(b.H_in, b.H_out, r, tp, 40, max_total_rank=sum(a.rank for a in b.adapters) + 8)
              for r in range(tp)]
    for L in layers:
        for a in b.adapters:
            L.load_adapter(a.id, a.rank, full[a.id][0], full[a.id][1], a.scale)
    xs = [to_torch(np.ascontiguousarray(b.x[:, L.in_lo:L.in_hi]), "cuda") for L in layers]
    ys = [to_torch(np.ascontiguousarray(b.y_in[:, L.out_lo:L.out_hi]), "cuda") for L in layers]
    vs = []
    for L, x in zip(layers, xs):
        L.pool.plan(b.seg_indptr, b.adapter_ids)
        v = torch.empty(L.pool.metadata()["v_floats"], dtype=torch.float32, device="cuda")
        L.pool.apply_shrink(x, b.seg_indptr, b.adapter_ids, v)
        vs.append(v)
    vsum = torch.stack(vs).sum(0)            # the SUM all-reduce, emulated
    md = layers[0].pool.metadata()
    assert vsum.numel() == md["v_floats"]
    vref = _compact_v_ref(md, b, ref_v)
    vg = vsum.cpu().double().numpy()
    assert np.linalg.norm(vg - vref) / np.linalg.norm(vref) <= 1e-5   # fp32 sums of bf16 products (P13)
    for L, y in zip(layers, ys):
        L.pool.apply_expand(y, vsum)
    torch.cuda.synchronize()
    y = np.concatenate([from_torch(t, "bf16") for t in ys], axis=1)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
    for L in layers:
        L.close()


def _nccl_world1(torch):
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            sk.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    return dist


@pytest.mark.parametrize("proj", ["q", "k", "down"])
def test_tp_library_nccl_world1(torch_cuda, proj):
    """lora_apply_tp through the library's own NCCL communicator (lora_tp_comm_create from an id
    broadcast over a world-1 torch NCCL group): column-parallel with the replicated x passed as a
    strided view; row-parallel adding into a strided column view of a full-width partial y; and
    inside a CUDA graph.  The communicator error path is reachable (LORA_ERR_NCCL)."""
    torch = torch_cuda
    dist = _nccl_world1(torch)
    import paper_2401_11240_b200 as L
    from paper_2401_11240_b200.binding import TPComm
    from paper_2401_11240_b200.tp import TPLoraLayer
    b = gen.config_c5(proj, y_zero=False)
    ref = O.delta_for_batch(b, n_threads=8)
    full = _pinned_full(b, torch)
    comm = TPComm.from_process_group()
    lay = TPLoraLayer(b.H_in, b.H_out, 0, 1, 40, max_total_rank=sum(a.rank for a in b.adapters), comm=comm)
    for a in b.adapters:
        lay.load_adapter(a.id, a.rank, full[a.id][0], full[a.id][1], a.scale)
    x = to_torch(b.x, "cuda")
    y = to_torch(b.y_in, "cuda")
    lay.apply(x, y, b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    assert rel_l2(from_torch(y, "bf16"), ref, "bf16") <= TOL["bf16"]
    # strided views: x with extra columns (row stride > H_in) and y inside a wider partial-sum buffer
    xw = torch.zeros(b.T, b.H_in + 64, dtype=torch.int16, device="cuda")
    xw[:, 32:32 + b.H_in] = x
    yw = torch.zeros(b.T, b.H_out + 128, dtype=torch.int16, device="cuda")
    yw[:, 64:64 + b.H_out] = to_torch(b.y_in, "cuda")
    lay.pool.apply_tp(xw[:, 32:32 + b.H_in], yw[:, 64:64 + b.H_out], b.seg_indptr, b.adapter_ids)
    torch.cuda.synchronize()
    assert rel_l2(from_torch(yw[:, 64:64 + b.H_out].contiguous(), "bf16"), ref, "bf16") <= TOL["bf16"]
    assert not yw[:, :64].any() and not yw[:, 64 + b.H_out:].any()   # columns outside the view untouched
    # CUDA graph: 3 replays add the delta 3 times
    y2 = to_torch(b.y_in, "cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        lay.apply(x, y2, b.seg_indptr, b.adapter_ids, stream=st)   # sizes scratch outside the capture
    torch.cuda.synchronize()
    y2.copy_(to_torch(b.y_in, "cuda"))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        lay.apply(x, y2, b.seg_indptr, b.adapter_ids, stream=st)
    y2.copy_(to_torch(b.y_in, "cuda"))
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y2, y)
    # the id must be 128 bytes; a garbage id fails inside NCCL with LORA_ERR_NCCL, not a crash
    with pytest.raises(L.LoraError) as ei:
        lay.pool.apply_tp(x, y, np.array([0, 1], np.int32), np.array([12345], np.int32))
    assert ei.value.code == 4   # unknown adapter: validated before any launch
    lay.close()
    comm.close()


def test_tp_shard_load_bytes_exact(torch_cuda):
    """lora_load_adapter_shard lands exactly the rank's columns of the full adapter (2D copies)."""
    torch = torch_cuda
    b = gen.config_c5("k")
    full = _pinned_full(b, torch)
    from paper_2401_11240_b200.tp import TPLoraLayer
    for tp, rank in ((2, 1), (8, 5)):
        lay = TPLoraLayer(b.H_in, b.H_out, rank, tp, 40, max_total_rank=sum(a.rank for a in b.adapters))
        for a in b.adapters:
            lay.load_adapter(a.id, a.rank, full[a.id][0], full[a.id][1], a.scale)
        torch.cuda.synchronize()
        for a in b.adapters[:6]:
            A, B = lay.pool.read_pages(a.id, a.rank)
            assert np.array_equal(A, a.A[:, lay.in_lo:lay.in_hi]) and np.array_equal(B, a.B[:, lay.out_lo:lay.out_hi])
        lay.close()


def test_split_apply_equals_fused_apply(torch_cuda):
    """shrink + expand (no collective) reproduces lora_apply bit for bit on decode batches."""
    torch = torch_cuda
    import paper_2401_11240_b200 as L
    from gpu_util import make_pool
    b = gen.config_c2(y_zero=False)
    pool = make_pool(b, L)
    x = to_torch(b.x, "cuda")
    y1 = to_torch(b.y_in, "cuda")
    y2 = to_torch(b.y_in, "cuda")
    pool.apply(x, y1, b.seg_indptr, b.adapter_ids)
    pool.plan(b.seg_indptr, b.adapter_ids)
    v = torch.empty(pool.metadata()["v_floats"], dtype=torch.float32, device="cuda")
    pool.apply_shrink(x, b.seg_indptr, b.adapter_ids, v)
    pool.apply_expand(y2, v)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    with pytest.raises(L.LoraError):
        pool.apply_expand(y2, v)             # no pending shrink
    pool.close()


@pytest.mark.parametrize("proj,tp,kind", [("q", 4, "column"), ("down", 2, "row")])
def test_tp_nocomm_schemes(torch_cuda, proj, tp, kind):
    """The TP schemes without a collective (bench c5 `nocomm`).  Column-parallel: every
    rank keeps A whole and B's output-column slice (the paper's scheme) -- its y slice is the
    oracle's, exactly as an unsharded apply.  Row-parallel: rank k keeps A's rows of its x shard and B
    whole and adds s·(x_k·A_k)·B into its partial y; the sum over ranks (the base layer's own
    all-reduce, emulated) is the unsharded oracle's delta (linearity; each partial y is rounded once)."""
    torch = torch_cuda
    import paper_2401_11240_b200 as L
    b = gen.config_c5(proj, y_zero=True)
    ref = O.delta_for_batch(b, n_threads=16).reshape(b.T, b.H_out)
    full = _pinned_full(b, torch)
    x = to_torch(b.x, "cuda")
    total = np.zeros((b.T, b.H_out))
    got_cols = []
    for k in range(tp):
        hi, ho = (b.H_in // tp, b.H_out) if kind == "row" else (b.H_in, b.H_out // tp)
        pool = L.LoraPool(hi, ho, 40, "bf16", max_total_rank=sum(a.rank for a in b.adapters) + 8)
        for a in b.adapters:
            A, B = full[a.id]
            pool.load_adapter_shard(a.id, a.rank, A, k * hi if kind == "row" else 0, B, 0 if kind == "row" else k * ho,
                                    a.scale)
        xk = x[:, k * hi:(k + 1) * hi].contiguous() if kind == "row" else x
        y = torch.zeros((b.T, ho), dtype=torch.int16, device="cuda")
        pool.apply(xk, y, b.seg_indptr, b.adapter_ids)
        torch.cuda.synchronize()
        yk = gen.storage_to_f64(from_torch(y, "bf16"), "bf16").reshape(b.T, ho)
        if kind == "row":
            total += yk
        else:
            got_cols.append(yk)
        pool.close()
    got = total if kind == "row" else np.concatenate(got_cols, axis=1)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= TOL["bf16"]
