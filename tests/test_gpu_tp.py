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


@pytest.mark.parametrize("proj,tp", [("q", 2), ("k", 4), ("down", 8), ("gate", 2)])
def test_tp_emulated_matches_unsharded_oracle(torch_cuda, proj, tp):
    torch = torch_cuda
    from paper_2401_11240_b200.tp import TPLoraLayer
    b = gen.config_c5(proj, y_zero=False)
    ref = O.delta_for_batch(b, n_threads=8)
    layers = [TPLoraLayer(b.H_in, b.H_out, r, tp, 40, max_total_rank=sum(a.rank for a in b.adapters) + 8)
              for r in range(tp)]
    for L in layers:
        for a in b.adapters:
            L.load_adapter(a.id, a.rank, a.A, a.B, a.scale)
    xs = [to_torch(np.ascontiguousarray(b.x[:, L.in_lo:L.in_hi]), "cuda") for L in layers]
    ys = [to_torch(np.ascontiguousarray(b.y_in[:, L.out_lo:L.out_hi]), "cuda") for L in layers]
    vs = [L.v_buffer(b.seg_indptr, b.adapter_ids) for L in layers]
    for L, x, v in zip(layers, xs, vs):
        L.pool.apply_shrink(x, b.seg_indptr, b.adapter_ids, v)
    vsum = torch.stack(vs).sum(0)            # the SUM all-reduce, emulated
    for L, y in zip(layers, ys):
        L.pool.apply_expand(y, vsum)
    torch.cuda.synchronize()
    y = np.concatenate([from_torch(t, "bf16") for t in ys], axis=1)
    assert rel_l2(y, ref, "bf16") <= TOL["bf16"]
    for L in layers:
        L.close()


def test_tp_layer_nccl_world1(torch_cuda):
    """TPLoraLayer.apply through a real NCCL process group (world size 1 on the single GPU)."""
    torch = torch_cuda
    import torch.distributed as dist
    from paper_2401_11240_b200.tp import TPLoraLayer
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            sk.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    b = gen.config_c5("q", y_zero=False)
    ref = O.delta_for_batch(b, n_threads=8)
    L = TPLoraLayer(b.H_in, b.H_out, 0, 1, 40, max_total_rank=sum(a.rank for a in b.adapters))
    L.split_in = True
    L.tp_size = 1
    for a in b.adapters:
        L.load_adapter(a.id, a.rank, a.A, a.B, a.scale)
    x = to_torch(b.x, "cuda")
    y = to_torch(b.y_in, "cuda")
    v = L.v_buffer(b.seg_indptr, b.adapter_ids)
    L.pool.apply_shrink(x, b.seg_indptr, b.adapter_ids, v)
    dist.all_reduce(v)                       # NCCL SUM over the (1-rank) TP group
    L.pool.apply_expand(y, v)
    torch.cuda.synchronize()
    assert rel_l2(from_torch(y, "bf16"), ref, "bf16") <= TOL["bf16"]
    L.close()
    dist.destroy_process_group()


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
