"""Helpers for the -m gpu parity tests: move a workloads.gen.Batch through the C ABI
(paper_2401_11240_b200.LoraPool) and compare with the fp64 oracle."""
import numpy as np

from oracle import oracle as O
from workloads import gen


def torch_mod():
    import torch
    return torch


def to_torch(a: np.ndarray, device=None, pin=False):
    torch = torch_mod()
    if a.dtype == np.uint16:
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.int16))
    else:
        t = torch.from_numpy(np.ascontiguousarray(a))
    if pin:
        t = t.pin_memory()
    if device is not None:
        t = t.to(device)
    return t


def from_torch(t, dtype: str) -> np.ndarray:
    a = t.detach().cpu().numpy()
    return a.view(np.uint16) if dtype == "bf16" else a


def make_pool(batch, L, extra_pages=0, max_adapters=None, L_tc=None):
    pool = L.LoraPool(batch.H_in, batch.H_out, max_adapters or (len(batch.adapters) + 4), batch.dtype,
                      max_total_rank=sum(a.rank for a in batch.adapters) + extra_pages + 1)
    if L_tc is not None:
        from paper_2401_11240_b200 import binding as B
        pool.set_option(B.LORA_OPT_TC_THRESHOLD, L_tc)
    for a in batch.adapters:
        pool.load_adapter(a.id, a.rank, to_torch(a.A, pin=True), to_torch(a.B, pin=True), a.scale)
    return pool


def run_gpu(batch, L, pool=None, y_in=None, stream=None, L_tc=None, seg_indptr=None, adapter_ids=None):
    torch = torch_mod()
    own = pool is None
    if own:
        pool = make_pool(batch, L, L_tc=L_tc)
    x = to_torch(batch.x, "cuda")
    y = to_torch(batch.y_in if y_in is None else y_in, "cuda")
    pool.apply(x, y, batch.seg_indptr if seg_indptr is None else seg_indptr,
               batch.adapter_ids if adapter_ids is None else adapter_ids, stream=stream)
    torch.cuda.synchronize()
    out = from_torch(y, batch.dtype)
    md = pool.metadata()
    if own:
        pool.close()
    return out, md


def rel_l2(y_gpu: np.ndarray, y_ref: np.ndarray, dtype: str) -> float:
    """max(global rel-L2 over all elements, every token row's own rel-L2).  The per-token term keeps
    one wrong row (or one wrong column chunk of a row) from hiding inside a large batch's global
    norm.  A row's denominator is max(its reference norm, 10 % of the batch's RMS row norm): a row
    whose delta nearly cancels (||x·A|| << ||x||·||A||, e.g. H_out = 8, rank 1) amplifies the
    fp32 / bf16 rounding of its shrink sum by that condition number -- arithmetic, not a fault
    (per-token reading).  A row whose reference is all zero must match exactly
    (reading R6): inf otherwise."""
    ref = np.asarray(y_ref, dtype=np.float64)
    g = gen.storage_to_f64(y_gpu, dtype).reshape(ref.shape)
    den = np.linalg.norm(ref)
    err = float(np.linalg.norm(g - ref) / (den if den > 0 else 1.0))
    if ref.ndim == 2 and ref.shape[0] > 0:
        dif = np.linalg.norm(g - ref, axis=1)
        rn = np.linalg.norm(ref, axis=1)
        zero = rn == 0
        if np.any(dif[zero] != 0):
            return float("inf")
        if np.any(~zero):
            floor = 0.1 * float(np.sqrt(np.mean(rn[~zero] ** 2)))
            err = max(err, float(np.max(dif[~zero] / np.maximum(rn[~zero], floor))))
    return err


TOL = {"f32": 1e-5, "bf16": 5e-3}   # BASELINE.json north_star
