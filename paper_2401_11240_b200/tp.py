"""Tensor-parallel LoRA delta (BASELINE.json north_star).

Scheme ("BJ scheme"): rank k of a tp-way group holds A[:, H_in slice k] and
B[:, H_out slice k].  Per apply:
    1. shrink    v_k = x[:, slice k] · A[slice k, :]          (library kernel, lora_apply_shrink)
    2. all-reduce v = Σ_k v_k  (fp32, rank-r sized: c5 decode 15 KB)  -- torch.distributed / NCCL
    3. expand    y[:, out slice k] += s · v · B[:, out slice k]    (library kernel, lora_apply_expand)
so adapter bytes per GPU scale as 1/tp.  The paper's own scheme ("partition B like the base
weight ... no extra communication") is the special case split_in=False (A replicated, no collective).
Row-parallel layers (o/down: x already sharded on H_in) use split_in=True with the caller's x shard
and add into the partial (pre-all-reduce) y of the base layer.

PyTorch is plumbing here: device buffers and the NCCL all-reduce through torch.distributed.
Every arithmetic step runs in liblora.so.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np

from .binding import LoraPool


def shard_bounds(H: int, tp: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) of rank's contiguous slice of a dimension of size H (H divisible by tp)."""
    if H % tp:
        raise ValueError("dimension %d not divisible by tp=%d" % (H, tp))
    w = H // tp
    return rank * w, (rank + 1) * w


class TPLoraLayer:
    """One adapted projection on one TP rank."""

    def __init__(self, hidden_in: int, hidden_out: int, tp_rank: int, tp_size: int, max_adapters: int,
                 max_total_rank: int = 0, dtype: str = "bf16", split_in: bool = True, split_out: bool = True,
                 group=None):
        self.H_in, self.H_out = hidden_in, hidden_out
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.split_in, self.split_out = split_in, split_out
        self.in_lo, self.in_hi = shard_bounds(hidden_in, tp_size, tp_rank) if split_in else (0, hidden_in)
        self.out_lo, self.out_hi = shard_bounds(hidden_out, tp_size, tp_rank) if split_out else (0, hidden_out)
        self.group = group
        self.pool = LoraPool(self.in_hi - self.in_lo, self.out_hi - self.out_lo, max_adapters, dtype,
                             max_total_rank=max_total_rank)
        # the split (shrink | all-reduce | expand) runs every token on the decode kernels; keep
        # lora_plan's sizing consistent with that by disabling the tensor-core prefill routing
        from .binding import LORA_OPT_TC_THRESHOLD
        self.pool.set_option(LORA_OPT_TC_THRESHOLD, 1 << 30)
        self._v = None

    def load_adapter(self, aid: int, rank: int, A_full: np.ndarray, B_full: np.ndarray, scale: float) -> None:
        """A_full [rank][H_in], B_full [rank][H_out] (host arrays of the whole adapter); this rank
        keeps its slices (copied into pinned host memory for the side-stream load)."""
        import torch
        A = np.ascontiguousarray(A_full[:, self.in_lo:self.in_hi])
        B = np.ascontiguousarray(B_full[:, self.out_lo:self.out_hi])
        view = (lambda a: a.view(np.int16)) if A.dtype == np.uint16 else (lambda a: a)
        self.pool.load_adapter(aid, rank, torch.from_numpy(view(A)).pin_memory(),
                               torch.from_numpy(view(B)).pin_memory(), scale)

    def v_buffer(self, seg_indptr, adapter_ids):
        import torch
        self.pool.plan(seg_indptr, adapter_ids)
        n = max(1, self.pool.metadata()["v_floats"])
        if self._v is None or self._v.numel() < n:
            self._v = torch.empty(n, dtype=torch.float32, device="cuda")
        return self._v[:n]

    def apply(self, x_shard, y_shard, seg_indptr, adapter_ids, stream=None, all_reduce=None) -> None:
        """x_shard [T][in slice] and y_shard [T][out slice] are this rank's device tensors.
        all_reduce: callable(tensor) summing it across the TP group (default: torch.distributed
        all_reduce on self.group when tp_size > 1 and split_in)."""
        v = self.v_buffer(seg_indptr, adapter_ids)
        self.pool.apply_shrink(x_shard, seg_indptr, adapter_ids, v, stream=stream)
        if self.split_in and self.tp_size > 1:
            if all_reduce is None:
                import torch.distributed as dist
                dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
            else:
                all_reduce(v)
        self.pool.apply_expand(y_shard, v, stream=stream)

    def close(self) -> None:
        self.pool.close()
