"""Tensor-parallel LoRA delta (BASELINE.json north_star).

Scheme ("BJ scheme"): rank k of a tp-way group holds A[:, H_in slice k] and
B[:, H_out slice k].  One lora_apply_tp call per apply, entirely inside liblora.so on the caller's
stream: shrink over the rank's H_in slice -> k-reduce into the compact fp32 v [Σ_gc ntok x r] ->
ncclAllReduce(SUM) of v over the group (the library's own communicator; c5 decode: 15,360 B) ->
expand into the rank's H_out slice.  Adapter bytes per GPU scale as 1/tp.  The paper's own scheme
(partition B like the base weight, no extra communication) is split_in=False
(A replicated, no collective: the pool's A holds all of H_in).
Column-parallel layers (q/k/v/gate/up: x replicated) pass x[:, slice] as a strided view; row-parallel
layers (o/down: x already sharded) pass their x shard and add into a strided view of the partial
(pre-all-reduce) y of the base layer (y[:, out slice] of the full-width partial sum).

Torch is plumbing here: tensors, and the process group that broadcasts the NCCL unique id.
"""
from __future__ import annotations

from typing import Optional, Tuple

from .binding import LORA_OPT_TC_THRESHOLD, LoraPool, TPComm


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
                 comm: Optional[TPComm] = None):
        self.H_in, self.H_out = hidden_in, hidden_out
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.split_in, self.split_out = split_in, split_out
        self.in_lo, self.in_hi = shard_bounds(hidden_in, tp_size, tp_rank) if split_in else (0, hidden_in)
        self.out_lo, self.out_hi = shard_bounds(hidden_out, tp_size, tp_rank) if split_out else (0, hidden_out)
        self.pool = LoraPool(self.in_hi - self.in_lo, self.out_hi - self.out_lo, max_adapters, dtype,
                             max_total_rank=max_total_rank)
        # the TP path runs every token on the decode kernels; keep lora_plan's sizing consistent
        self.pool.set_option(LORA_OPT_TC_THRESHOLD, 1 << 30)
        self.comm = comm
        if comm is not None:
            self.pool.tp_init(comm)

    def load_adapter(self, aid: int, rank: int, A_full, B_full, scale: float) -> None:
        """A_full [rank][H_in], B_full [rank][H_out]: the WHOLE adapter in pinned host memory (torch
        tensors); the library copies this rank's columns with 2D copies on its side stream."""
        self.pool.load_adapter_shard(aid, rank, A_full, self.in_lo, B_full, self.out_lo, scale)

    def apply(self, x, y, seg_indptr, adapter_ids, stream=None) -> None:
        """x: [T][H_in] replicated activations (column-parallel, split_in) or this rank's [T][in slice]
        shard; y: this rank's [T][out slice] output, or the full-width partial y of a row-parallel
        layer.  Strided column views are passed through (no copies)."""
        xs = x[:, self.in_lo:self.in_hi] if x.shape[1] == self.H_in and self.split_in else x
        ys = y[:, self.out_lo:self.out_hi] if y.shape[1] == self.H_out and self.split_out else y
        if self.comm is None and self.split_in and self.tp_size > 1:
            raise ValueError("split_in with tp_size > 1 needs a TPComm (the v all-reduce)")
        if self.comm is None or not self.split_in:
            # the paper's scheme (A replicated) needs no collective: the plain apply on the B shard
            if xs.is_contiguous() and ys.is_contiguous():
                self.pool.apply(xs, ys, seg_indptr, adapter_ids, stream=stream)
                return
            raise ValueError("without a communicator x and y must be contiguous shards")
        self.pool.apply_tp(xs, ys, seg_indptr, adapter_ids, stream=stream)

    def close(self) -> None:
        self.pool.close()
