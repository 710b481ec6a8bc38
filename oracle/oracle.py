"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain reference for the batched multi-adapter LoRA delta, written from the
paper.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module.  It shares no
code with the CUDA path and never imports ``paper_2401_11240_b200``.

Contents
  * ``delta``            -- the fp64 per-token delta (C, lora_oracle.c), §2.1 Eq. 1
                             applied per request and added to the base
                            output, with BASELINE north_star's scale s_a.
  * ``canonical_metadata`` -- step a1 of SURVEY §8(a): the batch metadata M1-M6 the
                            library must reproduce bit for bit (readings R8-R10).
                            The M6 features are the paper's performance-model inputs,
                            |S|·max rank (BGMV) and Σ rank (MBGMV), §5 P:751-755.
  * ``PageAllocatorReplay`` -- the pool's page allocator replayed from the sequence of
                            load/unload calls (reading R9: a page is one rank component,
                            lowest free indices first).
  * ``adapter_bytes``    -- pool byte accounting r·(H_in+H_out)·b (pin P11).

Parity pins: see tests/test_oracle_pins.py.  Parity unpinned: none of these
functions (every one has at least one pin there).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lora_oracle.c")
_LIB_DIR = os.path.join(_HERE, "_build")
_LIB = os.path.join(_LIB_DIR, "liboracle.so")

ORACLE_OK, ORACLE_ERR_UNKNOWN_ADAPTER, ORACLE_ERR_ARG = 0, 1, 2

KIND_NONE, KIND_DECODE, KIND_PREFILL = -1, 0, 1


def build(force: bool = False) -> str:
    """Compile lora_oracle.c with gcc (fp64, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        os.makedirs(_LIB_DIR, exist_ok=True)
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        lib.oracle_lora_delta.restype = ctypes.c_int
        lib.oracle_lora_delta.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int,
            P(ctypes.c_int32), P(ctypes.c_int32),
            ctypes.c_int, P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_double),
            P(ctypes.c_void_p), P(ctypes.c_void_p),
            P(ctypes.c_double), P(ctypes.c_double), P(ctypes.c_double),
            P(ctypes.c_uint8), P(ctypes.c_double), ctypes.c_int, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def delta(H_in: int, H_out: int, seg_indptr, adapter_ids, adapters: Sequence[Tuple[int, int, float, np.ndarray, np.ndarray]],
          x: np.ndarray, y_in: np.ndarray, token_mask: Optional[np.ndarray] = None,
          want_v: bool = False, n_threads: int = 1):
    """fp64 delta.  ``adapters`` = [(id, rank, scale, A[r][H_in] f64, B[r][H_out] f64)].
    x [T][H_in] and y_in [T][H_out] are float64.  Returns y_out (float64) or
    (y_out, v) with v [T][max_rank] the scaled intermediate s·(x_t A).
    Rows of masked-out tokens are returned as NaN."""
    lib = _load()
    ip = np.ascontiguousarray(seg_indptr, dtype=np.int32)
    ids = np.ascontiguousarray(adapter_ids, dtype=np.int32)
    S = int(ids.shape[0])
    assert ip.shape[0] == S + 1
    T = int(ip[-1]) if S > 0 else 0
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(T, H_in)
    y_in = np.ascontiguousarray(y_in, dtype=np.float64).reshape(T, H_out)
    y_out = np.full((T, H_out), np.nan, dtype=np.float64)
    n = len(adapters)
    ad_id = np.array([a[0] for a in adapters], dtype=np.int32)
    ad_rank = np.array([a[1] for a in adapters], dtype=np.int32)
    ad_scale = np.array([a[2] for a in adapters], dtype=np.float64)
    As = [np.ascontiguousarray(a[3], dtype=np.float64) for a in adapters]
    Bs = [np.ascontiguousarray(a[4], dtype=np.float64) for a in adapters]
    for (aid, r, _s, A, B) in zip(ad_id, ad_rank, ad_scale, As, Bs):
        assert A.shape == (r, H_in) and B.shape == (r, H_out), (aid, A.shape, B.shape)
    pA = (ctypes.c_void_p * max(n, 1))(*[a.ctypes.data for a in As])
    pB = (ctypes.c_void_p * max(n, 1))(*[b.ctypes.data for b in Bs])
    mask = None
    if token_mask is not None:
        mask = np.ascontiguousarray(token_mask, dtype=np.uint8)
        assert mask.shape == (T,)
    v_stride = max([int(r) for r in ad_rank] + [1])
    v = np.zeros((T, v_stride), dtype=np.float64) if want_v else None
    rc = lib.oracle_lora_delta(
        H_in, H_out, S, _ptr(ip, ctypes.c_int32), _ptr(ids, ctypes.c_int32),
        n, _ptr(ad_id, ctypes.c_int32), _ptr(ad_rank, ctypes.c_int32), _ptr(ad_scale, ctypes.c_double),
        pA, pB, _ptr(x, ctypes.c_double), _ptr(y_in, ctypes.c_double), _ptr(y_out, ctypes.c_double),
        None if mask is None else _ptr(mask, ctypes.c_uint8),
        None if v is None else _ptr(v, ctypes.c_double), v_stride, int(n_threads))
    if rc == ORACLE_ERR_UNKNOWN_ADAPTER:
        raise KeyError("unknown adapter id in adapter_ids")
    if rc != ORACLE_OK:
        raise ValueError("oracle_lora_delta: bad arguments (rc=%d)" % rc)
    return (y_out, v) if want_v else y_out


def adapter_bytes(rank: int, H_in: int, H_out: int, elem_bytes: int) -> int:
    """Bytes one adapter occupies in a pool: r·(H_in + H_out)·b (A rows + B rows)."""
    return int(rank) * (int(H_in) + int(H_out)) * int(elem_bytes)


# --------------------------------------------------------------------------
# page allocator replay (reading R9)
# --------------------------------------------------------------------------
class PoolFull(Exception):
    pass


class PageAllocatorReplay:
    """A pool of ``n_pages`` pages (one page = one rank component) and at most
    ``max_adapters`` resident adapters.  load(id, r) takes the r lowest free
    page indices in ascending order; unload(id) frees them at call time."""

    def __init__(self, n_pages: int, max_adapters: int):
        self.n_pages = int(n_pages)
        self.max_adapters = int(max_adapters)
        self.free = [True] * self.n_pages
        self.table: Dict[int, Tuple[int, float, List[int]]] = {}

    def load(self, aid: int, rank: int, scale: float = 1.0) -> List[int]:
        if aid in self.table:
            raise KeyError("adapter %d already loaded" % aid)
        if len(self.table) >= self.max_adapters:
            raise PoolFull("adapter slots exhausted")
        pages = [p for p in range(self.n_pages) if self.free[p]][:rank]
        if len(pages) < rank:
            raise PoolFull("page budget exhausted")
        for p in pages:
            self.free[p] = False
        self.table[aid] = (int(rank), float(np.float32(scale)), pages)
        return list(pages)

    def unload(self, aid: int) -> None:
        rank, scale, pages = self.table.pop(aid)
        for p in pages:
            self.free[p] = True

    def pages_of(self, aid: int) -> List[int]:
        return list(self.table[aid][2])


# --------------------------------------------------------------------------
# canonical batch metadata M1-M6 (readings R8, R10)
# --------------------------------------------------------------------------
def canonical_metadata(seg_indptr, adapter_ids, table: Dict[int, Tuple[int, float, List[int]]],
                       L_tc: int) -> Dict[str, object]:
    """table: id -> (rank, scale, pages).  Returns the M1-M6 dict:
      tok_seg[T]                            M1
      group_id/rank/scale/ntok/page_off/tok_off   M2 (groups = distinct ids >= 0 owning >= 1 token, ascending)
      group_tokens[]                        M3 (token indices per group, ascending)
      pages[sum_G r]                        M4 (each group's pages in rank order)
      seg_kind[S]                           M5 (PREFILL if id>=0 and len >= L_tc; DECODE if id>=0 and 1<=len<L_tc; else NONE)
      features: n_seg, max_rank, nseg_x_maxrank, sum_rank_seg, sum_rank_groups, sum_rank_tokens  M6
    """
    ip = [int(v) for v in seg_indptr]
    ids = [int(v) for v in adapter_ids]
    S = len(ids)
    T = ip[S] if S > 0 else 0
    for i in ids:
        if i >= 0 and i not in table:
            raise KeyError("unknown adapter id %d" % i)
    tok_seg = []
    for i in range(S):
        for _t in range(ip[i], ip[i + 1]):
            tok_seg.append(i)
    owned = sorted(set(ids[i] for i in range(S) if ids[i] >= 0 and ip[i + 1] > ip[i]))
    group_id, group_rank, group_scale, group_ntok, group_page_off, group_tok_off = [], [], [], [], [], []
    group_tokens, pages = [], []
    for g in owned:
        rank, scale, pg = table[g]
        toks = [t for t in range(T) if ids[tok_seg[t]] == g]
        group_id.append(g)
        group_rank.append(rank)
        group_scale.append(float(np.float32(scale)))
        group_ntok.append(len(toks))
        group_page_off.append(len(pages))
        group_tok_off.append(len(group_tokens))
        group_tokens.extend(toks)
        pages.extend(pg[:rank])
    seg_kind = []
    n_seg, max_rank, sum_rank_seg, sum_rank_tokens = 0, 0, 0, 0
    for i in range(S):
        L = ip[i + 1] - ip[i]
        if ids[i] < 0 or L == 0:
            seg_kind.append(KIND_NONE)
            continue
        seg_kind.append(KIND_PREFILL if L >= L_tc else KIND_DECODE)
        r = table[ids[i]][0]
        n_seg += 1
        max_rank = max(max_rank, r)
        sum_rank_seg += r
        sum_rank_tokens += r * L
    return {
        "T": T, "S": S, "G": len(owned), "L_tc": int(L_tc),
        "tok_seg": np.array(tok_seg, dtype=np.int32),
        "group_id": np.array(group_id, dtype=np.int32),
        "group_rank": np.array(group_rank, dtype=np.int32),
        "group_scale": np.array(group_scale, dtype=np.float32),
        "group_ntok": np.array(group_ntok, dtype=np.int32),
        "group_page_off": np.array(group_page_off, dtype=np.int32),
        "group_tok_off": np.array(group_tok_off, dtype=np.int32),
        "group_tokens": np.array(group_tokens, dtype=np.int32),
        "pages": np.array(pages, dtype=np.int32),
        "seg_kind": np.array(seg_kind, dtype=np.int32),
        "n_seg": n_seg, "max_rank": max_rank, "nseg_x_maxrank": n_seg * max_rank,
        "sum_rank_seg": sum_rank_seg, "sum_rank_groups": int(sum(group_rank)),
        "sum_rank_tokens": sum_rank_tokens,
    }


def work_units(kind: str, ranks: Sequence[int], H: int) -> int:
    """SPEC batched_kernels instrumentation: multiply-accumulates charged
    by a padded BGMV (|S|·max r·2H) or a padding-free MBGMV (Σ r·2H).  Defined from the
    M6 features so the pin checks those features against the paper's toy numbers."""
    if kind == "bgmv":
        return len(ranks) * max(ranks) * 2 * H
    if kind == "mbgmv":
        return sum(ranks) * 2 * H
    raise ValueError(kind)


# --------------------------------------------------------------------------
# convenience: run the oracle on a workloads.gen.Batch
# --------------------------------------------------------------------------
def delta_for_batch(batch, token_mask=None, want_v: bool = False, n_threads: int = 1, y_in=None):
    from workloads.gen import storage_to_f64
    ads = [(a.id, a.rank, a.scale, storage_to_f64(a.A, batch.dtype), storage_to_f64(a.B, batch.dtype))
           for a in batch.adapters]
    x = storage_to_f64(batch.x, batch.dtype)
    y = storage_to_f64(batch.y_in if y_in is None else y_in, batch.dtype)
    return delta(batch.H_in, batch.H_out, batch.seg_indptr, batch.adapter_ids, ads, x, y,
                 token_mask=token_mask, want_v=want_v, n_threads=n_threads)
