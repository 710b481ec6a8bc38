"""Thin ctypes binding of liblora.so (include/lora_delta.h): argument marshalling only.

Every step of the LoRA delta runs in the library's sm_100a kernels; this module only
turns Python ints / numpy arrays / torch tensors into the C ABI's pointers and sizes.
There is no fallback: if liblora.so is missing or fails to load, import raises.
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import Dict, List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "lib", "liblora.so")
HEADER = os.path.join(ROOT, "include", "lora_delta.h")

LORA_F32, LORA_BF16 = 0, 1
LORA_POOL_HOST_ONLY = 1
LORA_KIND_NONE, LORA_KIND_DECODE, LORA_KIND_PREFILL = -1, 0, 1
LORA_OPT_TC_THRESHOLD, LORA_OPT_RESERVE_TOKENS = 1, 2
LORA_OPT_PAD_MAX_RANK, LORA_OPT_LOAD_KERNEL = 5, 6
LORA_MAX_RANK = 256

STATUS = {0: "LORA_OK", 1: "LORA_ERR_ARG", 2: "LORA_ERR_SHAPE", 3: "LORA_ERR_ALIGN",
          4: "LORA_ERR_UNKNOWN_ADAPTER", 5: "LORA_ERR_EXISTS", 6: "LORA_ERR_POOL_FULL",
          7: "LORA_ERR_NOT_PINNED", 8: "LORA_ERR_CUDA", 9: "LORA_ERR_NCCL", 10: "LORA_ERR_UNSUPPORTED"}


class LoraError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("%s: %s" % (STATUS.get(code, code), msg))
        self.code = code
        self.name = STATUS.get(code, str(code))


class PoolInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("hidden_in", "hidden_out", "max_adapters", "max_total_rank", "dtype", "elem_bytes",
                 "resident_adapters", "free_pages", "tc_threshold", "device")] + \
               [("pool_bytes", ctypes.c_int64), ("resident_bytes", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64)]


_P32 = ctypes.POINTER(ctypes.c_int32)


class MetadataView(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int32), ("S", ctypes.c_int32), ("G", ctypes.c_int32), ("L_tc", ctypes.c_int32),
                ("tok_seg", _P32), ("group_id", _P32), ("group_rank", _P32),
                ("group_scale", ctypes.POINTER(ctypes.c_float)), ("group_ntok", _P32),
                ("group_page_off", _P32), ("group_tok_off", _P32), ("group_tokens", _P32),
                ("pages", _P32), ("seg_kind", _P32),
                ("n_seg", ctypes.c_int64), ("max_rank", ctypes.c_int64), ("nseg_x_maxrank", ctypes.c_int64),
                ("sum_rank_seg", ctypes.c_int64), ("sum_rank_groups", ctypes.c_int64),
                ("sum_rank_tokens", ctypes.c_int64),
                ("n_decode_units", ctypes.c_int32), ("n_prefill_tiles", ctypes.c_int32),
                ("n_shrink_units", ctypes.c_int32), ("n_expand_units", ctypes.c_int32),
                ("v_floats", ctypes.c_int64), ("reserved0", ctypes.c_int32), ("reserved1", ctypes.c_int32),
                ("n_prefill_ctas", ctypes.c_int32), ("prefill_cluster", ctypes.c_int32)]


def header_symbols() -> List[str]:
    """Function names declared in include/lora_delta.h."""
    src = open(HEADER).read()
    return re.findall(r"^\s*(?:lora_status|const char\*|int)\s+(lora_\w+)\s*\(", src, re.M)


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError("liblora.so not built (run __graft_entry__.build() or "
                          "python paper_2401_11240_b200/build.py): " + LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    P, c_int, c_i32, c_i64, vp = ctypes.POINTER, ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "lora_pool_create": [c_int, c_int, c_int, c_int, c_int, P(vp)],
        "lora_pool_create_ex": [c_int, c_int, c_int, c_int, c_int, ctypes.c_uint, P(vp)],
        "lora_pool_destroy": [vp],
        "lora_load_adapter": [vp, c_i32, c_int, vp, vp, ctypes.c_float],
        "lora_unload_adapter": [vp, c_i32],
        "lora_adapter_ready": [vp, c_i32, P(c_int)],
        "lora_apply": [vp, vp, vp, vp, vp, c_int, vp],          # seg_indptr / adapter_ids as addresses
        "lora_plan": [vp, vp, vp, c_int],
        "lora_set_option": [vp, c_int, c_i64],
        "lora_pool_info": [vp, P(PoolInfo)],
        "lora_debug_metadata": [vp, P(MetadataView)],
        "lora_debug_adapter_pages": [vp, c_i32, _P32, c_int, P(c_int)],
        "lora_debug_read_pages": [vp, c_i32, vp, vp],
        "lora_debug_set_trace": [vp, vp],
        "lora_apply_shrink": [vp, vp, vp, vp, c_int, vp, c_i64, vp],
        "lora_apply_multi": [P(vp), P(vp), P(vp), c_int, vp, vp, c_int, vp],
        "lora_apply_expand": [vp, vp, vp, vp],
        "lora_apply_fused_base": [vp, vp, vp, vp, vp, vp, c_int, vp],
        "lora_tp_unique_id": [vp],
        "lora_tp_comm_create": [vp, c_int, c_int, P(vp)],
        "lora_tp_comm_destroy": [vp],
        "lora_tp_init": [vp, vp],
        "lora_apply_tp": [vp, vp, c_i64, vp, c_i64, vp, vp, c_int, vp],
        "lora_load_adapter_shard": [vp, c_i32, c_int, vp, c_i64, c_i64, vp, c_i64, c_i64, ctypes.c_float],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = c_int
    lib.lora_last_error.restype = ctypes.c_char_p
    lib.lora_last_error.argtypes = []
    lib.lora_abi_version.restype = c_int
    lib.lora_abi_version.argtypes = []
    return lib


LIB = _load()


def _check(rc: int) -> None:
    if rc != 0:
        raise LoraError(rc, LIB.lora_last_error().decode())


def _i32(a) -> np.ndarray:
    if type(a) is np.ndarray and a.dtype == np.int32 and a.flags.c_contiguous:
        return a   # the per-apply fast path: no copy, no conversion
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


_ADDR_CACHE: list = []   # (array, address) of the last few int32 arrays (kept alive by the cache)


def _addr(a: np.ndarray) -> int:
    """a.ctypes.data without building a ctypes helper per call (the same seg_indptr / adapter_ids
    arrays are passed to every pool of a decode step)."""
    for arr, ad in _ADDR_CACHE:
        if arr is a:
            return ad
    ad = a.__array_interface__["data"][0]
    _ADDR_CACHE.insert(0, (a, ad))
    del _ADDR_CACHE[8:]
    return ad


def _stream_ptr(stream) -> int:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    return stream if isinstance(stream, int) else int(stream.cuda_stream)


def _ptr_of(t) -> int:
    """device/host address of a torch tensor, numpy array or int."""
    if t is None:
        return 0
    dp = getattr(t, "data_ptr", None)
    if dp is not None:
        return int(dp())
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        return int(t.ctypes.data)
    raise TypeError(type(t))


TP_UNIQUE_ID_BYTES = 128


def tp_unique_id() -> bytes:
    """lora_tp_unique_id: the TP group's rendezvous id (rank 0 creates it, the others receive it)."""
    buf = ctypes.create_string_buffer(TP_UNIQUE_ID_BYTES)
    _check(LIB.lora_tp_unique_id(buf))
    return buf.raw


class TPComm:
    """lora_tp_comm: one tensor-parallel group's NCCL communicator, owned by the library."""

    def __init__(self, unique_id: bytes, tp_rank: int, tp_size: int):
        if len(unique_id) != TP_UNIQUE_ID_BYTES:
            raise ValueError("unique id must be %d bytes" % TP_UNIQUE_ID_BYTES)
        h = ctypes.c_void_p()
        _check(LIB.lora_tp_comm_create(ctypes.create_string_buffer(unique_id, TP_UNIQUE_ID_BYTES), int(tp_rank),
                                       int(tp_size), ctypes.byref(h)))
        self.handle, self.rank, self.size = h, tp_rank, tp_size

    @classmethod
    def from_process_group(cls, group=None):
        """Rank 0 of `group` (torch.distributed) creates the id and broadcasts it; collective."""
        import torch
        import torch.distributed as dist
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.zeros(TP_UNIQUE_ID_BYTES, dtype=torch.uint8, device=dev)
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(tp_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return cls(bytes(t.cpu().numpy().tobytes()), rank, size)

    def close(self) -> None:
        if self.handle:
            _check(LIB.lora_tp_comm_destroy(self.handle))
            self.handle = None


def _ld_of(t, width: int) -> int:
    """row stride (elements) of a 2D torch tensor view whose rows hold `width` contiguous elements."""
    if hasattr(t, "stride") and t.dim() == 2:
        if t.stride(1) != 1:
            raise ValueError("rows must be contiguous")
        return int(t.stride(0))
    return int(width)


def apply_multi(pools, xs, ys, seg_indptr, adapter_ids, stream=None) -> None:
    """lora_apply_multi: pools[i] applies to (xs[i], ys[i]) in one fused launch pair."""
    n = len(pools)
    ip, ids = _i32(seg_indptr), _i32(adapter_ids)
    sp = _stream_ptr(stream)
    VP = ctypes.c_void_p * n
    hp = VP(*[p.handle.value for p in pools])
    xp = VP(*[_ptr_of(x) for x in xs])
    yp = VP(*[_ptr_of(y) for y in ys])
    _check(LIB.lora_apply_multi(hp, xp, yp, n, _addr(ip), _addr(ids), int(ids.shape[0]), sp))


class LoraPool:
    """One paged adapter pool (one projection shape).  Mirrors the C calls one to one."""

    def __init__(self, hidden_in: int, hidden_out: int, max_adapters: int, dtype: str = "bf16",
                 max_total_rank: int = 0, host_only: bool = False):
        self.hidden_in, self.hidden_out = int(hidden_in), int(hidden_out)
        self.dtype = dtype
        code = {"f32": LORA_F32, "bf16": LORA_BF16}[dtype]
        h = ctypes.c_void_p()
        _check(LIB.lora_pool_create_ex(hidden_in, hidden_out, max_adapters, code, max_total_rank,
                                       LORA_POOL_HOST_ONLY if host_only else 0, ctypes.byref(h)))
        self.handle = h
        self._keep: Dict[int, tuple] = {}   # host buffers that must outlive their load

    def close(self) -> None:
        if self.handle:
            _check(LIB.lora_pool_destroy(self.handle))
            self.handle = None
            self._keep.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_adapter(self, aid: int, rank: int, A_host, B_host, scale: float) -> None:
        """A_host [rank][hidden_in], B_host [rank][hidden_out]: pinned host tensors (or None
        for host-only pools).  They are kept alive by the pool object until unload."""
        _check(LIB.lora_load_adapter(self.handle, int(aid), int(rank), _ptr_of(A_host), _ptr_of(B_host),
                                     float(scale)))
        self._keep[int(aid)] = (A_host, B_host)

    def unload_adapter(self, aid: int) -> None:
        _check(LIB.lora_unload_adapter(self.handle, int(aid)))
        self._keep.pop(int(aid), None)

    def adapter_ready(self, aid: int) -> bool:
        r = ctypes.c_int()
        _check(LIB.lora_adapter_ready(self.handle, int(aid), ctypes.byref(r)))
        return bool(r.value)

    def apply(self, x, y, seg_indptr, adapter_ids, stream=None) -> None:
        """x, y: device tensors (or raw pointers); seg_indptr / adapter_ids: host int32 arrays;
        stream: a torch.cuda.Stream, a raw cudaStream_t int, or None (current torch stream)."""
        ip, ids = _i32(seg_indptr), _i32(adapter_ids)
        _check(LIB.lora_apply(self.handle, _ptr_of(x), _ptr_of(y), _addr(ip), _addr(ids),
                              int(ids.shape[0]), _stream_ptr(stream)))

    def apply_shrink(self, x, seg_indptr, adapter_ids, v_out, stream=None) -> None:
        """Tensor-parallel first half: partial v (fp32, caller-owned device buffer v_out) over
        this pool's H_in shard.  The caller sums v_out across TP ranks, then calls apply_expand."""
        ip, ids = _i32(seg_indptr), _i32(adapter_ids)
        cap = int(v_out.numel()) if hasattr(v_out, "numel") else 0
        _check(LIB.lora_apply_shrink(self.handle, _ptr_of(x), _addr(ip), _addr(ids),
                                     int(ids.shape[0]), _ptr_of(v_out), cap, _stream_ptr(stream)))

    def apply_expand(self, y, v_in, stream=None) -> None:
        _check(LIB.lora_apply_expand(self.handle, _ptr_of(y), _ptr_of(v_in), _stream_ptr(stream)))

    def tp_init(self, comm) -> None:
        """lora_tp_init: bind this (shard) pool to the TP group's communicator (None unbinds)."""
        _check(LIB.lora_tp_init(self.handle, comm.handle if comm is not None else None))
        self._tp_comm = comm   # the communicator must outlive the binding

    def apply_tp(self, x, y, seg_indptr, adapter_ids, stream=None) -> None:
        """lora_apply_tp: shrink -> k-reduce -> NCCL all-reduce of the compact v -> expand, on `stream`.
        x / y may be strided 2D views (e.g. x[:, k0:k1] of the replicated activations)."""
        ip, ids = _i32(seg_indptr), _i32(adapter_ids)
        _check(LIB.lora_apply_tp(self.handle, _ptr_of(x), _ld_of(x, self.hidden_in), _ptr_of(y),
                                 _ld_of(y, self.hidden_out), _addr(ip), _addr(ids), int(ids.shape[0]),
                                 _stream_ptr(stream)))

    def load_adapter_shard(self, aid: int, rank: int, A_full, a_col0: int, B_full, b_col0: int, scale: float) -> None:
        """lora_load_adapter_shard: A_full [rank][H_in_full] / B_full [rank][H_out_full] pinned host tensors of
        the whole adapter; this pool keeps columns [a_col0, a_col0 + hidden_in) / [b_col0, b_col0 + hidden_out)."""
        _check(LIB.lora_load_adapter_shard(self.handle, int(aid), int(rank), _ptr_of(A_full), int(A_full.shape[1]),
                                           int(a_col0), _ptr_of(B_full), int(B_full.shape[1]), int(b_col0),
                                           float(scale)))
        self._keep[int(aid)] = (A_full, B_full)

    def apply_fused_base(self, x, W, y, seg_indptr, adapter_ids, stream=None) -> None:
        """y = x·W + s·(x·A)·B in one kernel (lora_apply_fused_base): W [H_in][H_out] bf16, y
        overwritten."""
        ip, ids = _i32(seg_indptr), _i32(adapter_ids)
        _check(LIB.lora_apply_fused_base(self.handle, _ptr_of(x), _ptr_of(W), _ptr_of(y), _addr(ip), _addr(ids),
                                         int(ids.shape[0]), _stream_ptr(stream)))

    def plan(self, seg_indptr, adapter_ids) -> None:
        ip, ids = _i32(seg_indptr), _i32(adapter_ids)
        _check(LIB.lora_plan(self.handle, _addr(ip), _addr(ids), int(ids.shape[0])))

    def set_option(self, option: int, value: int) -> None:
        _check(LIB.lora_set_option(self.handle, int(option), int(value)))

    def info(self) -> Dict[str, int]:
        i = PoolInfo()
        _check(LIB.lora_pool_info(self.handle, ctypes.byref(i)))
        return {n: getattr(i, n) for n, _ in PoolInfo._fields_}

    def metadata(self) -> Dict[str, object]:
        m = MetadataView()
        _check(LIB.lora_debug_metadata(self.handle, ctypes.byref(m)))

        def arr(p, n, dt=np.int32):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)

        G = m.G
        ntok = arr(m.group_ntok, G)
        out = {"T": m.T, "S": m.S, "G": G, "L_tc": m.L_tc,
               "tok_seg": arr(m.tok_seg, m.T), "group_id": arr(m.group_id, G),
               "group_rank": arr(m.group_rank, G), "group_scale": arr(m.group_scale, G, np.float32),
               "group_ntok": ntok, "group_page_off": arr(m.group_page_off, G),
               "group_tok_off": arr(m.group_tok_off, G),
               "group_tokens": arr(m.group_tokens, int(ntok.sum())),
               "pages": arr(m.pages, int(m.sum_rank_groups)), "seg_kind": arr(m.seg_kind, m.S)}
        for k in ("n_seg", "max_rank", "nseg_x_maxrank", "sum_rank_seg", "sum_rank_groups", "sum_rank_tokens",
                  "n_decode_units", "n_prefill_tiles", "n_shrink_units", "n_expand_units", "v_floats",
                  "n_prefill_ctas", "prefill_cluster"):
            out[k] = int(getattr(m, k))
        return out

    def release_host_buffers(self) -> None:
        """Drop the references to host buffers of adapters whose load has completed."""
        for aid in list(self._keep):
            if self.adapter_ready(aid):
                del self._keep[aid]

    def set_trace(self, dev_buf) -> None:
        _check(LIB.lora_debug_set_trace(self.handle, _ptr_of(dev_buf)))

    def adapter_pages(self, aid: int) -> List[int]:
        r = ctypes.c_int()
        _check(LIB.lora_debug_adapter_pages(self.handle, int(aid), None, 0, ctypes.byref(r)))
        buf = np.zeros(r.value, dtype=np.int32)
        _check(LIB.lora_debug_adapter_pages(self.handle, int(aid), buf.ctypes.data_as(_P32), r.value,
                                            ctypes.byref(r)))
        return buf.tolist()

    def read_pages(self, aid: int, rank: int) -> tuple:
        esz = 2 if self.dtype == "bf16" else 4
        dt = np.uint16 if esz == 2 else np.float32
        A = np.zeros((rank, self.hidden_in), dtype=dt)
        B = np.zeros((rank, self.hidden_out), dtype=dt)
        _check(LIB.lora_debug_read_pages(self.handle, int(aid), A.ctypes.data, B.ctypes.data))
        return A, B
