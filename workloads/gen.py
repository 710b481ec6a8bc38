"""Seeded synthetic workloads for the batched multi-adapter LoRA delta.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA
path (``paper_2401_11240_b200/``).  It draws random numbers and lays out
buffers; it contains none of the method's arithmetic (no products, no sums of
x·A·B).  Casting float32 draws to bf16 (round-to-nearest-even) and decoding
bf16 bit patterns back to float are storage conversions, not the method.

Recipe:
  * x ~ N(0,1); A_a[j][k] ~ N(0, 1/H_in); B_a[j][n] ~ N(0, 1/r_a);
    s_a = 16 / r_a (alpha = 16, LoRA convention); y_in = 0 (run A) or N(0,1) (run B).
  * The paper serves dummy LoRA weights (§6.1), so any
    distribution is faithful; these keep bf16 values O(1).
  * A is stored rank-major, [r][H_in] (row j = column j of the paper's
    A ∈ R^{H1×r}), B as [r][H_out] (the paper's B ∈ R^{r×H2}).
  * Every array is derived from numpy PCG64 seeded by a SeedSequence over
    (config seed, stream tag, indices), so any adapter can be regenerated
    alone (the 1000-adapter pool of config 4 is never materialised at once).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

BASE_SEED = 240111240  # seed = 240111240 + config index

DTYPES = ("f32", "bf16")

# stream tags for SeedSequence entropy
_TAG_X, _TAG_Y, _TAG_A, _TAG_B, _TAG_BATCH = 1, 2, 3, 4, 5


# --------------------------------------------------------------------------
# storage conversions (bf16 is carried as uint16 bit patterns)
# --------------------------------------------------------------------------
def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round float32 to bf16 with round-to-nearest-even; returns uint16 bits."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


def storage_to_f64(a: np.ndarray, dtype: str) -> np.ndarray:
    """Exact widening of a stored buffer (bf16 bits or float32) to float64."""
    if dtype == "bf16":
        return bf16_bits_to_f32(a).astype(np.float64)
    if dtype == "f32":
        return np.asarray(a, dtype=np.float32).astype(np.float64)
    raise ValueError(dtype)


def f32_to_storage(a: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return f32_to_bf16_bits(a)
    if dtype == "f32":
        return np.ascontiguousarray(a, dtype=np.float32)
    raise ValueError(dtype)


def elem_bytes(dtype: str) -> int:
    return {"f32": 4, "bf16": 2}[dtype]


def _rng(*entropy: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(e) for e in entropy])))


# --------------------------------------------------------------------------
# data classes
# --------------------------------------------------------------------------
@dataclasses.dataclass
class Adapter:
    id: int
    rank: int
    scale: float          # exactly representable float32
    A: np.ndarray         # [rank][H_in]  storage dtype
    B: np.ndarray         # [rank][H_out] storage dtype


@dataclasses.dataclass
class Batch:
    """One lora_apply call's inputs."""
    name: str
    dtype: str
    H_in: int
    H_out: int
    seg_indptr: np.ndarray   # int32 [S+1]
    adapter_ids: np.ndarray  # int32 [S]; < 0 = no adapter
    x: np.ndarray            # [T][H_in]  storage
    y_in: np.ndarray         # [T][H_out] storage
    adapters: List[Adapter]  # adapters the batch may reference (loaded in this order)

    @property
    def T(self) -> int:
        return int(self.seg_indptr[-1])

    @property
    def S(self) -> int:
        return int(self.adapter_ids.shape[0])

    def adapter_by_id(self) -> Dict[int, Adapter]:
        return {a.id: a for a in self.adapters}


# --------------------------------------------------------------------------
# primitive draws
# --------------------------------------------------------------------------
def make_adapter(seed: int, tag: int, aid: int, rank: int, H_in: int, H_out: int, dtype: str,
                 scale: Optional[float] = None, zero_A: bool = False, zero_B: bool = False) -> Adapter:
    ra = _rng(seed, _TAG_A, tag, aid, rank)
    rb = _rng(seed, _TAG_B, tag, aid, rank)
    A = ra.standard_normal((rank, H_in), dtype=np.float32) * np.float32(1.0 / np.sqrt(H_in))
    B = rb.standard_normal((rank, H_out), dtype=np.float32) * np.float32(1.0 / np.sqrt(rank))
    if zero_A:
        A[:] = 0
    if zero_B:
        B[:] = 0
    s = float(np.float32(16.0 / rank)) if scale is None else float(np.float32(scale))
    return Adapter(aid, rank, s, f32_to_storage(A, dtype), f32_to_storage(B, dtype))


def make_rows(seed: int, tag: int, sub: int, T: int, H: int, dtype: str, zero: bool = False) -> np.ndarray:
    if zero:
        return f32_to_storage(np.zeros((T, H), np.float32), dtype)
    r = _rng(seed, tag, sub, T, H)
    return f32_to_storage(r.standard_normal((T, H), dtype=np.float32), dtype)


def segments_to_indptr(lengths: Sequence[int]) -> np.ndarray:
    ip = np.zeros(len(lengths) + 1, dtype=np.int64)
    ip[1:] = np.cumsum(np.asarray(lengths, dtype=np.int64))
    return ip.astype(np.int32)


def zipf_ids(rng: np.random.Generator, n_ids: int, n_draws: int, s: float = 1.0,
             perm: Optional[np.ndarray] = None) -> np.ndarray:
    """Zipf(s) popularity over a permutation of ids (SURVEY §8(c) reading 16)."""
    k = np.arange(1, n_ids + 1, dtype=np.float64)
    p = k ** (-s)
    p /= p.sum()
    ranks = rng.choice(n_ids, size=n_draws, p=p)
    if perm is None:
        perm = np.arange(n_ids)
    return perm[ranks].astype(np.int32)


def zipf_perm(seed: int, n_ids: int) -> np.ndarray:
    return _rng(seed, _TAG_BATCH, 99, n_ids).permutation(n_ids)


def build_batch(name: str, seed: int, dtype: str, H_in: int, H_out: int,
                lengths: Sequence[int], ids: Sequence[int], adapter_ranks: Dict[int, int],
                y_zero: bool = True, tag: int = 0, scales: Optional[Dict[int, float]] = None,
                zero_A_ids: Sequence[int] = (), zero_B_ids: Sequence[int] = ()) -> Batch:
    ip = segments_to_indptr(lengths)
    T = int(ip[-1])
    adapters = [make_adapter(seed, tag, aid, r, H_in, H_out, dtype,
                             scale=None if scales is None else scales.get(aid),
                             zero_A=aid in zero_A_ids, zero_B=aid in zero_B_ids)
                for aid, r in sorted(adapter_ranks.items())]
    x = make_rows(seed, _TAG_X, tag, T, H_in, dtype)
    y = make_rows(seed, _TAG_Y, tag, T, H_out, dtype, zero=y_zero)
    return Batch(name, dtype, H_in, H_out, ip, np.asarray(ids, dtype=np.int32), x, y, adapters)


# --------------------------------------------------------------------------
# the BASELINE.json configs (SURVEY.md §8(d) "Configs")
# --------------------------------------------------------------------------
def config_c1(y_zero: bool = True) -> Batch:
    """tiny fp32: 64->64, adapters 0..3 ranks {1,2,4,8}; 16 one-token segments
    (adapter i mod 4, order shuffled) + two 8-token segments on adapters 3 and 0."""
    seed = BASE_SEED + 0
    rng = _rng(seed, _TAG_BATCH)
    ids = [i % 4 for i in range(16)]
    rng.shuffle(ids)
    ids = list(ids) + [3, 0]
    lengths = [1] * 16 + [8, 8]
    return build_batch("c1", seed, "f32", 64, 64, lengths, ids, {0: 1, 1: 2, 2: 4, 3: 8}, y_zero=y_zero)


def config_c1_prefill_tiles(y_zero: bool = True, dtype: str = "bf16", H: int = 256) -> Batch:
    """Extra bf16 prefill tiles (not a BJ config): segment lengths {1,63,64,127,128,129,300},
    ranks {1,8,24,128} -- spans several 128-row tiles and ragged tails."""
    seed = BASE_SEED + 10
    lengths = [1, 63, 64, 127, 128, 129, 300]
    ranks = {0: 1, 1: 8, 2: 24, 3: 128}
    ids = [i % 4 for i in range(len(lengths))]
    return build_batch("c1p", seed, dtype, H, H, lengths, ids, ranks, y_zero=y_zero)


C2_RANKS = (8, 16, 32, 64)


def config_c2(y_zero: bool = True, tag: int = 0, zipf: bool = False, H: int = 4096,
              T: int = 64, n_adapters: int = 32) -> Batch:
    """Llama-2-7B q/k/v/o projection (4096->4096) bf16 decode: 64 one-token segments over
    32 adapters with ranks [8,16,32,64][a mod 4]; token t -> adapter t mod 32, shuffled."""
    seed = BASE_SEED + 1
    rng = _rng(seed, _TAG_BATCH, tag)
    if zipf:
        ids = zipf_ids(rng, n_adapters, T, 1.0, zipf_perm(seed, n_adapters))
    else:
        ids = np.array([t % n_adapters for t in range(T)], dtype=np.int32)
        rng.shuffle(ids)
    ranks = {a: C2_RANKS[a % 4] for a in range(n_adapters)}
    return build_batch("c2", seed, "bf16", H, H, [1] * T, ids, ranks, y_zero=y_zero, tag=tag)


C3_RANKS = (8, 16, 32, 64, 128)


def config_c3(y_zero: bool = True, n_seg: int = 32, seg_len: int = 512, H: int = 4096, tag: int = 0) -> Batch:
    """Llama-2-7B prefill: 32 requests x 512-token prompts, one distinct adapter each,
    rank [8,16,32,64,128][i mod 5] (the paper's synthetic workload)."""
    seed = BASE_SEED + 2
    ranks = {i: C3_RANKS[i % 5] for i in range(n_seg)}
    return build_batch("c3", seed, "bf16", H, H, [seg_len] * n_seg, list(range(n_seg)), ranks,
                       y_zero=y_zero, tag=tag)


C4_RANKS = (8, 16, 32, 64, 128)


def c4_rank(aid: int) -> int:
    return C4_RANKS[aid % 5]


def config_c4_draw(step: int, n_decode: int = 64, prefill_len: int = 512, n_adapters: int = 1000,
                   s: float = 1.0, world: int = 1, rank: int = 0, n_prefill: int = 1) -> Dict[str, np.ndarray]:
    """One iteration of config 4's trace: Zipf(s) adapter ids for the decode tokens and
    n_prefill prefill segments.  Returns ids only; adapters are generated on demand."""
    seed = BASE_SEED + 3
    rng = _rng(seed, _TAG_BATCH, step, world, rank)
    perm = zipf_perm(seed, n_adapters)
    dec = zipf_ids(rng, n_adapters, n_decode, s, perm)
    pre = zipf_ids(rng, n_adapters, n_prefill, s, perm)
    return {"decode_ids": dec, "prefill_id": pre, "prefill_len": np.int32(prefill_len)}


def c4_adapter(aid: int, H: int = 5120, dtype: str = "bf16", tag: int = 0) -> Adapter:
    return make_adapter(BASE_SEED + 3, tag, aid, c4_rank(aid), H, H, dtype)


C5_SHAPES = {"q": (8192, 8192), "k": (8192, 1024), "v": (8192, 1024), "o": (8192, 8192),
             "gate": (8192, 28672), "up": (8192, 28672), "down": (28672, 8192)}
C5_RANKS = (16, 32, 64, 128)


def config_c5(proj: str, y_zero: bool = True, prefill: bool = False, n_adapters: int = 32) -> Batch:
    """Llama-2-70B per-layer projection shapes; ranks [16,32,64,128][a mod 4];
    decode: 64 one-token segments, prefill: 8 x 512."""
    seed = BASE_SEED + 4
    H_in, H_out = C5_SHAPES[proj]
    tag = list(C5_SHAPES).index(proj)
    rng = _rng(seed, _TAG_BATCH, tag, int(prefill))
    if prefill:
        lengths, ids = [512] * 8, list(range(8))
    else:
        ids = np.array([t % n_adapters for t in range(64)], dtype=np.int32)
        rng.shuffle(ids)
        lengths = [1] * 64
    used = sorted(set(int(i) for i in ids))
    ranks = {a: C5_RANKS[a % 4] for a in used}
    return build_batch("c5_" + proj, seed, "bf16", H_in, H_out, lengths, ids, ranks, y_zero=y_zero, tag=tag)


def random_batch(seed: int, dtype: str, H_in: int, H_out: int, max_seg: int = 16, max_rank: int = 16,
                 max_len: int = 4, n_adapters: int = 6, p_none: float = 0.1, y_zero: bool = False,
                 allow_empty: bool = True) -> Batch:
    """Randomised batch for the SPEC acceptance-3 style sweep."""
    rng = _rng(seed, _TAG_BATCH, 7)
    S = int(rng.integers(1, max_seg + 1))
    lo = 0 if allow_empty else 1
    lengths = [int(rng.integers(lo, max_len + 1)) for _ in range(S)]
    n_ad = int(rng.integers(1, n_adapters + 1))
    ranks = {a: int(rng.integers(1, max_rank + 1)) for a in range(n_ad)}
    ids = [int(rng.integers(0, n_ad)) if rng.random() >= p_none else -1 for _ in range(S)]
    return build_batch("rand%d" % seed, seed, dtype, H_in, H_out, lengths, ids, ranks, y_zero=y_zero, tag=seed)
