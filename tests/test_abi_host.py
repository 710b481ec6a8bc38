"""CPU tests of the C-ABI library: it loads, exports every symbol the header declares,
and its host logic (page allocator, canonical metadata M1-M6, validation, byte
accounting) matches the oracle bit for bit.  Host-only pools make no CUDA calls."""
import ctypes

import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

import paper_2401_11240_b200 as L
from paper_2401_11240_b200 import binding as B


def test_library_exports_every_header_symbol():
    names = L.header_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L.LIB, n), n
        assert ctypes.cast(getattr(L.LIB, n), ctypes.c_void_p).value
    assert L.LIB.lora_abi_version() == 2


def _compare_md(md, ref):
    for k in ("T", "S", "G", "L_tc", "n_seg", "max_rank", "nseg_x_maxrank", "sum_rank_seg", "sum_rank_groups",
              "sum_rank_tokens"):
        assert md[k] == ref[k], k
    for k in ("tok_seg", "group_id", "group_rank", "group_ntok", "group_page_off", "group_tok_off",
              "group_tokens", "pages", "seg_kind"):
        assert np.array_equal(md[k], ref[k]), k
    assert np.array_equal(md["group_scale"].view(np.uint32), ref["group_scale"].view(np.uint32))


def test_allocator_and_metadata_match_oracle_replay_random():
    rng = np.random.default_rng(2024)
    for trial in range(40):
        n_pages = int(rng.integers(8, 200))
        max_ad = int(rng.integers(1, 12))
        pool = L.LoraPool(64, 32, max_ad, "bf16", max_total_rank=n_pages, host_only=True)
        ref = O.PageAllocatorReplay(n_pages, max_ad)
        for step in range(60):
            if rng.random() < 0.6 or not ref.table:
                aid, r = int(rng.integers(0, 20)), int(rng.integers(1, 33))
                s = float(np.float32(rng.choice([1.0, 0.5, 16.0 / r, 0.3])))
                try:
                    ref.load(aid, r, s)
                    exp = None
                except KeyError:
                    exp = "LORA_ERR_EXISTS"
                except O.PoolFull:
                    exp = "LORA_ERR_POOL_FULL"
                if exp is None:
                    pool.load_adapter(aid, r, None, None, s)
                    assert pool.adapter_pages(aid) == ref.pages_of(aid)
                else:
                    with pytest.raises(L.LoraError) as ei:
                        pool.load_adapter(aid, r, None, None, s)
                    assert ei.value.name == exp
            else:
                aid = int(rng.choice(list(ref.table)))
                ref.unload(aid)
                pool.unload_adapter(aid)
            info = pool.info()
            assert info["free_pages"] == sum(ref.free)
            assert info["resident_adapters"] == len(ref.table)
            # a random batch over the resident adapters (+ an unloaded id sometimes)
            if ref.table and rng.random() < 0.3:
                S = int(rng.integers(0, 12))
                lens = rng.integers(0, 90, size=S)
                ip = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
                ids = np.array([int(rng.choice(list(ref.table))) if rng.random() > 0.2 else -1 for _ in range(S)],
                               np.int32)
                Ltc = int(rng.choice([1, 16, 64, 1000]))
                pool.set_option(B.LORA_OPT_TC_THRESHOLD, Ltc)
                pool.plan(ip, ids)
                _compare_md(pool.metadata(), O.canonical_metadata(ip, ids, ref.table, Ltc))
        pool.close()


def test_metadata_for_baseline_configs():
    for b in (gen.config_c1(), gen.config_c2(), gen.config_c3(n_seg=8, seg_len=64, H=256), gen.config_c1_prefill_tiles()):
        pool = L.LoraPool(b.H_in, b.H_out, 64, b.dtype, max_total_rank=4096, host_only=True)
        ref = O.PageAllocatorReplay(4096, 64)
        for a in b.adapters:
            pool.load_adapter(a.id, a.rank, None, None, a.scale)
            ref.load(a.id, a.rank, a.scale)
        pool.plan(b.seg_indptr, b.adapter_ids)
        _compare_md(pool.metadata(), O.canonical_metadata(b.seg_indptr, b.adapter_ids, ref.table, 64))
        pool.close()


def test_validation_errors():
    pool = L.LoraPool(64, 64, 4, "f32", max_total_rank=32, host_only=True)
    pool.load_adapter(1, 4, None, None, 1.0)
    cases = [
        (lambda: pool.plan([0, 2, 1], [1, 1]), "LORA_ERR_ARG"),          # decreasing indptr
        (lambda: pool.plan([1, 2], [1]), "LORA_ERR_ARG"),                # indptr[0] != 0
        (lambda: pool.plan([0, 2], [7]), "LORA_ERR_UNKNOWN_ADAPTER"),
        (lambda: pool.load_adapter(2, 0, None, None, 1.0), "LORA_ERR_SHAPE"),
        (lambda: pool.load_adapter(2, 65, None, None, 1.0), "LORA_ERR_SHAPE"),
        (lambda: pool.load_adapter(-3, 1, None, None, 1.0), "LORA_ERR_ARG"),
        (lambda: pool.load_adapter(1, 1, None, None, 1.0), "LORA_ERR_EXISTS"),
        (lambda: pool.load_adapter(2, 29, None, None, 1.0), "LORA_ERR_POOL_FULL"),
        (lambda: pool.unload_adapter(9), "LORA_ERR_UNKNOWN_ADAPTER"),
        (lambda: pool.apply(0, 0, [0, 1], [1], stream=0), "LORA_ERR_UNSUPPORTED"),
        (lambda: pool.set_option(B.LORA_OPT_TC_THRESHOLD, 0), "LORA_ERR_ARG"),
    ]
    for fn, name in cases:
        with pytest.raises(L.LoraError) as ei:
            fn()
        assert ei.value.name == name, (name, str(ei.value))
        assert str(ei.value)
    # failed calls have no side effects
    assert pool.info()["free_pages"] == 28 and pool.info()["resident_adapters"] == 1
    with pytest.raises(L.LoraError) as ei:
        L.LoraPool(60, 64, 4, "bf16", host_only=True)      # 60 % 8 != 0
    assert ei.value.name == "LORA_ERR_ALIGN"
    with pytest.raises(L.LoraError) as ei:
        L.LoraPool(0, 64, 4, "bf16", host_only=True)
    assert ei.value.name == "LORA_ERR_SHAPE"
    # empty batch is a no-op plan
    pool.plan([0], [])
    assert pool.metadata()["T"] == 0
    pool.close()


def test_p11_resident_bytes_closed_form():
    """P11 (tests/golden/p11_adapter_bytes.txt): rank-64 adapters on W_Q,
    W_K, W_V of 32 Llama2-7B layers occupy exactly 100,663,296 B (96 MiB) of 16-bit pools."""
    total = 0
    for _layer in range(32):
        for _proj in "qkv":
            pool = L.LoraPool(4096, 4096, 1, "bf16", max_total_rank=64, host_only=True)
            pool.load_adapter(0, 64, None, None, 0.25)
            info = pool.info()
            assert info["pool_bytes"] == info["resident_bytes"]
            total += info["resident_bytes"]
            pool.close()
    assert total == 100663296


def test_device_pool_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(L.LoraError) as ei:
        L.LoraPool(64, 64, 2, "bf16")
    assert ei.value.name == "LORA_ERR_CUDA"


def test_pad_max_rank_keeps_metadata_and_pads_work():
    """LORA_OPT_PAD_MAX_RANK (BGMV comparison mode): canonical metadata is unchanged,
    the decode work lists grow to the batch's max rank for every group (units per group of the
    max rank)."""
    b = gen.config_c2()
    pools = []
    for pad in (0, 1):
        pool = L.LoraPool(b.H_in, b.H_out, 40, "bf16", max_total_rank=sum(a.rank for a in b.adapters), host_only=True)
        pool.set_option(B.LORA_OPT_PAD_MAX_RANK, pad)
        for a in b.adapters:
            pool.load_adapter(a.id, a.rank, None, None, a.scale)
        pool.plan(b.seg_indptr, b.adapter_ids)
        pools.append(pool.metadata())
        pool.close()
    plain, padded = pools
    _compare_md(padded, plain)
    # c2: ranks 8/16/32/64 -> every group padded to 64: shrink units = ksplit x 64/16 per gc
    n_gc = len(set(b.adapter_ids.tolist()))
    assert padded["n_shrink_units"] % (n_gc * (64 // 16)) == 0
    assert padded["n_shrink_units"] > plain["n_shrink_units"]
    assert padded["n_expand_units"] > plain["n_expand_units"]


def _mma_unit_smem(r, nc, ntok):
    # bf16 expand CTA layout (kernel_config.h expand_mma_smem): header + v tiles | B rows | y rows |
    # fp32 D^T | pages
    rp = (r + 15) & ~15
    boff = (320 + ((ntok + 3) >> 2) * 8 * (rp + 8) * 2 + 127) & ~127
    pitch = nc * 2 + 16
    return boff + r * pitch + ntok * pitch + ntok * (nc + 4) * 4 + r * 4


def _pow2_units(r, H):
    c = 1
    while c * 2 <= 32768 // (r * 2):
        c *= 2
    c = min(c, 1024)
    return -(-H // c), c


def test_expand_unit_sizing_rule():
    """Decode expand units (DESIGN.md §6 N1): a single-pool batch whose power-of-two 32 KB units fit
    one wave keeps them; a bigger one switches to the widest multiple-of-16 units of <= 56 KB each,
    so the expand grid stays within 4 CTAs per SM."""
    b = gen.config_c2()
    pool = L.LoraPool(b.H_in, b.H_out, 40, "bf16", max_total_rank=sum(a.rank for a in b.adapters), host_only=True)
    for a in b.adapters:
        pool.load_adapter(a.id, a.rank, None, None, a.scale)
    pool.plan(b.seg_indptr, b.adapter_ids)
    md = pool.metadata()
    pool.close()
    ranks = {a.id: a.rank for a in b.adapters}
    want = sum(_pow2_units(ranks[i], b.H_out)[0] for i in sorted(set(b.adapter_ids.tolist())))
    assert md["n_expand_units"] == want == 256

    # 256 adapters x 2 tokens: power-of-two units would need 2048 CTAs (> 3 x 148)
    n_ad, H = 256, 4096
    rk = [8, 16, 32, 64]
    pool = L.LoraPool(H, H, n_ad, "bf16", max_total_rank=sum(rk[i % 4] for i in range(n_ad)), host_only=True)
    for i in range(n_ad):
        pool.load_adapter(i, rk[i % 4], None, None, 1.0)
    ids = np.repeat(np.arange(n_ad, dtype=np.int32), 2)
    ip = np.arange(len(ids) + 1, dtype=np.int32)
    pool.plan(ip, ids)
    md = pool.metadata()
    pool.close()
    units = 0
    for i in range(n_ad):
        r = rk[i % 4]
        nu = (H + 2047) // 2048
        while True:
            nc = ((H + nu - 1) // nu + 15) & ~15
            if nc <= 16 or _mma_unit_smem(r, nc, 2) <= 56 * 1024:
                break
            nu += 1
        assert _mma_unit_smem(r, nc, 2) <= 56 * 1024 and nc % 16 == 0
        units += -(-H // nc)
    assert md["n_expand_units"] == units
    assert units < sum(_pow2_units(rk[i % 4], H)[0] for i in range(n_ad))
