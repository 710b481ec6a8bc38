"""GPU parity of the pipelined decode schedule (LORA_OPT_DECODE_CHUNK_KB, decode_kernel.cu
launch_pair): shrink(0) | expand(0) + shrink(1) | ... | expand(n-1) over chunks of group-chunks.

Same kernels bodies, same arithmetic order, so every test checks the chunked schedule BITWISE
against the one-shrink-grid / one-expand-grid schedule (chunk 0) on the same pool and inputs, and
within BASELINE.json's tolerance against the fp64 oracle (SURVEY.md §8(c) GPU parity matrix): c2,
c2-Zipf, c5 70B shapes (incl. H_out = 1024 and H_in = 28672), ragged H, ranks 1..256 with
multi-token adapters (token chunks of 8), id < 0 rows, the fused q/k/v call (chunks across pools),
CUDA-graph replay of a dependent chain, and a batch whose metadata takes the device-upload path."""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

from gpu_util import TOL, from_torch, make_pool, rel_l2, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2401_11240_b200 as lib
    return lib


def _apply(L, pool, b, chunk, y_in=None, seg_indptr=None, adapter_ids=None):
    import torch
    from paper_2401_11240_b200 import binding as B
    pool.set_option(B.LORA_OPT_DECODE_CHUNK_KB, ck)
    x = to_torch(b.x, "cuda")
    y = to_torch(b.y_in if y_in is None else y_in, "cuda")
    pool.apply(x, y, b.seg_indptr if seg_indptr is None else seg_indptr,
               b.adapter_ids if adapter_ids is None else adapter_ids)
    torch.cuda.synchronize()
    return y


def _check(L, b, chunks=(256,), oracle=True):
    pool = make_pool(b, L)
    y_one = _apply(L, pool, b, 0)
    for ck in chunks:
        y_chunk = _apply(L, pool, b, ck)
        assert np.array_equal(from_torch(y_chunk, "bf16"), from_torch(y_one, "bf16")), ck
    pool.close()
    if oracle:
        ref = O.delta_for_batch(b, n_threads=8)
        assert rel_l2(from_torch(y_one, "bf16"), ref, "bf16") <= TOL["bf16"]


@pytest.mark.parametrize("y_zero", [True, False], ids=["runA_delta", "runB_accumulate"])
def test_chunked_c2(L, y_zero):
    _check(L, gen.config_c2(y_zero=y_zero), chunks=(64, 1024, 4096, 8192, 1 << 20))


def test_chunked_c2_zipf(L):
    _check(L, gen.config_c2(zipf=True, y_zero=False))


@pytest.mark.parametrize("proj", ["k", "q", "gate", "down"])
def test_chunked_c5_shapes(L, proj):
    _check(L, gen.config_c5(proj, y_zero=False), oracle=proj in ("k", "down"))


@pytest.mark.parametrize("H_in,H_out", [(1000, 1000), (2056, 3080), (64, 4104), (5120, 5120)])
def test_chunked_ragged_hidden(L, H_in, H_out):
    rng = np.random.default_rng(H_in * 7 + H_out)
    lengths = [int(v) for v in rng.integers(1, 12, size=20)]
    ranks = {a: int(v) for a, v in enumerate(rng.choice([1, 3, 8, 17, 24, 40, 64, 100, 128], size=10))}
    ranks = {a: min(r, H_in, H_out) for a, r in ranks.items()}
    ids = [int(v) for v in rng.integers(-1, 10, size=20)]
    b = gen.build_batch("rr", 4242 + H_in, "bf16", H_in, H_out, lengths, ids, ranks, y_zero=False)
    _check(L, b, chunks=(16, 512))


def test_chunked_ranks_to_256_multi_token(L):
    # decode segments up to 63 tokens (L_tc = 64): adapters with several 8-token chunks, ranks to 256
    rng = np.random.default_rng(5)
    lengths = [int(v) for v in rng.integers(1, 40, size=12)]
    ranks = {0: 256, 1: 255, 2: 129, 3: 1, 4: 16, 5: 200}
    ids = [int(v) for v in rng.integers(-1, 6, size=12)]
    b = gen.build_batch("r256", 777, "bf16", 2048, 1536, lengths, ids, ranks, y_zero=False)
    _check(L, b)


def test_chunked_random_sweep(L):
    rng = np.random.default_rng(99)
    for trial in range(40):
        H_in = int(rng.integers(1, 40)) * 8 * int(rng.choice([1, 16]))
        H_out = int(rng.integers(1, 40)) * 8 * int(rng.choice([1, 16]))
        b = gen.random_batch(5000 + trial, "bf16", H_in, H_out, max_seg=64, max_rank=min(128, H_in, H_out),
                             max_len=int(rng.choice([1, 4, 40])), n_adapters=8, y_zero=bool(trial % 2))
        if b.T == 0:
            continue
        _check(L, b, chunks=(int(rng.choice([4, 64, 1024])),), oracle=trial % 4 == 0)


def test_chunked_multi_qkv_equals_pair(L):
    import torch
    from paper_2401_11240_b200 import binding as B
    shapes = [(4096, 4096), (4096, 1024), (4096, 1024)]
    batches = []
    ids = list(gen.config_c2().adapter_ids)   # one batch layout for the three pools
    for i, (hin, hout) in enumerate(shapes):
        b = gen.build_batch("mq%d" % i, 910 + i, "bf16", hin, hout, [1] * 64, ids,
                            {a: gen.C2_RANKS[a % 4] for a in range(32)}, y_zero=False)
        batches.append(b)
    for b in batches[1:]:
        b.x = batches[0].x.copy()
    pools = [make_pool(b, L) for b in batches]
    xs = [to_torch(b.x, "cuda") for b in batches]
    outs = {}
    for ck in (0, 8192, 3000):
        for p in pools:
            p.set_option(B.LORA_OPT_DECODE_CHUNK_KB, ck)
        ys = [to_torch(b.y_in, "cuda") for b in batches]
        L.apply_multi(pools, xs, ys, batches[0].seg_indptr, batches[0].adapter_ids)
        torch.cuda.synchronize()
        outs[ck] = ys
    for b, y0, y1, y2 in zip(batches, outs[0], outs[8192], outs[3000]):
        assert torch.equal(y0, y1) and torch.equal(y0, y2)
        ref = O.delta_for_batch(b, n_threads=8)
        assert rel_l2(from_torch(y1, "bf16"), ref, "bf16") <= TOL["bf16"]
    for p in pools:
        p.close()


def test_chunked_graph_replay_and_chain(L):
    """A CUDA graph of 6 dependent chunked applies (each apply's x = the previous apply's y) replays
    bitwise equal to the same chain issued eagerly unchunked."""
    import torch
    from paper_2401_11240_b200 import binding as B
    b = gen.config_c2(y_zero=False)
    pool = make_pool(b, L)
    x0 = to_torch(b.x, "cuda")

    def chain(ck, graph):
        pool.set_option(B.LORA_OPT_DECODE_CHUNK_KB, ck)
        bufs = [x0.clone()] + [to_torch(b.y_in, "cuda") for _ in range(6)]
        st = torch.cuda.Stream()
        def run():
            for i in range(6):
                pool.apply(bufs[i], bufs[i + 1], b.seg_indptr, b.adapter_ids, stream=st)
        if graph:
            run()   # warm-up outside the capture (scratch sizing)
            torch.cuda.synchronize()
            for i in range(1, 7):
                bufs[i].copy_(to_torch(b.y_in, "cuda"))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                run()
            for i in range(1, 7):
                bufs[i].copy_(to_torch(b.y_in, "cuda"))
            torch.cuda.synchronize()
            g.replay()
        else:
            with torch.cuda.stream(st):
                run()
        torch.cuda.synchronize()
        return bufs[6].clone()

    ref = chain(0, False)
    assert torch.equal(chain(2048, True), ref)
    assert torch.equal(chain(2048, False), ref)
    pool.close()


def test_chunked_huge_batch_metadata_upload(L):
    # 512 tokens over 256 adapters: the metadata exceeds the kernel parameters (device upload path)
    ranks = {a: [8, 16, 32, 64][a % 4] for a in range(256)}
    ids = [a % 256 for a in range(512)]
    b = gen.build_batch("huge", 31337, "bf16", 1024, 1024, [1] * 512, ids, ranks, y_zero=False)
    _check(L, b, chunks=(1024,))
