"""Multi-process (world size 2, gloo, CPU) coverage of the tensor-parallel decomposition and
of the request-partitioned data-parallel placement.  The arithmetic here is the
fp64 oracle; what is tested is the sharding (which slice of A/B/x/y each rank owns), the SUM
all-reduce of the rank-r intermediate, and that the re-assembled result equals the unsharded
oracle -- the same decomposition paper_2401_11240_b200.tp runs with the CUDA kernels + NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2401_11240_b200.tp import shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(seed=5, H_in=64, H_out=48):
    rng = np.random.default_rng(seed)
    lens = [1, 1, 3, 1, 5, 2]
    ip = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = np.array([0, 1, 2, 1, 0, -1], np.int32)
    ads = [(a, r, s, rng.standard_normal((r, H_in)), rng.standard_normal((r, H_out)))
           for a, r, s in ((0, 3, 0.5), (1, 8, 2.0), (2, 1, 1.0))]
    T = int(ip[-1])
    return H_in, H_out, ip, ids, ads, rng.standard_normal((T, H_in)), rng.standard_normal((T, H_out))


def _tp_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H_in, H_out, ip, ids, ads, x, y0 = _problem()
    lo, hi = shard_bounds(H_in, world, rank)
    olo, ohi = shard_bounds(H_out, world, rank)
    # partial v over this rank's H_in slice (the oracle's v = s * x A)
    sh = [(a, r, s, A[:, lo:hi], B) for (a, r, s, A, B) in ads]
    _, v = O.delta(hi - lo, H_out, ip, ids, sh, x[:, lo:hi], np.zeros_like(y0), want_v=True)
    vt = torch.from_numpy(v.copy())
    dist.all_reduce(vt, op=dist.ReduceOp.SUM)          # the rank-r all-reduce
    v = vt.numpy()
    tab = {a[0]: a for a in ads}
    y = y0[:, olo:ohi].copy()
    for i in range(len(ids)):
        if ids[i] < 0:
            continue
        _, r, s, A, B = tab[int(ids[i])]
        for t in range(ip[i], ip[i + 1]):
            y[t] += v[t, :r] @ B[:, olo:ohi]
    parts = [torch.zeros_like(torch.from_numpy(y)) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(y))
    if rank == 0:
        out.put(np.concatenate([p.numpy() for p in parts], axis=1))
    dist.destroy_process_group()


def test_tp_decomposition_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    y_tp = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    H_in, H_out, ip, ids, ads, x, y0 = _problem()
    ref = O.delta(H_in, H_out, ip, ids, ads, x, y0)
    assert np.allclose(y_tp, ref, rtol=1e-12, atol=1e-12)


def _dp_worker(rank, world, port, out):
    """Request-partitioned data parallelism: every rank routes the same global step (64 decode requests
    + 1 prompt per GPU) with Algorithm 1 (serving.route_requests) and keeps its share; no data-path
    collective -- the gathers below only check the partition."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from workloads import gen
    from paper_2401_11240_b200 import scheduler as S
    from paper_2401_11240_b200.serving import home_gpu, route_requests
    hot = [int(v) for v in gen.zipf_perm(gen.BASE_SEED + 3, 1000)[:16]]
    d = gen.config_c4_draw(step=3, n_decode=64 * world, n_prefill=world)
    dec, pre = [int(a) for a in d["decode_ids"]], [int(a) for a in d["prefill_id"]]
    dec_to, pre_to = route_requests(dec, pre, 512, world, hot, S.measured_model("mbgmv", 1), gen.c4_rank)
    mine = [i for i, g in enumerate(dec_to + pre_to) if g == rank]
    ok = all(home_gpu(a, world, hot) in (None, rank) for i, a in enumerate(dec + pre) if i in set(mine))
    t = torch.zeros(len(dec) + len(pre), dtype=torch.int64)
    t[mine] = 1
    dist.all_reduce(t)                       # how many ranks served each request
    flag = torch.tensor([int(ok)], dtype=torch.int64)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        out.put((t.tolist(), int(flag.item())))
    dist.destroy_process_group()


def test_request_partition_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    served, hosted_ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert served == [1] * (64 * 2 + 2)     # every request served exactly once
    assert hosted_ok == 1                    # and only by a GPU hosting its adapter
