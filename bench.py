#!/usr/bin/env python
"""Benchmark of the batched multi-adapter LoRA delta (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1], "c2"): Llama-2-7B q/k/v/o projections (4096->4096,
bf16), decode batch of 64 tokens over 32 adapters with ranks [8,16,32,64][a mod 4], for
every one of the model's 32 layers: one STEP = one decode iteration's LoRA delta over all
32 layers x 4 projections = 128 lora_apply calls, each on its own paged pool (distinct
adapter weights per layer and projection, as in real serving).  The working set
(128 pools x 15.7 MB of adapter rows + x/y) is 2.2 GB >> the 126 MB L2, so no L2 flush
is needed between steps ("inputs larger than L2").

Per layer the step issues one lora_apply_multi for q/k/v (they share x and are independent) and
one lora_apply for o (its input is the attention output); --qkv-mode serial issues 4 applies.

value   tokens/s = (64 tokens x ranks) / step time, device-timed with CUDA events around K
        replays of a CUDA graph of one step (inputs resident in HBM), max over ranks.
e2e     the same metric through the public API (LoraPool.apply / lora_apply_multi) with host
        buffers: every step copies that step's x (pinned host -> device), runs the applies
        eagerly and reads all y back (device -> pinned host), pipelined in 4 layer chunks on two
        copy streams.
roofline  the decode kernel (the only kernel in the step): algorithmic bytes per launch
        (adapter rows once + x once + y read and write) / average launch time.
cpu_baseline  the fp64 oracle (oracle/, C, OpenMP over tokens) on a bounded sample.

Multi-GPU (torchrun): weak scaling, each rank serves its own 64-token batch over its own
pools (request partitioning, no data-path collective; the process group is only used for
the barrier and the max-over-ranks timing).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import gen  # noqa: E402

LAYERS = 32
PROJS = ("q", "k", "v", "o")
T_DECODE = 64
H = 4096
METRIC = "LoRA-delta tokens/s + % HBM roofline (decode) / % TC peak (prefill), 1/2/4/8 B200"
UNIT = "tokens/s"
WORKLOAD = "c2: Llama-2-7B q/k/v/o (4096->4096) bf16 decode, 64 tokens over 32 adapters, ranks 8/16/32/64, x 32 layers"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--layers", type=int, default=LAYERS)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-layers", type=int, default=2)
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--prefill-layers", type=int, default=2,
                    help="layers of the c3 prefill measurement reported in the 'prefill' object (0 = skip)")
    ap.add_argument("--prefill-steps", type=int, default=20)
    ap.add_argument("--qkv-mode", choices=["serial", "fused", "streams"], default="fused",
                    help="q/k/v (same x, independent deltas; the paper adapts W_Q/W_K/W_V together, P:875): one "
                         "lora_apply_multi (default), one lora_apply each in stream order, or forked onto 3 streams; "
                         "o (input = attention output) is always its own lora_apply")
    ap.add_argument("--min-window-ms", type=float, default=200.0,
                    help="repeat the K-step timed window until this much device time is covered (median reported)")
    ap.add_argument("--c4-steps", type=int, default=40, help="config 4 (Zipf paged pool, cold starts) steps; 0 = skip")
    ap.add_argument("--cold-start", type=int, choices=[0, 1], default=1,
                    help="cold-start latency by rank + the paper's CPU-assist comparison (rank 0)")
    ap.add_argument("--c5-reps", type=int, default=5, help="config 5 (70B shapes, tp 1/2/4/8 shards) timing reps; 0 = skip")
    ap.add_argument("--fused-base-reps", type=int, default=5,
                    help="NEXT f2 (delta fused into the base GEMM) timing reps on c3 shapes; 0 = skip")
    return ap.parse_args()


# ---------------------------------------------------------------- distributed plumbing
# test-only: LORA_BENCH_SHARE_GPU=1 runs every rank on cuda:0 with gloo plumbing, so the N > 1
# control flow (barriers, max over ranks, rank-0 line, request partitioning) can be exercised on a
# one-GPU box (NCCL refuses two ranks on one device).  Never used for reported numbers.
SHARE_GPU = os.environ.get("LORA_BENCH_SHARE_GPU") == "1"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if SHARE_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, local):
    import torch
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if SHARE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world > 1


def max_over_ranks(v: float, use_dist: bool) -> float:
    if not use_dist:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if SHARE_GPU else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(use_dist):
    import torch
    if use_dist:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


# ---------------------------------------------------------------- clocks sampler
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,clocks.mem")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons, mem, pw = [], 0.0, set(), [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for lst, v in ((pw, parts[2]), (mem, parts[7] if len(parts) > 7 else "")):
                try:
                    lst.append(float(v))
                except ValueError:
                    pass
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "mem_mhz": float(np.median(mem)) if mem else None, "power_w": float(np.median(pw)) if pw else None}


# ---------------------------------------------------------------- workload
def layer_batch_meta(rank: int):
    """seg_indptr / adapter_ids of the c2 decode batch (same for every layer and projection:
    a decode request keeps its adapter across layers)."""
    b = gen.config_c2(tag=0)
    return b.seg_indptr, b.adapter_ids


def make_pool_adapters(layer: int, proj: int, world_rank: int):
    """The 32 adapters of one (layer, projection) pool, generated by workloads.gen with a
    distinct seed tag per (rank, layer, projection)."""
    tag = 1 + ((world_rank * LAYERS + layer) * len(PROJS) + proj)
    return [gen.make_adapter(gen.BASE_SEED + 1, tag, a, gen.C2_RANKS[a % 4], H, H, "bf16") for a in range(32)]


def algorithmic_bytes_per_apply(ranks_sum: int, T: int) -> int:
    """b·[Σ_G r·(H_in+H_out) + T·H_in + 2·T·H_out]."""
    return 2 * (ranks_sum * (H + H) + T * H + 2 * T * H)


def load_ncu_traffic(key="dram_bytes_per_launch"):
    """DRAM bytes per launch from the committed ncu --set full summary (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get(key)
    except Exception:
        return None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- CPU oracle baseline
def _oracle_work(n_layers_sample: int, world_rank: int = 0):
    """Inputs of the fp64 oracle for n_layers_sample layers x 4 projections of the bench workload."""
    ip, ids = layer_batch_meta(world_rank)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((T_DECODE, H))
    x = gen.storage_to_f64(gen.f32_to_bf16_bits(x.astype(np.float32)), "bf16")
    work = []
    for l in range(n_layers_sample):
        for p in range(len(PROJS)):
            ads = make_pool_adapters(l, p, world_rank)
            work.append([(a.id, a.rank, a.scale, gen.storage_to_f64(a.A, "bf16"), gen.storage_to_f64(a.B, "bf16"))
                         for a in ads])
    return ip, ids, x, np.zeros((T_DECODE, H)), work


def _oracle_run(w, n_threads: int) -> float:
    """seconds for one pass of the oracle over the work of _oracle_work"""
    from oracle import oracle as O
    ip, ids, x, y0, work = w
    t0 = time.perf_counter()
    for ads in work:
        O.delta(H, H, ip, ids, ads, x, y0, n_threads=n_threads)
    return time.perf_counter() - t0


def cpu_oracle_tokens_per_s(n_layers_sample: int, world_rank: int = 0, n_threads: int = 0, reps: int = 1):
    """The fp64 oracle on n_layers_sample layers x 4 projections of the same workload,
    extrapolated to the metric's unit (tokens through all 32 layers x 4 projections)."""
    n_threads = n_threads or len(os.sched_getaffinity(0))
    w = _oracle_work(n_layers_sample, world_rank)
    dt = sum(_oracle_run(w, n_threads) for _ in range(reps))
    frac = (n_layers_sample * reps) / LAYERS
    return T_DECODE * frac / dt, n_threads, dt


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the oracle (fp64 C, OpenMP on every host core) as the reference arm, same
    metric, workload and unit.  Each of the --steps K timed steps (after --warmup W untimed ones) is a
    bounded sample of one bench step: the oracle over 1 of the 32 layers (q/k/v/o, 64 tokens), the
    step time extrapolated x32 (layers are identical work)."""
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    n_threads = len(os.sched_getaffinity(0))
    w = _oracle_work(1, 0)
    for _ in range(args.warmup):
        _oracle_run(w, n_threads)
    dts = [_oracle_run(w, n_threads) for _ in range(args.steps)]
    step_s = float(np.median(dts)) * LAYERS
    v = T_DECODE / step_s
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": len(dts), "warmup": args.warmup, "ms_per_step": 1000.0 * step_s,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (workloads.gen, seeded)",
            "config": {"workload": WORKLOAD, "layers": LAYERS, "tokens_per_step": T_DECODE, "adapters": 32,
                       "parallelism": "dp%d" % world},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": n_threads, "kind": "oracle", "cpu_model": _cpu_model(),
                             "sample": "per step: 1 of 32 layers (4 applies x 64 tokens), median of %d steps, "
                                       "extrapolated x32; %.1f s of CPU work" % (len(dts), sum(dts))},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- prefill (config 3) measurement
def bench_prefill(L, layers: int, steps: int, dev, hbm_peak: float, tc_peak: float, world_rank: int = 0):
    """c3: 32 requests x 512-token prompts over 32 adapters (ranks 8..128), 4096->4096 bf16, per
    layer q/k/v/o on distinct pools; x/y (256 MB per layer) >> L2.  Returns the 'prefill' object."""
    import torch
    T, n_seg, seg_len = 32 * 512, 32, 512
    ranks = {i: gen.C3_RANKS[i % 5] for i in range(n_seg)}
    ip = gen.segments_to_indptr([seg_len] * n_seg)
    ids = np.arange(n_seg, dtype=np.int32)
    pools = []
    with cf.ThreadPoolExecutor(max_workers=min(16, len(os.sched_getaffinity(0)))) as ex:
        futs = [ex.submit(lambda lp: [gen.make_adapter(gen.BASE_SEED + 2, 1000 + lp + 10000 * world_rank, a, ranks[a],
                                                       H, H, "bf16") for a in range(n_seg)], lp)
                for lp in range(layers * len(PROJS))]
        for f in futs:
            ads = f.result()
            pool = L.LoraPool(H, H, n_seg, "bf16", max_total_rank=sum(a.rank for a in ads))
            for a in ads:
                pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                                  torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
            pools.append(pool)
    torch.cuda.synchronize()
    for pool in pools:
        pool.release_host_buffers()
    g = torch.Generator(device="cpu").manual_seed(gen.BASE_SEED + 200 + world_rank)
    xs = [torch.randn(T, H, generator=g).to(torch.bfloat16).to(dev) for _ in range(2)]
    ys = [torch.zeros(T, H, dtype=torch.bfloat16, device=dev) for _ in pools]
    st = torch.cuda.Stream(device=dev)

    def step():
        for i, (pool, y) in enumerate(zip(pools, ys)):
            pool.apply(xs[0 if i % 4 < 3 else 1], y, ip, ids, stream=st)

    with torch.cuda.stream(st):
        step()
    torch.cuda.synchronize()
    md = pools[0].metadata()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        step()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        for _ in range(steps):
            graph.replay()
    e1.record(st)
    torch.cuda.synchronize()
    ms_apply = e0.elapsed_time(e1) / steps / len(pools)
    sum_r = sum(ranks.values())
    bytes_apply = 2 * (sum_r * 2 * H + T * H + 2 * T * H)
    flops_apply = sum(2 * ranks[i] * seg_len * 2 * H for i in range(n_seg))
    gbs = bytes_apply / (ms_apply * 1e-3) / 1e9
    tfs = flops_apply / (ms_apply * 1e-3) / 1e12
    out = {"workload": "c3: Llama-2-7B prefill 32 x 512 tokens, 32 adapters ranks 8..128, 4096->4096 bf16, "
                       "%d layers x q/k/v/o" % layers,
           "value": round(T / (ms_apply * 1e-3), 1), "unit": "tokens/s per projection apply",
           "ms_per_apply": round(ms_apply, 5), "tensor_core_tiles_per_apply": md["n_prefill_tiles"],
           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(gbs / hbm_peak, 4), "algorithmic_bytes_per_launch": bytes_apply,
                        "kernel": "lora_prefill_tc_kernel (tcgen05)",
                        "traffic": load_ncu_traffic("prefill_dram_bytes_per_launch")},
           "tensor": {"achieved_tflops": round(tfs, 2), "peak_tflops": tc_peak, "frac": round(tfs / tc_peak, 5),
                      "ceiling_frac": round((flops_apply / tc_peak / 1e12) / (bytes_apply / hbm_peak / 1e9), 4),
                      "note": "algorithmic flops; HBM-bound at AI %.1f flop/B" % (flops_apply / bytes_apply)}}
    for pool in pools:
        pool.close()
    return out


# ---------------------------------------------------------------- config 4: Zipf paged pool + cold starts
def bench_c4(L, dev, steps: int, world: int, rank: int, use_dist: bool = False):
    """Llama-2-13B (5120) projection, 1000 adapters (ranks 8..128) in pinned host memory, a pool of
    20% of their ranks per GPU, Zipf(1.0) requests: per step 64 decode tokens + one 512-token prompt
    PER GPU (weak scaling), drawn as one global list and routed across the N GPUs by the paper's
    rank-aware Algorithm 1 (serving.route_requests: candidates = the GPUs hosting the adapter, home
    id mod N with the 16 hottest replicated; cost from the models fitted to this library's kernels).
    Misses load on the side stream (LRU eviction) and overlap the applies.  Reports tokens/s with the
    loads included (all GPUs, max over ranks), hit rate, and the cold-start latency next to the
    measured pinned H2D bandwidth."""
    import torch
    import time as _t
    from paper_2401_11240_b200.serving import AdapterCache, HostRepository, route_requests, serves
    from paper_2401_11240_b200.scheduler import measured_model
    H, n_ad, hot = 5120, 1000, list(range(16))
    hot_ids = [int(gen.zipf_perm(gen.BASE_SEED + 3, n_ad)[i]) for i in hot]
    mine = [a for a in range(n_ad) if serves(a, rank, world, hot_ids)]
    repo = HostRepository()
    t0 = _t.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=min(16, len(os.sched_getaffinity(0)))) as ex:
        for a, ad in zip(mine, ex.map(lambda a: gen.c4_adapter(a, H), mine)):
            repo.add(a, ad.rank, ad.scale, torch.from_numpy(ad.A.view(np.int16)).pin_memory(),
                     torch.from_numpy(ad.B.view(np.int16)).pin_memory())
    gen_s = _t.perf_counter() - t0
    budget = sum(gen.c4_rank(a) for a in range(n_ad)) // 5
    pool = L.LoraPool(H, H, n_ad, "bf16", max_total_rank=budget)
    load_kernel = int(os.environ.get("LORA_BENCH_C4_LOAD_KERNEL", "1"))   # A/B of the two load paths
    pool.set_option(L.binding.LORA_OPT_LOAD_KERNEL, load_kernel)
    cache = AdapterCache(pool, repo, budget, n_ad)
    st = torch.cuda.Stream(device=dev)
    model = measured_model("mbgmv", invocations=1)
    T_max = 64 * world + 512 * world
    g = torch.Generator(device="cpu").manual_seed(gen.BASE_SEED + 300 + rank)
    x = torch.randn(T_max, H, generator=g).to(torch.bfloat16).to(dev)
    y = torch.zeros(T_max, H, dtype=torch.bfloat16, device=dev)
    routed = {"decode": 0, "prefill": 0}

    def draw(step):
        """this GPU's share of the step's global requests (Algorithm 1), as (seg_indptr, ids)."""
        d = gen.config_c4_draw(step, n_decode=64 * world, prefill_len=512, n_adapters=n_ad, n_prefill=world)
        dec, pre = [int(a) for a in d["decode_ids"]], [int(a) for a in d["prefill_id"]]
        dec_to, pre_to = route_requests(dec, pre, 512, world, hot_ids, model, gen.c4_rank)
        my_dec = [a for a, g_ in zip(dec, dec_to) if g_ == rank]
        my_pre = [a for a, g_ in zip(pre, pre_to) if g_ == rank]
        routed["decode"] += len(my_dec)
        routed["prefill"] += len(my_pre)
        ip_ = gen.segments_to_indptr([1] * len(my_dec) + [512] * len(my_pre))
        return ip_, np.array(my_dec + my_pre, np.int32)

    def step(ip_, ids):
        cache.ensure(ids.tolist())
        pool.apply(x, y, ip_, ids, stream=st)
        return int(ip_[-1])

    for s_ in range(5):                      # warm the cache
        step(*draw(1000000 + s_))
    torch.cuda.synchronize()
    h0, m0, b0 = cache.hits, cache.misses, cache.loaded_bytes
    routed["decode"] = routed["prefill"] = 0
    # requests are routed when they arrive (the paper's scheduler runs per request), not
    # inside a decode iteration: the steps' routings are computed before the timed region
    draws = [draw(s_) for s_ in range(steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(use_dist)
    w0 = _t.perf_counter()
    e0.record(st)
    tokens = 0
    for ip_, ids_ in draws:
        tokens += step(ip_, ids_)
    e1.record(st)
    torch.cuda.synchronize()
    wall = _t.perf_counter() - w0
    ms = max(e0.elapsed_time(e1), wall * 1e3) / steps
    ms_max = max_over_ranks(ms, use_dist)
    tok_all = tokens
    if use_dist:
        import torch.distributed as dist
        tt = torch.tensor([float(tokens)], dtype=torch.float64, device=dev)
        dist.all_reduce(tt)
        tok_all = float(tt.item())
    # overlap: the same steps on a pool holding every adapter this GPU serves (no loads)
    full = L.LoraPool(H, H, n_ad, "bf16", max_total_rank=sum(gen.c4_rank(a) for a in mine) + 1)
    for a in mine:
        r_, s_a, A_, B_ = repo.items[a]
        full.load_adapter(a, r_, A_, B_, s_a)
    torch.cuda.synchronize()
    for ip_, ids_ in draws[:3]:
        full.apply(x, y, ip_, ids_, stream=st)
    torch.cuda.synchronize()
    w1 = _t.perf_counter()
    e0.record(st)
    for ip_, ids_ in draws:
        full.apply(x, y, ip_, ids_, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ms_noload = max(e0.elapsed_time(e1), (_t.perf_counter() - w1) * 1e3) / steps
    full.close()
    hits, misses = cache.hits - h0, cache.misses - m0
    loaded = cache.loaded_bytes - b0
    # cold-start latency: load 8 non-resident adapters one at a time, call -> ready
    lat = []
    cold = [a for a in mine if a not in cache.lru][:8]
    for a in cold:
        cache.ensure([a])
        t1 = _t.perf_counter()
        while not pool.adapter_ready(a):
            pass
        lat.append((_t.perf_counter() - t1) * 1e3)
    lat_bytes = np.mean([repo.bytes_of(a, 2) for a in cold]) if cold else 0
    peak = h2d_d2h_peak(dev)["h2d"]
    out = {"workload": "c4: Llama-2-13B 5120->5120 bf16, 1000 adapters ranks 8..128 in pinned host memory, pool = 20%% "
                       "of their ranks, Zipf(1.0), per GPU 64 decode + 1x512 prefill tokens/step routed by Algorithm 1, "
                       "LRU, %d GPU(s)" % world,
           "value": round(tok_all / steps / (ms_max * 1e-3), 1), "unit": "tokens/s, all GPUs (loads included)",
           "ms_per_step": round(ms_max, 4),
           "routing": {"policy": "Algorithm 1 (rank-aware, P:781-814), MBGMV model fitted on B200",
                       "this_gpu_decode_requests_per_step": round(routed["decode"] / steps, 2),
                       "this_gpu_prompts_per_step": round(routed["prefill"] / steps, 3)},
           "load_path": "zero-copy gather kernel (LORA_OPT_LOAD_KERNEL=1)" if load_kernel else
                        "cudaMemcpyAsync per page run (default)",
           "ms_per_step_all_resident": round(ms_noload, 4),
           "overlap": round(ms_noload / ms, 3),   # 1.0 = the cold-start loads cost nothing
           "steps": steps, "hit_rate": round(hits / max(1, hits + misses), 4), "loads_per_step": round(misses / steps, 2),
           "load_GBps_effective": round(loaded / (ms * steps * 1e-3) / 1e9, 2),
           "cold_start_ms_per_adapter": round(float(np.median(lat)), 3) if lat else None,
           "cold_start_bytes_per_adapter": int(lat_bytes),
           "cold_start_GBps": round(lat_bytes / (np.median(lat) * 1e-3) / 1e9, 2) if lat else None,
           "h2d_pinned_peak_GBps": round(peak, 1), "host_repo_setup_s": round(gen_s, 1)}
    pool.close()
    return out


def h2d_d2h_peak(dev, mib: int = 256, reps: int = 20):
    """pinned host <-> device copy bandwidth (GB/s), best of `reps` 256 MiB copies each way."""
    import torch
    src = torch.empty(mib * 2 ** 20, dtype=torch.uint8).pin_memory()
    dst = torch.empty(mib * 2 ** 20, dtype=torch.uint8, device=dev)
    out = {}
    for name, (a, b_) in (("h2d", (dst, src)), ("d2h", (src, dst))):
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a.copy_(b_, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = round(src.numel() / (best * 1e-3) / 1e9, 2)
    return out


def bench_cold_start(L, dev, H: int = 5120, reps: int = 15):
    """Cold start (§2.3 C1, P:341-343 / P:358-362: load latency grows with the rank) and the
    paper's CPU-assisted prefill (NEXT f1) re-measured on B200:
      load_by_rank: one 13B projection adapter (5120 -> 5120, bf16) of rank r, lora_load_adapter call ->
        lora_adapter_ready (host polling), median (and best) of `reps`, by the default cudaMemcpyAsync path and by
        the zero-copy gather kernel (LORA_OPT_LOAD_KERNEL), next to the measured pinned H2D peak;
      cpu_delta: the paper's CPU LoRA for a prompt of L tokens while that adapter loads -- torch CPU
        (x @ A) @ B in bf16 on all host cores, best of 7 -- vs the best load latency of the same rank.
        cpu_wins marks the cells where computing on the host would beat waiting for the load."""
    import torch
    import time as _t
    peak = h2d_d2h_peak(dev)
    ranks = (8, 16, 32, 64, 128)
    lengths = (1, 16, 128, 512)
    res = {"h2d_pinned_peak_GBps": peak["h2d"], "d2h_pinned_peak_GBps": peak["d2h"],
           "pcie_gen5_x16_nominal_GBps": 64.0, "load_by_rank": {}, "cpu_delta": {}}
    torch.set_num_threads(len(os.sched_getaffinity(0)))
    for r in ranks:
        ad = gen.make_adapter(gen.BASE_SEED + 3, 77, 1, r, H, H, "bf16")
        A = torch.from_numpy(ad.A.view(np.int16)).pin_memory()
        B = torch.from_numpy(ad.B.view(np.int16)).pin_memory()
        row = {"bytes": int(r * 2 * H * 2)}
        for name, kern in (("memcpy", 0), ("gather_kernel", 1)):
            pool = L.LoraPool(H, H, 4, "bf16", max_total_rank=256)
            pool.set_option(L.binding.LORA_OPT_LOAD_KERNEL, kern)
            lat = []
            for i in range(reps + 2):
                t1 = _t.perf_counter()
                pool.load_adapter(i, r, A, B, ad.scale)
                while not pool.adapter_ready(i):
                    pass
                lat.append((_t.perf_counter() - t1) * 1e6)
                pool.unload_adapter(i)
                torch.cuda.synchronize()
            us = float(np.median(lat[2:]))
            row[name + "_us"] = round(us, 1)
            row[name + "_GBps"] = round(row["bytes"] / (us * 1e-6) / 1e9, 2)
            row[name + "_best_us"] = round(float(np.min(lat[2:])), 1)
            pool.close()
        res["load_by_rank"][str(r)] = row
        Ac = A.view(torch.bfloat16).reshape(r, H).t().contiguous()   # stored rank-major [r][H_in]
        Bc = B.view(torch.bfloat16).reshape(r, H)
        # both sides best-of: the fastest load of this rank vs the fastest host computation
        load_us = min(row["memcpy_best_us"], row["gather_kernel_best_us"])
        cells = {}
        for n in lengths:
            xc = torch.randn(n, H).to(torch.bfloat16)
            (xc @ Ac) @ Bc
            cts = []
            for _ in range(7):
                t1 = _t.perf_counter()
                (xc @ Ac) @ Bc
                cts.append((_t.perf_counter() - t1) * 1e6)
            cpu_us = float(np.min(cts))
            cells[str(n)] = {"cpu_us": round(cpu_us, 1), "load_us": load_us, "cpu_wins": bool(cpu_us < load_us)}
        res["cpu_delta"][str(r)] = cells
    res["cpu_threads"] = torch.get_num_threads()
    res["cpu_wins_any"] = any(c["cpu_wins"] for v in res["cpu_delta"].values() for c in v.values())
    return res


# ---------------------------------------------------------------- config 5: Llama-2-70B shapes, TP shards
def bench_fused_base(L, dev, reps: int, tc_peak: float):
    """NEXT f2: y = x·W + s·(x·A)·B on c3 shapes (32 x 512 tokens, 4096 -> 4096, ranks 8..128).
    fused = lora_apply_fused_base (one tcgen05 kernel); unfused = cuBLAS x·W then lora_apply (the
    delta pass reads and writes y again); base = cuBLAS x·W alone.  CUDA graphs of 4 calls, L2
    flushed before each replay, median of `reps`."""
    import torch
    b = gen.config_c3()
    pool = L.LoraPool(b.H_in, b.H_out, 64, "bf16", max_total_rank=sum(a.rank for a in b.adapters))
    for a in b.adapters:
        pool.load_adapter(a.id, a.rank, torch.from_numpy(a.A.view(np.int16)).pin_memory(),
                          torch.from_numpy(a.B.view(np.int16)).pin_memory(), a.scale)
    g = torch.Generator(device="cpu").manual_seed(gen.BASE_SEED + 300)
    x = torch.from_numpy(b.x.view(np.int16)).to(dev).view(torch.bfloat16)
    W = (torch.randn(b.H_in, b.H_out, generator=g) / b.H_in ** 0.5).to(torch.bfloat16).to(dev)
    y = torch.empty(b.T, b.H_out, dtype=torch.bfloat16, device=dev)
    st = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)
    NP = 4
    calls = {
        "fused": lambda: pool.apply_fused_base(x, W, y, b.seg_indptr, b.adapter_ids, stream=st),
        "unfused": lambda: (torch.matmul(x, W, out=y), pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)),
        "base": lambda: torch.matmul(x, W, out=y),
    }
    sum_tr = sum(int(b.seg_indptr[i + 1] - b.seg_indptr[i]) * gen.C3_RANKS[i % 5] for i in range(len(b.adapter_ids)))
    flops = 2.0 * b.T * b.H_in * b.H_out + 2.0 * sum_tr * (b.H_in + b.H_out)
    out = {"workload": "c3 shapes: 32 x 512 tokens, 4096 -> 4096, 32 adapters ranks 8..128, W random bf16",
           "tflop_per_call": round(flops / 1e12, 4), "peak_tflops": tc_peak}
    for name, fn in calls.items():
        with torch.cuda.stream(st):
            fn()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            for _ in range(NP):
                fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st):
                graph.replay()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / NP)
        us = float(np.median(ts))
        out[name] = {"us": round(us, 1), "tflops": round(flops / (us * 1e-6) / 1e12, 1),
                     "frac_tc_peak": round(flops / (us * 1e-6) / 1e12 / tc_peak, 3)}
        del graph
    out["fused_vs_unfused"] = round(out["unfused"]["us"] / out["fused"]["us"], 3)
    pool.close()
    return out


def _graph_us(body, st, reps: int, n_per_replay: int) -> float:
    """median device time (us) per call of `body` (n_per_replay calls per replay) from a CUDA graph."""
    import torch
    with torch.cuda.stream(st):
        body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        body()
    ts = []
    for _ in range(max(1, reps)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n_per_replay)
    del g
    return float(np.median(ts))


def bench_c5(L, dev, reps: int, hbm_peak: float, world: int = 1, rank: int = 0, use_dist: bool = False):
    """c5: Llama-2-70B per-layer projection shapes (q/o 8192^2, k/v 8192->1024, gate/up 8192->28672,
    down 28672->8192), decode 64 tokens over 32 adapters of ranks [16,32,64,128][a mod 4].
    tp = 1: lora_apply on the full shape.  tp > 1 (BJ scheme): the rank's shard pool
    (lora_load_adapter_shard from the full pinned adapters) and
      shard_kernels: lora_apply_shrink (shrink + k-reduce into the compact v) + lora_apply_expand --
                     one rank's kernels without the collective;
      apply_tp:      lora_apply_tp = the same kernels + ncclAllReduce of the compact v (15,360 B) on the
                     library's communicator.  With one GPU (this run) the communicator is world-1 (its
                     all-reduce is a local no-op); under torchrun with N GPUs the tp = N row runs the
                     real N-rank all-reduce over NVLink, timed as the max over ranks.
      nocomm:        the scheme without a collective: column-parallel shapes (q, kv, gate_up)
                     keep A whole and split B by output columns (the paper's scheme); the row-parallel
                     shape (down) splits A with its x shard and keeps B whole, adding the full-width delta of
                     its partial v into the partial y that the base layer's own all-reduce completes
                     (linearity) -- more adapter bytes per GPU, no exchange.  `pick` names the faster.
    Device time per apply from a CUDA graph over enough distinct pools that the adapter rows exceed L2."""
    import torch
    from paper_2401_11240_b200.binding import TPComm
    shapes = {"q": (8192, 8192), "kv": (8192, 1024), "gate_up": (8192, 28672), "down": (28672, 8192)}
    ranks = [gen.C5_RANKS[a % 4] for a in range(32)]
    b = gen.config_c5("q")
    ip, ids = b.seg_indptr, b.adapter_ids
    T = 64
    st = torch.cuda.Stream(device=dev)
    comm = TPComm.from_process_group() if use_dist else TPComm(L.binding.tp_unique_id(), 0, 1)
    out = {}
    for name, (H_in, H_out) in shapes.items():
        full = [gen.make_adapter(gen.BASE_SEED + 4, 50 + list(shapes).index(name), a, ranks[a], H_in, H_out, "bf16")
                for a in range(32)]
        pinned = [(torch.from_numpy(a.A.view(np.int16)).pin_memory(), torch.from_numpy(a.B.view(np.int16)).pin_memory())
                  for a in full]
        row = {}
        for tp in (1, 2, 4, 8):
            if use_dist and tp != world:
                continue   # multi-GPU: the tp = N row with the real collective only
            trank = rank if use_dist else 0
            hi, ho = H_in // tp, H_out // tp
            adapter_bytes = sum(ranks) * (hi + ho) * 2
            n_pools = max(2, -(-400_000_000 // adapter_bytes))
            pools = []
            for _ in range(n_pools):
                pool = L.LoraPool(hi, ho, 32, "bf16", max_total_rank=sum(ranks))
                for a, (A, B) in zip(full, pinned):   # this rank's shard, straight from the full adapter
                    pool.load_adapter_shard(a.id, a.rank, A, trank * hi, B, trank * ho, a.scale)
                if tp > 1:
                    pool.tp_init(comm)
                pools.append(pool)
            torch.cuda.synchronize()
            x = torch.randn(T, hi).to(torch.bfloat16).to(dev)
            ys = [torch.zeros(T, ho, dtype=torch.bfloat16, device=dev) for _ in pools]
            byts = adapter_bytes + T * hi * 2 + 2 * T * ho * 2
            r = {"adapter_MB_per_gpu": round(adapter_bytes / 1e6, 2)}
            if tp == 1:
                us = _graph_us(lambda: [p.apply(x, y, ip, ids, stream=st) for p, y in zip(pools, ys)], st, reps, n_pools)
                r.update({"us_per_apply": round(us, 3), "GBps": round(byts / (us * 1e-6) / 1e9, 1),
                          "roofline_frac": round(byts / (us * 1e-6) / 1e9 / hbm_peak, 4)})
            else:
                pools[0].plan(ip, ids)
                nv = pools[0].metadata()["v_floats"]
                vs = [torch.zeros(max(1, nv), dtype=torch.float32, device=dev) for _ in pools]
                us_k = _graph_us(lambda: [(p.apply_shrink(x, ip, ids, v, stream=st), p.apply_expand(y, v, stream=st))
                                          for p, y, v in zip(pools, ys, vs)], st, reps, n_pools)
                us_tp = _graph_us(lambda: [p.apply_tp(x, y, ip, ids, stream=st) for p, y in zip(pools, ys)], st, reps,
                                  n_pools)
                if use_dist:
                    us_k = max_over_ranks(us_k, True)
                    us_tp = max_over_ranks(us_tp, True)
                # the scheme without a collective: plain lora_apply on the wider shard
                row_par = name == "down"
                nhi, nho = (hi, H_out) if row_par else (H_in, ho)
                nb = sum(ranks) * (nhi + nho) * 2
                npools = max(2, -(-400_000_000 // nb))
                npl = []
                for _ in range(npools):
                    pool = L.LoraPool(nhi, nho, 32, "bf16", max_total_rank=sum(ranks))
                    for a, (A, B) in zip(full, pinned):
                        pool.load_adapter_shard(a.id, a.rank, A, trank * hi if row_par else 0, B, 0 if row_par else trank * ho,
                                                a.scale)
                    npl.append(pool)
                torch.cuda.synchronize()
                xn = torch.randn(T, nhi).to(torch.bfloat16).to(dev)
                yn = [torch.zeros(T, nho, dtype=torch.bfloat16, device=dev) for _ in npl]
                us_n = _graph_us(lambda: [p.apply(xn, y, ip, ids, stream=st) for p, y in zip(npl, yn)], st, reps, npools)
                if use_dist:
                    us_n = max_over_ranks(us_n, True)
                for pool in npl:
                    pool.close()
                del npl, yn
                r.update({"nocomm": {"scheme": "A split, B whole, delta into the partial y" if row_par
                                     else "A whole, B split (the paper's)",
                                     "adapter_MB_per_gpu": round(nb / 1e6, 2), "us": round(us_n, 3)},
                          "pick": "nocomm" if us_n < us_tp else "allreduce_v"})
                r.update({"v_allreduce_bytes": int(nv * 4),
                          "shard_kernels_us": round(us_k, 3),
                          "shard_kernels_roofline_frac": round(byts / (us_k * 1e-6) / 1e9 / hbm_peak, 4),
                          "apply_tp_us": round(us_tp, 3),
                          "allreduce_us": round(us_tp - us_k, 3),
                          "comm": "NCCL %d ranks (NVLink)" % world if use_dist else "NCCL world 1 (local: no transfer)"})
                del vs
            row["tp%d" % tp] = r
            for pool in pools:
                pool.close()
            del pools, ys
        if "tp1" in row:
            for tp in (2, 4, 8):
                if "tp%d" % tp in row:
                    row["tp%d" % tp]["shard_speedup_vs_tp1"] = round(row["tp1"]["us_per_apply"] /
                                                                     row["tp%d" % tp]["shard_kernels_us"], 2)
        out[name] = row
    comm.close()
    if use_dist:
        return {"workload": "c5 TP decode, tp = %d across the N GPUs of this run" % world, "per_shape": out}
    # prefill 8 x 512 tokens (32 token tiles: the planner splits each tile's columns over SMs/tiles CTAs)
    pf = {}
    for proj in ("q", "gate", "down"):
        b = gen.config_c5(proj, prefill=True)
        pools = []
        for _ in range(2):
            pool = L.LoraPool(b.H_in, b.H_out, 16, "bf16", max_total_rank=sum(a_.rank for a_ in b.adapters))
            for a_ in b.adapters:
                pool.load_adapter(a_.id, a_.rank, torch.from_numpy(a_.A.view(np.int16)).pin_memory(),
                                  torch.from_numpy(a_.B.view(np.int16)).pin_memory(), a_.scale)
            pools.append(pool)
        torch.cuda.synchronize()
        x = torch.from_numpy(b.x.view(np.int16)).to(dev)
        ys = [torch.zeros(b.T, b.H_out, dtype=torch.int16, device=dev) for _ in pools]

        n_rounds = 4   # 8 applies per replay (the two pools alternate): the graph launch is amortised

        def body():
            for _ in range(n_rounds):
                for pool, y in zip(pools, ys):
                    pool.apply(x, y, b.seg_indptr, b.adapter_ids, stream=st)

        with torch.cuda.stream(st):
            body()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            body()
        ts = []
        for _ in range(max(1, reps)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st):
                g.replay()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / (n_rounds * len(pools)))
        us = float(np.median(ts))
        sum_r = sum(a_.rank for a_ in b.adapters)
        byts = 2 * (sum_r * (b.H_in + b.H_out) + b.T * b.H_in + 2 * b.T * b.H_out)
        pf[proj] = {"shape": [b.H_in, b.H_out], "tokens": b.T, "us_per_apply": round(us, 2),
                    "roofline_frac": round(byts / (us * 1e-6) / 1e9 / hbm_peak, 4)}
        for pool in pools:
            pool.close()
        del pools, ys
    return {"workload": "c5: Llama-2-70B projection shapes, decode 64 tokens over 32 adapters ranks 16..128, bf16; "
                        "tp>1 = one rank's shard pool: shard kernels alone and lora_apply_tp (+ the library's NCCL "
                        "all-reduce of the compact v); prefill_tp1: 8 x 512 tokens over 8 adapters on the tcgen05 kernel",
            "prefill_tp1": pf,
            "shapes": {k: list(v) for k, v in shapes.items()}, "per_shape": out}


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    use_dist = init_dist(world, local)
    import paper_2401_11240_b200 as L

    layers = args.layers
    ip, ids = layer_batch_meta(rank)
    dev = torch.device("cuda", local)

    # ---- pools: generate adapters (threads), load through the cold-start path
    t_gen = time.perf_counter()
    pools = []
    with cf.ThreadPoolExecutor(max_workers=min(16, len(os.sched_getaffinity(0)))) as ex:
        futs = {(l, p): ex.submit(make_pool_adapters, l, p, rank) for l in range(layers) for p in range(len(PROJS))}
        ranks_sum = None
        for l in range(layers):
            row = []
            for p in range(len(PROJS)):
                ads = futs[(l, p)].result()
                pool = L.LoraPool(H, H, 32, "bf16", max_total_rank=sum(a.rank for a in ads))
                for a in ads:
                    A = torch.from_numpy(a.A.view(np.int16)).pin_memory()
                    B = torch.from_numpy(a.B.view(np.int16)).pin_memory()
                    pool.load_adapter(a.id, a.rank, A, B, a.scale)
                ranks_sum = sum(a.rank for a in ads)
                row.append(pool)
            pools.append(row)
    torch.cuda.synchronize()
    for row in pools:
        for pool in row:
            pool.release_host_buffers()
    t_gen = time.perf_counter() - t_gen

    # ---- activations: x per layer (attention input for q/k/v, o-proj input), y per projection
    g = torch.Generator(device="cpu").manual_seed(gen.BASE_SEED + 100 + rank)
    # one contiguous buffer per kind (per-layer views go to the API), so the e2e step moves the whole
    # step's x in one H2D and all y in one D2H copy
    xs_all = torch.empty(layers, 2, T_DECODE, H, dtype=torch.bfloat16, device=dev)
    for l in range(layers):
        for i in range(2):
            xs_all[l, i].copy_(torch.randn(T_DECODE, H, generator=g).to(torch.bfloat16))
    ys_all = torch.zeros(layers, len(PROJS), T_DECODE, H, dtype=torch.bfloat16, device=dev)
    xs = [[xs_all[l, i] for i in range(2)] for l in range(layers)]
    ys = [[ys_all[l, p] for p in range(len(PROJS))] for l in range(layers)]
    stream = torch.cuda.Stream(device=dev)

    mode = args.qkv_mode
    fuse = mode == "fused"
    side = [torch.cuda.Stream(device=dev) for _ in range(2)]

    def step(st, only=None):
        for l in (range(layers) if only is None else [only]):
            if mode == "fused":   # q, k, v share x and the batch: one fused launch pair (lora_apply_multi), then o
                L.apply_multi(pools[l][:3], [xs[l][0]] * 3, ys[l][:3], ip, ids, stream=st)
                pools[l][3].apply(xs[l][1], ys[l][3], ip, ids, stream=st)
            elif mode == "streams":   # q, k, v are independent: fork onto 3 streams, join before o
                ev = torch.cuda.Event()
                ev.record(st)
                for k, s2 in enumerate(side):
                    s2.wait_event(ev)
                    pools[l][k + 1].apply(xs[l][0], ys[l][k + 1], ip, ids, stream=s2)
                pools[l][0].apply(xs[l][0], ys[l][0], ip, ids, stream=st)
                for s2 in side:
                    e2 = torch.cuda.Event()
                    e2.record(s2)
                    st.wait_event(e2)
                pools[l][3].apply(xs[l][1], ys[l][3], ip, ids, stream=st)
            else:
                for p in range(len(PROJS)):
                    pools[l][p].apply(xs[l][0 if p < 3 else 1], ys[l][p], ip, ids, stream=st)

    with torch.cuda.stream(stream):
        step(stream)               # sizes the pools' scratch outside capture
    torch.cuda.synchronize()
    launches0 = sum(pool.info()["kernel_launches"] for row in pools for pool in row)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step(stream)
    launches_per_step = sum(pool.info()["kernel_launches"] for row in pools for pool in row) - launches0
    for _ in range(max(3, args.warmup)):
        graph.replay()
    barrier(use_dist)

    # timed windows of exactly K steps, each bracketed by barrier + synchronize, max over ranks;
    # repeated until >= min_window_ms of device time is covered (so the clock sampler sees the load
    # and run-to-run spread is visible); the median window is reported
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    windows = []
    with ClockSampler(local) as clk:
        while True:
            barrier(use_dist)
            ev0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(args.steps):
                    graph.replay()
            ev1.record(stream)
            torch.cuda.synchronize()
            barrier(use_dist)
            windows.append(max_over_ranks(ev0.elapsed_time(ev1), use_dist))
            done = sum(windows) >= args.min_window_ms and len(windows) >= 3
            if use_dist:   # every rank takes the same decision (rank 0's)
                flag = torch.tensor([1.0 if done else 0.0], dtype=torch.float64,
                                    device="cpu" if SHARE_GPU else dev)
                import torch.distributed as dist
                dist.broadcast(flag, 0)
                done = bool(flag.item() > 0.5)
            if done or len(windows) >= 10000:
                break
    ms_total = float(np.median(windows))
    ms_step = ms_total / args.steps
    tokens_per_step_all = T_DECODE * world
    value = tokens_per_step_all / (ms_step / 1000.0)

    # ---- roofline of the decode kernel (the only kernel of the step)
    hbm_peak, tc_peak, peak_src = measured_peaks()
    bytes_apply = algorithmic_bytes_per_apply(ranks_sum, T_DECODE)
    n_applies = layers * len(PROJS)
    kernel_us = ms_step * 1000.0 / n_applies      # per projection apply; includes inter-kernel gaps
    achieved = bytes_apply / (kernel_us * 1e-6) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": load_ncu_traffic(),
                "kernel": "decode: lora_shrink_mma_kernel + lora_expand_mma_kernel (PDL-chained pair per apply; "
                          "q/k/v mode %s)" % mode,
                "algorithmic_bytes_per_launch": bytes_apply,
                "avg_launch_us": round(kernel_us, 3), "peak_source": peak_src,
                "note": "per projection apply: graph step time / 128 applies (gaps included); traffic = ncu dram "
                        "read+write per projection apply (profiles/ncu_decode_summary.json)"}

    # ---- e2e through the public API with host buffers
    x_host = xs_all.cpu().pin_memory()
    y_host = torch.empty(tuple(ys_all.shape), dtype=torch.bfloat16).pin_memory()
    h2d = x_host.numel() * 2
    d2h = y_host.numel() * 2

    # pipelined in NCH layer chunks on two copy streams (PCIe is full duplex): chunk k's x H2D, its
    # applies, its y D2H.  Only true buffer reuse orders consecutive steps: step i+1's x H2D of chunk
    # k waits for step i's applies of chunk k (they read x), and its applies of chunk k wait for step
    # i's y D2H of chunk k (it reads y) -- so the next step's H2D and applies overlap this step's D2H
    NCH = 4 if layers % 4 == 0 else 1
    LPC = layers // NCH
    h2d_st = torch.cuda.Stream(device=dev)
    d2h_st = torch.cuda.Stream(device=dev)
    ev_x = [torch.cuda.Event() for _ in range(NCH)]      # x chunk k landed
    ev_used = [torch.cuda.Event() for _ in range(NCH)]   # applies of chunk k done (x free, y ready)
    ev_out = [torch.cuda.Event() for _ in range(NCH)]    # y chunk k left for the host
    for k in range(NCH):
        ev_used[k].record(stream)
        ev_out[k].record(d2h_st)

    def e2e_step():
        for k in range(NCH):
            sl = slice(k * LPC, (k + 1) * LPC)
            h2d_st.wait_event(ev_used[k])
            with torch.cuda.stream(h2d_st):
                xs_all[sl].copy_(x_host[sl], non_blocking=True)
                ev_x[k].record(h2d_st)
        for k in range(NCH):
            sl = slice(k * LPC, (k + 1) * LPC)
            stream.wait_event(ev_x[k])
            stream.wait_event(ev_out[k])
            with torch.cuda.stream(stream):
                for l in range(k * LPC, (k + 1) * LPC):
                    step(stream, only=l)
                ev_used[k].record(stream)
            d2h_st.wait_event(ev_used[k])
            with torch.cuda.stream(d2h_st):
                y_host[sl].copy_(ys_all[sl], non_blocking=True)
                ev_out[k].record(d2h_st)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    barrier(use_dist)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    h2d_st.wait_event(e0)           # the first timed copy starts after e0
    d2h_st.wait_event(e0)
    for _ in range(args.e2e_steps):
        e2e_step()
    stream.wait_stream(d2h_st)      # the timed region ends when the last step's y has landed
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1000.0
    e2e_ms = max(e0.elapsed_time(e1), wall) / args.e2e_steps
    e2e_ms = max_over_ranks(e2e_ms, use_dist)
    e2e = {"value": tokens_per_step_all / (e2e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": args.e2e_steps, "ms_per_step": round(e2e_ms, 4)}

    # ---- config 3 prefill on the tensor-core kernel (reported beside the decode headline)
    prefill = None
    if args.prefill_layers > 0:
        prefill = bench_prefill(L, args.prefill_layers, args.prefill_steps, dev, hbm_peak, tc_peak, rank)

    c4 = None
    if args.c4_steps > 0:
        c4 = bench_c4(L, dev, args.c4_steps, world, rank, use_dist and not SHARE_GPU)

    cold = None
    if args.cold_start and rank == 0:
        cold = bench_cold_start(L, dev)

    c5 = None
    if args.c5_reps > 0:
        c5 = bench_c5(L, dev, args.c5_reps, hbm_peak, world, rank, use_dist and not SHARE_GPU)

    fused_base = None
    if args.fused_base_reps > 0 and rank == 0:
        fused_base = bench_fused_base(L, dev, args.fused_base_reps, tc_peak)

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, dt = cpu_oracle_tokens_per_s(args.cpu_sample_layers, 0)
        reps = max(1, int(10.0 / max(dt, 1e-3)))
        if reps > 1:
            v, cores, dt = cpu_oracle_tokens_per_s(args.cpu_sample_layers, 0, reps=min(reps, 100))
        v1, _, dt1 = cpu_oracle_tokens_per_s(1, 0, n_threads=1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": "%d of 32 layers x 4 projections (64 tokens), fp64 C oracle, OpenMP over tokens, "
                         "extrapolated to 32 layers; %.1f s of CPU work" % (args.cpu_sample_layers, dt),
               "cpu_model": _cpu_model(),
               "single_thread_value": v1,
               "single_thread_sample": "1 layer x 4 projections, 1 thread, extrapolated; %.1f s" % dt1}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (workloads.gen seeded PCG64 adapters; random-init, no checkpoints)",
                "config": {"workload": WORKLOAD, "layers": layers, "projections": list(PROJS),
                           "tokens_per_step_per_gpu": T_DECODE, "adapters_per_pool": 32,
                           "ranks": list(gen.C2_RANKS), "hidden": H, "parallelism": "dp%d (request partition)" % world,
                           "l2": "inputs larger than L2 (%.2f GB adapter working set per GPU)" %
                                 (layers * len(PROJS) * ranks_sum * 2 * H * 2 / 1e9),
                           "timing": "CUDA graph of one step, K replays per window, CUDA events, max over ranks; "
                                     "median of %d windows" % len(windows),
                           "qkv_mode": mode},
                "windows": {"n": len(windows), "ms_per_step_min": round(min(windows) / args.steps, 5),
                            "ms_per_step_max": round(max(windows) / args.steps, 5),
                            "covered_ms": round(sum(windows), 1)},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
                "gpu_launches": int(launches_per_step * args.steps),
                "prefill": prefill,
                "c4": c4,
                "cold_start": cold,
                "c5": c5,
                "fused_base": fused_base,
                "setup_s": round(t_gen, 1)}
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as fh:
                fh.write(s + "\n")
    for row in pools:
        for pool in row:
            pool.close()
    if use_dist:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
