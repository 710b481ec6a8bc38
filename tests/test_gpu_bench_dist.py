"""The bench's N > 1 control flow (torchrun, barriers, max over ranks, a single rank-0 JSON line,
request partitioning in c4) on a one-GPU box: LORA_BENCH_SHARE_GPU=1 puts both ranks on cuda:0 with
gloo plumbing (the driver's scaling run uses one GPU per rank and NCCL)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    # a fixed port can still be held on a reused box (the first run here failed that way)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(args, port=None):
    port = port or _free_port()
    env = dict(os.environ, LORA_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2"] + args
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 only
    return json.loads(lines[0])


def test_bench_two_ranks_one_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    d = _run(["--steps", "10", "--warmup", "3", "--layers", "2", "--e2e-steps", "2", "--prefill-layers", "0",
              "--c4-steps", "2", "--c5-reps", "0", "--fused-base-reps", "0"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["cpu_baseline"] is None
    assert d["c4"]["value"] > 0 and "2 GPU(s)" in d["c4"]["workload"]
    assert d["c4"]["routing"]["policy"].startswith("Algorithm 1")
    ref = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert ref["impl"] == "reference" and ref["e2e"]["h2d_bytes_per_step"] == 0
