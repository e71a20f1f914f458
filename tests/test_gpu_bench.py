"""bench.py's multi-GPU launch path on the one GPU of a test
box: torchrun with 2 ranks sharing cuda:0 over gloo (LVN_DIST_BACKEND=gloo;
the 8-GPU run uses the library's NCCL communicator), config C1 with every pass
sharded; rank 0 prints one JSON line of the bench contract."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_gloo_on_one_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    env = dict(os.environ, LVN_DIST_BACKEND="gloo", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "c1", "--no-cpu-baseline", "--shard-min-arcs-log2", "16"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0 and d["unit"] == "edges/s"
    assert d["config"]["workload"] == "c1" and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and 0.05 < d["modularity"] < 1.0
    assert d["sharded_passes"] >= 1
