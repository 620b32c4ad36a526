"""bench.py's N > 1 path (vocab-sharded head, what the driver's 2/4/8-GPU
scaling run executes) on the one GPU available: torchrun with 2 ranks, both
on cuda:0 over gloo (the test-only SPARTON_BENCH_DEVICE / SPARTON_BENCH_BACKEND
overrides; NCCL refuses two ranks on one device).  Checks the contract's JSON
line: whole-job value, e2e through the sharded public API with host copies,
the cfg4 record, and max-over-ranks timing keys."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_one_gpu(cuda_device):
    env = dict(os.environ, SPARTON_BENCH_DEVICE="0", SPARTON_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(REPO / "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "cfg2", "--no-cpu"]
    r = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    assert d["config"]["workload"] == "cfg2" and d["config"]["parallelism"] == "vocab-shard2"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["gpu_launches"] > 0 and d["roofline"]["achieved"] > 0
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    c4 = d["cfg4"]
    assert c4["config"]["workload"] == "cfg4" and c4["config"]["D"] == 1024 and c4["config"]["B"] == 2048
    assert c4["value"] > 0 and c4["ms_per_step"] > 0
    fg = d["fused_gather"]
    assert "unavailable" in fg or fg["value"] > 0
