"""bench.py's multi-GPU path (request sharding, barriers, max-over-ranks
timing, token sum) under torchrun with two ranks.  One GPU is all gpurun
offers, so the two ranks share it with the gloo backend (BENCH_BACKEND=gloo)
on the tiny model; with N real GPUs the driver runs the same code over NCCL."""
import json
import os
import socket
import subprocess
import sys

import pytest

import vc_testlib as T

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_small(cuda):
    env = dict(os.environ, BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(T.ROOT, "bench.py"),
           "--gpus", "2", "--small", "--steps", "3", "--warmup", "2", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=T.ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 prints the one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 32 and d["scaling"] == "weak"
    assert d["tokens_identical_to_full_kv"] and d["value"] > 0


def test_two_ranks_remote_prefix_small(cuda):
    """configs[3] under torchrun: each rank streams its own requests' payloads
    over its own copy engine; tokens summed, makespan max over ranks."""
    env = dict(os.environ, BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(T.ROOT, "bench.py"),
           "--gpus", "2", "--small", "--config", "4", "--out-tokens", "32"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=T.ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 8 and d["tokens_identical_to_full_kv"]
    assert d["value"] > 0 and d["vericache"]["verifies"] > 0
