"""Sharded paths at world > 1 over NCCL; runs whenever two or more
GPUs are visible, skips otherwise (the gloo world-2 tests cover the host logic)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_torchrun_world2_matches_goldens():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29547", "tools/dist_check.py"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = next(l for l in out.stdout.splitlines() if l.startswith("DIST_CHECK "))
    d = json.loads(line[len("DIST_CHECK "):])
    assert d["world"] == 2
    assert d["by_vector_err"] <= 1e-10 and d["by_term_err"] <= 1e-10 and d["cfg4_zz_err"] <= 1e-10


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_bench_under_torchrun_world2():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29548", "bench.py", "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--replicas", "2", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["cfg4_circuits"]["circuits"] == 1024
