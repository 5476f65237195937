"""The data-parallel training step on the B200 (one rank): bench.py under
torch.distributed.run with CANVAS_DP_SELFTEST=1 builds the NCCL process group,
issues the bucketed gradient all-reduces (dp.GradBuckets) on the side stream and
captures the whole step, collectives included, in one CUDA graph — the N-GPU
code path, exercised on a 1-GPU box."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dp_step_captured_with_nccl():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, CANVAS_DP_SELFTEST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "bench.py"), "--gpus", "1", "--batch", "32", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-context"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["config"]["parallelism"] == "dp1"
    assert line["config"]["cuda_graph"].startswith("whole step captured"), line["config"]["cuda_graph"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0
