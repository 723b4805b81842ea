"""The one-process-per-rank path: CUDA-IPC wiring exchanged through torch.distributed (gloo), two
processes on the test box's single B200, result checked against the oracle by rank 0."""
import json
import os
import subprocess
import sys

import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("policy,sliced,k", [("interleave", 1, 2), ("stage", 0, 1)])
def test_two_processes_ipc(policy, sliced, k):
    need_gpu()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tools", "mp_coldstart.py"),
           "--same-gpu", "--policy", policy, "--sliced", str(sliced), "--k", str(k)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["rel"] <= 1e-2 and d["trials_identical"]


@pytest.mark.parametrize("policy,sliced,k", [("interleave", 1, 2), ("stage", 0, 1)])
def test_two_devices_oracle_parity(policy, sliced, k):
    """Cross-device run (one process per GPU, CUDA IPC over NVLink, device-side readiness words written into a peer's
    memory) checked against the oracle; runs only where the box has two GPUs."""
    need_gpu()
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29519", os.path.join(ROOT, "tools", "mp_coldstart.py"),
           "--policy", policy, "--sliced", str(sliced), "--k", str(k)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["rel"] <= 1e-2 and d["trials_identical"]
