"""bench.py's N>1 path (torchrun, one process per rank, CUDA-IPC wiring, shared-memory host image,
max-over-ranks timing) exercised with 2 ranks on the single test GPU (gloo for the host-side plumbing)."""
import json
import os
import subprocess
import sys

import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_same_gpu():
    need_gpu()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29541", "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "1", "--workload", "C1", "--dist-backend", "gloo", "--same-gpu", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["policy"] == "interleave"


def test_bench_self_launch_without_torchrun():
    """`python bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (the driver's SCALE invocation)."""
    need_gpu()
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "1", "--workload", "C1",
           "--same-gpu", "--no-cpu-baseline"]
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
