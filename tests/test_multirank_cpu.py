"""Host-side logic of the N>1 path on CPU (gloo, world_size 2): every rank builds the same plan through
the C ABI, and the shared-memory host image (bench.py's one-DRAM-copy mode) equals the single-process one."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, tmp, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import harness
    from paper_2503_17707_b200.api import Plan
    from synth.configs import WORKLOADS
    w = WORKLOADS["C1"]
    plan = Plan(w.model, w.adapters, world, policy="interleave", vocab_sliced=1, chunk_bytes=64 << 10)
    dumps = [None] * world
    dist.all_gather_object(dumps, plan.dump())
    n = plan.sizes.host_base_bytes
    path = os.path.join(tmp, "base")
    if rank == 0:
        t = torch.from_file(path, shared=True, size=n, dtype=torch.uint8)
        t.zero_()
        harness.fill_host_images(plan, t.data_ptr(), None)
    dist.barrier()
    t = torch.from_file(path, shared=True, size=n, dtype=torch.uint8)
    digest = int(t.numpy().astype(np.uint64).sum())
    dg = [None] * world
    dist.all_gather_object(dg, digest)
    if rank == 0:
        out.put((all(d == dumps[0] for d in dumps), len(set(dg)) == 1, digest))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_plan_agreement_and_shared_host_image():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as tmp:
        ps = [ctx.Process(target=_worker, args=(r, 2, 29531, tmp, q)) for r in range(2)]
        for p in ps:
            p.start()
        same_plan, same_bytes, digest = q.get(timeout=300)
        for p in ps:
            p.join(timeout=60)
    assert same_plan and same_bytes
    import harness
    from paper_2503_17707_b200.api import Plan
    from synth.configs import WORKLOADS
    w = WORKLOADS["C1"]
    plan = Plan(w.model, w.adapters, 2, policy="interleave", vocab_sliced=1, chunk_bytes=64 << 10)
    buf = np.zeros(plan.sizes.host_base_bytes, dtype=np.uint8)
    harness.fill_host_images(plan, buf.ctypes.data, None)
    assert int(buf.astype(np.uint64).sum()) == digest
