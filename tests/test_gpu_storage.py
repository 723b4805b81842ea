"""f4 — storage tier: the cold start reads its base weights from a checkpoint FILE through a pinned staging ring
(pb_ctx_set_file_source) and must give exactly what the pinned-DRAM path gives: logits bit-identical, every
rank's weights byte-identical; small chunks force many groups through a 2-3 slot ring (slot reuse)."""
import os
import tempfile

import numpy as np
import pytest
import torch

import harness
import synth
from paper_2503_17707_b200 import _binding as B
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import TINY_LLAMA, TINY_OPT, lora
from gpu_util import need_gpu

pytestmark = pytest.mark.gpu


def cold(plan, base, ada, toks, path=None, staging=0):
    Bn, T = toks.shape
    engs = [RankEngine(plan, r, base, ada, max_batch=Bn, max_seq=T) for r in range(plan.n_gpus)]
    for e in engs:
        e.wire_local(engs)
        e.invalidate()
        if path:
            e.set_file_source(path, staging)
    for e in engs:
        e.enqueue(1, toks if e.rank == 0 else None, Bn, T, adapter_id=0)
    out = [e.wait(want_logits=True) for e in engs][0]
    return engs, out


@pytest.mark.parametrize("model", [TINY_OPT, TINY_LLAMA], ids=["opt", "llama"])
@pytest.mark.parametrize("n,policy", [(1, "stage"), (2, "interleave")])
def test_file_source_matches_pinned(model, n, policy):
    need_gpu()
    ads = (lora(8),)
    toks = synth.tokens(2, 20, model.vocab)
    plan = Plan(model, ads, n, policy=policy, vocab_sliced=1 if n > 1 else 0, chunk_bytes=16 << 10)
    base, ada = harness.build_host_images(plan)
    ref_engs, (t0, l0) = cold(plan, base, ada, toks)
    w0 = [e.weights.clone() for e in ref_engs]
    for e in ref_engs:
        e.close()
    with tempfile.NamedTemporaryFile(dir="/tmp", delete=False) as f:
        base.numpy().tofile(f)
        path = f.name
    try:
        slot = 8 << 20    # >= the largest copy group (chunks < 256 KiB coalesce: up to the whole 7 MB model)
        engs, (t1, l1) = cold(plan, base, ada, toks, path=path, staging=3 * slot)
        assert np.array_equal(l1.view(np.uint32), l0.view(np.uint32))
        assert np.array_equal(t1, t0)
        tens = plan.tensors()
        for e, w in zip(engs, w0):
            for (name, rows, cols, ho, layer, off) in tens:
                nb = rows * cols * 2
                assert torch.equal(e.weights[off:off + nb], w[off:off + nb]), (e.rank, name)
        for e in engs:
            e.close()
    finally:
        os.unlink(path)


def test_file_source_errors():
    need_gpu()
    plan = Plan(TINY_OPT, (lora(8),), 1, chunk_bytes=1 << 20)
    base, ada = harness.build_host_images(plan)
    e = RankEngine(plan, 0, base, ada, max_batch=1, max_seq=8)
    with pytest.raises(B.PBError) as ei:
        e.set_file_source("/nonexistent/checkpoint.bin", 64 << 20)
    assert ei.value.status == B.PB_EINVAL
    with tempfile.NamedTemporaryFile(dir="/tmp") as f:
        with pytest.raises(B.PBError) as ei:
            e.set_file_source(f.name, 4096)
        assert ei.value.status == B.PB_ENOMEM
    e.close()
