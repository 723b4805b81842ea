"""f4 — storage tier: the cold start reads its base weights from a checkpoint FILE through a pinned staging ring
(pb_ctx_set_file_source) and must give exactly what the pinned-DRAM path gives: logits bit-identical, every
rank's weights byte-identical; small chunks force many groups through a 2-3 slot ring (slot reuse). The file-sourced
run is also checked against the oracle and the host bytes themselves: logits within 1e-2 of the bf16-contract
forward (G10 token rule), unadapted tensors equal to the checkpoint bytes, adapted tensors to the oracle merge."""
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
from checks import logits_vs_oracle, weights_vs_oracle

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
@pytest.mark.parametrize("n,policy,slots,readers", [(1, "stage", 3, None), (2, "interleave", 3, None),
                                                    (2, "interleave", 2, "16"), (1, "stage", 2, "7")])
def test_file_source_matches_pinned(model, n, policy, slots, readers, monkeypatch):
    """slots=2 with many reader threads: readers that finish their slice run ahead and must wait for their
    group's turn of a slot (storage.cpp Slot::turn) instead of writing into one still being filled / copied."""
    need_gpu()
    if readers:
        monkeypatch.setenv("PB_FILE_READERS", readers)
    monkeypatch.setenv("PB_FILE_SLOTS", str(slots))   # ring length (the slot size is the largest copy group)
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
        logits_vs_oracle(model, ads, toks, l1, t1)
        weights_vs_oracle(plan, engs[0].weights_bytes(), base.numpy(), model, ads)
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
