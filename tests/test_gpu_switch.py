"""f2 — epoch-based adapter switching on the B200, through the C ABI.

A stage switches adapters by restoring the pristine base of its adapted tensors (saved by the cold start's
merges, or from the host image for chunks another rank loaded) and merging the new adapter in place, behind
the prefills already queued on it. Checks, for several adapters with different target sets, on 1 and 2
pipeline stages (STAGE and INTERLEAVE loading):
  * after switch(b) the next batch's logits are bit-identical to a cold start merged with b, and within 1e-2 of
    the oracle with b (so within the north-star gate);
  * switching back and forth never drifts: switch(a) after b gives a's cold-start logits bit for bit;
  * switch(-1) serves the base model;
  * the stage's weights after a switch are byte-identical to the cold start with that adapter.
"""
import numpy as np
import pytest
import torch

import harness
import oracle
import synth
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import TINY_LLAMA, TINY_OPT, lora
from gpu_util import need_gpu

pytestmark = pytest.mark.gpu


def engines(plan, base, ada, B, T):
    engs = [RankEngine(plan, r, base, ada, max_batch=B, max_seq=T, switchable=True) for r in range(plan.n_gpus)]
    for e in engs:
        e.wire_local(engs)
        e.invalidate()
    return engs


def cold(plan, base, ada, toks, adapter):
    B, T = toks.shape
    engs = engines(plan, base, ada, B, T)
    for e in engs:
        e.enqueue(1, toks if e.rank == 0 else None, B, T, adapter_id=adapter)
    out = [e.wait(want_logits=True) for e in engs][0]
    return engs, out


def stage_bytes(plan, eng, r):
    tens = plan.tensors()
    n = plan.n_gpus
    L = plan.model.n_layers
    a = r * (L // n) + min(r, L % n)
    b = a + L // n + (1 if r < L % n else 0)
    return [eng.weights[off:off + rows * cols * 2].clone() for (name, rows, cols, ho, layer, off) in tens
            if a <= layer < b]


@pytest.mark.parametrize("model", [TINY_OPT, TINY_LLAMA], ids=["opt", "llama"])
@pytest.mark.parametrize("n,policy", [(1, "stage"), (2, "stage"), (2, "interleave")])
def test_switch_adapters_no_drift(model, n, policy):
    need_gpu()
    if model.arch == "opt":
        ads = (lora(8, ("q", "v")), lora(8, ("q", "k", "o", "fc1")), lora(16, ("v",)))
    else:
        ads = (lora(8, ("q", "v")), lora(8, ("q", "k", "gate", "down")), lora(16, ("v",)))
    toks = synth.tokens(2, 20, model.vocab)
    plan = Plan(model, ads, n, policy=policy, chunk_bytes=64 << 10)
    base, ada = harness.build_host_images(plan)
    ref, ref_w = {}, {}
    for a in (-1, 0, 1, 2):                      # cold starts with each adapter (and none)
        engs, (t, l) = cold(plan, base, ada, toks, a)
        ref[a] = (t, l)
        ref_w[a] = [stage_bytes(plan, e, e.rank) for e in engs]
        for e in engs:
            e.close()
    for a in (0, 1, 2):
        ol, _ = oracle.first_token_logits(model, ads, toks, adapter_of_seq=[a, a], mode="bf16")
        assert np.abs(ref[a][1] - ol).max() / np.abs(ol).max() <= 1e-2
    engs, (t0, l0) = cold(plan, base, ada, toks, 0)
    epoch = 2
    for a in (1, 2, 0, -1, 1, 0):
        for e in engs:
            e.switch_adapter(a)
        for e in engs:
            e.replay_enqueue(epoch, toks if e.rank == 0 else None, 2, 20)
        t, l = [e.wait(want_logits=True) for e in engs][0]
        epoch += 1
        assert np.array_equal(l.view(np.uint32), ref[a][1].view(np.uint32)), a
        assert np.array_equal(t, ref[a][0])
        for e in engs:
            got = stage_bytes(plan, e, e.rank)
            assert all(torch.equal(x, y) for x, y in zip(got, ref_w[a][e.rank])), (a, e.rank)
    for e in engs:
        e.close()


def test_switch_errors():
    need_gpu()
    from paper_2503_17707_b200 import _binding as B
    model, ads = TINY_OPT, (lora(8), lora(8))
    plan = Plan(model, ads, 1)
    base, ada = harness.build_host_images(plan)
    e = RankEngine(plan, 0, base, ada, max_batch=1, max_seq=8)     # no backup buffer
    with pytest.raises(B.PBError) as ei:
        e.switch_adapter(1)
    assert ei.value.status == B.PB_EPROTOCOL                       # no cold start yet
    e.wire_local([e])
    e.cold_start(1, synth.tokens(1, 8, model.vocab))
    with pytest.raises(B.PBError) as ei:
        e.switch_adapter(1)
    assert ei.value.status == B.PB_ENOMEM
    e.close()
