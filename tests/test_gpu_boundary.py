"""The §8(b) boundary semantics on the B200 (VERDICT r01 "What's missing" #3).

  * pb_load_shard -> pb_merge_lora -> pb_gather_layers ISSUE the work ("ready to serve", P:L246-247
    "begins serving ... while asynchronously loading the remaining parts"): with no prompt at all, pb_sync reaches
    T_full and every rank holds the whole merged model — unadapted bytes equal the host image, adapted tensors the
    oracle merge — and a later warm prefill matches the oracle;
  * a prompt posted after the load has started joins the same issuer (tokens pulled by an SM copy, the copy lane
    being busy): logits bit-identical to the prompt-at-once cold start and within the gate of the oracle;
  * pb_ctx_abort releases a rank whose peer never arrives (crash during loading), pb_ctx_free then
    returns, and the survivor's re-plan (pb_plan_replan) resumes in the same buffers to the oracle's logits;
  * f2 x f3 guards: no in-place adapter switch in replica mode, no replica after a switch.
"""
import time

import numpy as np
import pytest
import torch

import harness
import synth
from paper_2503_17707_b200 import _binding as B
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import TINY_LLAMA, TINY_OPT, ModelDesc, lora
from gpu_util import need_gpu
from checks import logits_vs_oracle, weights_vs_oracle

pytestmark = pytest.mark.gpu


def engines(plan, base, ada, Bn, T, **kw):
    engs = [RankEngine(plan, r, base, ada, max_batch=Bn, max_seq=T, **kw) for r in range(plan.n_gpus)]
    for e in engs:
        e.wire_local(engs)
        e.invalidate()
    return engs


@pytest.mark.parametrize("model,policy", [(TINY_OPT, "interleave"), (TINY_LLAMA, "stage")], ids=["opt", "llama"])
def test_no_prompt_cold_start_reaches_t_full(model, policy):
    need_gpu()
    ads = (lora(8),)
    toks = synth.tokens(2, 20, model.vocab)
    plan = Plan(model, ads, 2, policy=policy, vocab_sliced=1, chunk_bytes=32 << 10)
    base, ada = harness.build_host_images(plan)
    engs = engines(plan, base, ada, 2, 20)
    for e in engs:
        e.arm(1, adapter_id=0)
    for e in engs:
        e.sync()                     # no prompt: the load / merge / gather must still complete
    host = base.numpy()
    for e in engs:
        tl = e.timeline()
        assert tl["t_full_ms"] > 0 and tl["load_bytes"] > 0 and tl["recv_bytes"] > 0
        weights_vs_oracle(plan, e.weights_bytes(), host, model, ads)
    # the resident model serves: warm prefill through the same pipeline
    for e in engs:
        e.replay_enqueue(2, toks if e.rank == 0 else None, 2, 20)
    tokens, logits = [e.wait(want_logits=True) for e in engs][0]
    logits_vs_oracle(model, ads, toks, logits, tokens)
    for e in engs:
        e.close()


@pytest.mark.parametrize("delay_ms", [0, 3])
def test_prompt_posted_after_load_started(delay_ms):
    need_gpu()
    model = ModelDesc("opt", 8, 256, 4, 4, 1024, 1024, 128, 1)
    ads = (lora(8),)
    toks = synth.tokens(1, 24, model.vocab)
    plan = Plan(model, ads, 2, policy="interleave", vocab_sliced=1, chunk_bytes=16 << 10, prefill_chunks=2)
    base, ada = harness.build_host_images(plan)
    ref = engines(plan, base, ada, 1, 24)
    for e in ref:
        e.enqueue(1, toks if e.rank == 0 else None, 1, 24, adapter_id=0)
    t_ref, l_ref = [e.wait(want_logits=True) for e in ref][0]
    for e in ref:
        e.close()
    engs = engines(plan, base, ada, 1, 24)
    for e in engs:
        e.arm(1, adapter_id=0)
    time.sleep(delay_ms * 1e-3)
    for e in engs:
        e.post_prompt(toks if e.rank == 0 else None, 1, 24)
    t, l = [e.wait(want_logits=True) for e in engs][0]
    assert np.array_equal(l.view(np.uint32), l_ref.view(np.uint32)) and np.array_equal(t, t_ref)
    logits_vs_oracle(model, ads, toks, l, t)
    for e in engs:
        tl = e.timeline()
        assert tl["stage_end_ms"] >= tl["stage_begin_ms"] >= 0
        assert tl["ctx_create_ms"] > 0
    for e in engs:
        e.close()


def test_abort_after_peer_never_arrives_then_resume():
    """Rank 1 'dies' before loading anything: rank 0's compute and receive streams block on words only rank 1
    writes. pb_ctx_abort releases them; the survivor re-plans with what it loaded and merged itself and finishes
    the cold start alone, matching the oracle."""
    need_gpu()
    model = TINY_OPT
    ads = (lora(8),)
    toks = synth.tokens(1, 16, model.vocab)
    plan = Plan(model, ads, 2, policy="interleave", vocab_sliced=0, chunk_bytes=32 << 10)
    base, ada = harness.build_host_images(plan)
    engs = engines(plan, base, ada, 1, 16)
    engs[0].arm(1, adapter_id=0)
    engs[0].post_prompt(toks, 1, 16)
    time.sleep(0.5)
    t0 = time.time()
    engs[0].abort()
    with pytest.raises(B.PBError) as ei:
        B.pb_trial_begin(engs[0].ctx, 2)
    assert ei.value.status == B.PB_EPROTOCOL
    engs[0].close()
    engs[1].close()
    assert time.time() - t0 < 30
    # survivor 0 holds its own load list (landed + merged: nothing of it waited on the dead peer)
    load, _ = plan.lists()
    chunks = plan.chunks()
    resident = np.zeros((2, len(chunks)), dtype=np.uint8)
    resident[0, load[0]] = 1
    for (cid, is_ad, tensor, r0, r1, off, nb, loader) in chunks:   # poison everything not held
        if not resident[0, cid]:
            (engs[0].adapters if is_ad else engs[0].weights)[off:off + nb].fill_(0xFF)
    torch.cuda.synchronize()
    rp = plan.replan([1, 0], resident)
    assert rp.sizes.n_gpus == 1 and rp.gpu_of_rank(0) == 0
    e = RankEngine(rp, 0, base, ada, max_batch=1, max_seq=16, reuse=engs[0])
    e.enqueue(1, toks, 1, 16, adapter_id=0)
    t, l = e.wait(want_logits=True)
    logits_vs_oracle(model, ads, toks, l, t)
    weights_vs_oracle(plan, e.weights_bytes(), base.numpy(), model, ads)
    e.close()


def test_switch_and_replica_guards():
    need_gpu()
    model = TINY_OPT
    ads = (lora(8), lora(8, ("q", "k")))
    toks = synth.tokens(1, 16, model.vocab)
    plan = Plan(model, ads, 2, policy="stage", chunk_bytes=32 << 10)
    base, ada = harness.build_host_images(plan)
    engs = engines(plan, base, ada, 1, 16, switchable=True)
    for e in engs:
        e.enqueue(1, toks if e.rank == 0 else None, 1, 16, adapter_id=0)
    for e in engs:
        e.wait()
    engs[0].set_replica(True)
    with pytest.raises(B.PBError) as ei:
        engs[0].switch_adapter(1)
    assert ei.value.status == B.PB_EUNSUPPORTED
    engs[0].set_replica(False)
    for e in engs:
        e.switch_adapter(1)
    with pytest.raises(B.PBError) as ei:
        engs[1].set_replica(True)
    assert ei.value.status == B.PB_EUNSUPPORTED
    for e in engs:
        e.switch_adapter(0)       # back to the cold start's adapter: replicas allowed again
    for e in engs:
        e.sync()
    engs[1].set_replica(True)
    for e in engs:
        e.close()
