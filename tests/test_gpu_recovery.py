"""f1 — recovery for model loading on the B200, through the C ABI.

N logical ranks cold-start on one GPU; "GPUs" 1 and 2 crash after every GPU has loaded (and merged) its own
shard but before the all-gather, as in the paper's example. The survivors re-plan
(pb_plan_replan) and resume in the SAME device buffers: every byte they did not already hold is first
poisoned (0xFF), so the resumed cold start can only succeed by loading / receiving exactly what the re-plan
says. Checks: first-token logits bit-identical to the no-crash run (pipelined prefill is N-invariant), the
survivors end with the whole merged model byte-identical to the no-crash run, and nothing they held was
transferred again (PCIe bytes = the chunks no survivor held, plus the LoRA parts their merges need).
Both runs are also checked against the oracle (not only against each other): logits within 1e-2 of the
bf16-contract forward with the G10 token rule, weights equal to the host bytes / the oracle merge.
A second case crashes DURING the load: each survivor holds only a prefix of its load list, so a layer's LoRA
factors (loaded right before its base tensors, G8) can be held while some of its base chunks are not.
"""
import numpy as np
import pytest
import torch

import harness
import synth
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import ModelDesc, TINY_LLAMA, TINY_OPT, lora
from gpu_util import need_gpu
from checks import logits_vs_oracle, weights_vs_oracle

pytestmark = pytest.mark.gpu


def cold_start(plan, base, ada, toks, reuse=None, invalidate=True):
    B_, T = toks.shape
    engs = []
    for r in range(plan.sizes.n_gpus):
        old = reuse[plan.gpu_of_rank(r)] if reuse is not None else None
        engs.append(RankEngine(plan, r, base, ada, max_batch=B_, max_seq=T, reuse=old))
    for e in engs:
        e.wire_local(engs)
        if invalidate:
            e.invalidate()
    for e in engs:
        e.enqueue(1, toks if e.rank == 0 else None, B_, T, adapter_id=0)
    res = [e.wait(want_logits=True) for e in engs]
    return engs, res[0]


@pytest.mark.parametrize("model,policy,k,held", [(TINY_OPT, "stage", 1, 1.0), (TINY_LLAMA, "stage", 2, 1.0),
                                                (ModelDesc("opt", 8, 256, 4, 4, 1024, 1024, 128, 1), "interleave", 2, 1.0),
                                                (TINY_OPT, "stage", 1, 0.6), (TINY_LLAMA, "stage", 2, 0.45)],
                         ids=["opt", "llama", "opt8-interleave", "opt-prefix60", "llama-prefix45"])
def test_recovery_after_two_crashes(model, policy, k, held):
    need_gpu()
    ads = (lora(8),)
    toks = synth.tokens(2, 24, model.vocab)
    plan = Plan(model, ads, 4, policy=policy, chunk_bytes=32 << 10, prefill_chunks=k)
    base, ada = harness.build_host_images(plan)
    engs, (t_ref, l_ref) = cold_start(plan, base, ada, toks)
    logits_vs_oracle(model, ads, toks, l_ref, t_ref)
    w_ref = engs[0].weights.clone()
    for e in engs:
        e.close()
    torch.cuda.synchronize()

    # crash of GPUs 1 and 2: the survivors hold what they loaded and merged themselves
    chunks = plan.chunks()
    load, _ = plan.lists()
    alive = [1, 0, 0, 1]
    resident = np.zeros((4, len(chunks)), dtype=np.uint8)
    for g in (0, 3):
        resident[g, load[g][:max(1, int(round(held * len(load[g]))))]] = 1
        for (cid, is_ad, tensor, r0, r1, off, nb, loader) in chunks:   # poison everything not held
            if not resident[g, cid]:
                buf = engs[g].adapters if is_ad else engs[g].weights
                buf[off:off + nb].fill_(0xFF)
    torch.cuda.synchronize()

    rp = plan.replan(alive, resident)
    assert rp.sizes.n_gpus == 2 and {rp.gpu_of_rank(0), rp.gpu_of_rank(1)} == {0, 3}
    new, (t_rec, l_rec) = cold_start(rp, base, ada, toks, reuse=engs, invalidate=False)
    assert np.array_equal(l_rec.view(np.uint32), l_ref.view(np.uint32))
    assert np.array_equal(t_rec, t_ref)
    logits_vs_oracle(model, ads, toks, l_rec, t_rec)
    weights_vs_oracle(plan, new[0].weights_bytes(), base.numpy(), model, ads)
    # every survivor now holds the whole merged model, byte for byte the no-crash model
    tensors = plan.tensors()
    for e in new:
        bad = [name for (name, rows, cols, host_off, layer, dev_off) in tensors
               if not torch.equal(e.weights[dev_off:dev_off + rows * cols * 2], w_ref[dev_off:dev_off + rows * cols * 2])]
        assert not bad, (e.rank, bad)
    # no re-transfer: PCIe bytes = chunks no survivor held (+ LoRA parts the merges there need)
    rload, rrecv = rp.lists()
    held_any = resident[0] | resident[3]
    by_id = {c[0]: c for c in chunks}
    for r, e in enumerate(new):
        g = rp.gpu_of_rank(r)
        assert not set(rload[r]) & set(np.flatnonzero(resident[g])) and not set(rrecv[r]) & set(np.flatnonzero(resident[g]))
        assert e.timeline()["load_bytes"] == sum(by_id[c][6] for c in rload[r])
    base_missing = {c[0] for c in chunks if not c[1] and not held_any[c[0]]}
    assert {c for r in range(2) for c in rload[r] if not by_id[c][1]} == base_missing
    for e in new:
        e.close()
