"""f3 — pipelined decode and the switch to single-GPU replicas on the B200, through the C ABI.

Checks:
  * every decode step's logits equal the oracle's plain forward over prompt + the tokens generated so far (the
    KV cache only accelerates that definition) within 1e-2, with the G10 argmax rule;
  * decode is pipeline-invariant: logits bit-identical for 1 and 2 stages (interleaved loading, vocab slices,
    prompt chunks);
  * after T_full each GPU serves its own NEW batch alone (replica mode, "batches ... submitted after the
    switching point"): prefill + decode logits bit-identical to the same batch on a single-GPU pipeline.
"""
import numpy as np
import pytest

import harness
import oracle
import synth
from paper_2503_17707_b200 import _binding as B
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import TINY_LLAMA, TINY_OPT, lora
from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
STEPS = 5


def start(model, ads, n, toks, policy="stage", sliced=0, k=1, max_seq=40):
    plan = Plan(model, ads, n, policy=policy, vocab_sliced=sliced, chunk_bytes=64 << 10, prefill_chunks=k)
    base, ada = harness.build_host_images(plan)
    Bn, T = toks.shape
    engs = [RankEngine(plan, r, base, ada, max_batch=4, max_seq=max_seq) for r in range(n)]
    for e in engs:
        e.wire_local(engs)
        e.invalidate()
    for e in engs:
        e.enqueue(1, toks if e.rank == 0 else None, Bn, T, adapter_id=0)
    first = [e.wait(want_logits=True) for e in engs][0]
    return engs, first


def decode(engs, steps, epoch0):
    toks, logits = [], []
    for i in range(steps):
        for e in engs:
            e.decode_enqueue(epoch0 + i)
        t, l = [e.wait(want_logits=True) for e in engs][0]
        toks.append(t)
        logits.append(l)
    return np.stack(toks, axis=1), np.stack(logits)


def check_oracle(model, ads, prompt, first, gen, logits):
    """gen [B, steps] GPU tokens; logits [steps, B, V]. Step 0 = the first token (prefill)."""
    allgen = np.concatenate([first[0][:, None], gen], axis=1)      # tokens fed to steps 1.. (teacher forcing)
    ol = oracle.teacher_forced_logits(model, ads, prompt, allgen[:, :-1], mode="bf16")
    gl = np.concatenate([first[1][None], logits], axis=0)
    for i in range(gl.shape[0]):
        for b in range(prompt.shape[0]):
            err = np.abs(gl[i, b].astype(np.float64) - ol[i, b]).max()
            assert err / np.abs(ol[i, b]).max() <= 1e-2, (i, b)
            srt = np.sort(ol[i, b])
            tok = allgen[b, i]
            assert tok == int(np.argmax(ol[i, b])) or ol[i, b][tok] >= srt[-1] - 2 * err, (i, b)


@pytest.mark.parametrize("model", [TINY_OPT, TINY_LLAMA], ids=["opt", "llama"])
def test_pipelined_decode_matches_oracle_and_is_n_invariant(model):
    need_gpu()
    ads = (lora(8),)
    prompt = synth.tokens(2, 17, model.vocab)
    ref = None
    for n, policy, sliced, k in [(1, "stage", 0, 1), (2, "interleave", 1, 2)]:
        engs, first = start(model, ads, n, prompt, policy, sliced, k)
        gen, logits = decode(engs, STEPS, 2)
        if ref is None:
            check_oracle(model, ads, prompt, first, gen, logits)
            ref = (first[1], gen, logits)
        else:
            assert np.array_equal(first[1].view(np.uint32), ref[0].view(np.uint32))
            assert np.array_equal(gen, ref[1])
            assert np.array_equal(logits.view(np.uint32), ref[2].view(np.uint32))
        for e in engs:
            e.close()


@pytest.mark.parametrize("model", [TINY_OPT, TINY_LLAMA], ids=["opt", "llama"])
def test_replicas_after_tfull(model):
    need_gpu()
    ads = (lora(8),)
    prompt0 = synth.tokens(1, 16, model.vocab)
    X = synth.tokens(3, 20, model.vocab)[1:]        # two new batches, one per GPU
    Y = synth.tokens(4, 11, model.vocab)[2:]
    want = {}
    for name, batch in (("X", X), ("Y", Y)):          # the same batches on a single-GPU pipeline
        engs, first = start(model, ads, 1, batch)
        gen, logits = decode(engs, STEPS, 2)
        want[name] = (first[1], gen, logits)
        engs[0].close()
    engs, _ = start(model, ads, 2, prompt0, policy="interleave", sliced=1, k=2)
    for e in engs:
        e.set_replica(True)
    for e, batch in zip(engs, (X, Y)):
        e.replay_enqueue(2, batch, batch.shape[0], batch.shape[1])
    firsts = [e.wait(want_logits=True) for e in engs]
    outs = [[], []]
    for i in range(STEPS):
        for e in engs:
            e.decode_enqueue(3 + i)
        for r, e in enumerate(engs):
            outs[r].append(e.wait(want_logits=True))
    for r, name in enumerate(("X", "Y")):
        f, g, l = want[name]
        assert np.array_equal(firsts[r][1].view(np.uint32), f.view(np.uint32)), name
        assert np.array_equal(np.stack([o[0] for o in outs[r]], axis=1), g), name
        assert np.array_equal(np.stack([o[1] for o in outs[r]]).view(np.uint32), l.view(np.uint32)), name
    for e in engs:
        e.close()


def test_decode_errors():
    need_gpu()
    model, ads = TINY_OPT, (lora(8),)
    prompt = synth.tokens(1, 16, model.vocab)
    plan = Plan(model, ads, 1)
    base, ada = harness.build_host_images(plan)
    e = RankEngine(plan, 0, base, ada, max_batch=1, max_seq=17)
    e.wire_local([e])
    with pytest.raises(B.PBError) as ei:
        e.decode_enqueue(1)
    assert ei.value.status == B.PB_EPROTOCOL
    e.cold_start(1, prompt)
    e.decode_enqueue(2)
    e.wait()
    with pytest.raises(B.PBError) as ei:           # position 17 would exceed max_seq = 17
        e.decode_enqueue(3)
    assert ei.value.status == B.PB_EINVAL
    e.set_replica(True)
    with pytest.raises(B.PBError) as ei:           # prefilled in pipeline mode: prefill again as a replica first
        e.decode_enqueue(4)
    assert ei.value.status == B.PB_EPROTOCOL
    e.close()
