"""CPU oracle for the PipeBoost layer-sharded cold start.

TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's
``cpu_baseline`` leg (and ``bench.py --impl reference``) may import, call or
execute anything under oracle/. The product path (paper_2503_17707_b200) never
imports it and shares no code with it; the only shared module is ``synth`` (the
seeded input generator, which holds none of the method's arithmetic).

  O1 plan.py     — planner (partition, tensor table, load lists, receive lists)
  O2 merge.py    — correctly rounded merged-LoRA weights (fp64)
  O3 forward.py  — sequential OPT / Llama forward, modes 'exact' and 'bf16'
  O4 forward.py  — first token = argmax, lowest index on ties
  model.py       — on-demand weights (synth values -> merge)

Parity pins live in tests/test_oracle_*.py. Timing is "parity unpinned"
(hardware-specific).
"""
from __future__ import annotations

import numpy as np

from . import forward, merge, numerics, plan
from .model import OracleWeights


def first_token_logits(model, adapters, tokens_bt, adapter_of_seq=None, mode="bf16", host_alias_layers=0):
    """Logits [B, V] and tokens [B] for a batch (each sequence with its adapter)."""
    ow = OracleWeights(model, adapters, host_alias_layers)
    B = tokens_bt.shape[0]
    if adapter_of_seq is None:
        adapter_of_seq = [0 if adapters else None] * B
    cache = {}
    out = []
    for b in range(B):
        a = adapter_of_seq[b]

        def W(name, a=a):
            if name.startswith("L"):          # stream layer weights; cache only embed/head/norms
                return ow.get(name, a)
            key = (name, a)
            if key not in cache:
                cache[key] = ow.get(name, a)
            return cache[key]

        out.append(forward.forward_logits(model, W, np.asarray(tokens_bt[b]), mode))
    logits = np.stack(out)
    return logits, np.array([forward.first_token(x) for x in logits], dtype=np.int32)


def teacher_forced_logits(model, adapters, prompt_bt, generated_bt, mode="bf16", adapter=0):
    """f3 pins ("the first token is generated and returned ... to GPU 0"): decode step
    i of sequence b must produce exactly the logits of the plain forward over prompt[b] + generated[b, :i] — the
    definition a KV cache only accelerates. Returns [n + 1, B, V]: entry i uses the first i generated tokens
    (entry 0 = the prompt alone, i.e. the first-token prefill)."""
    B, n = generated_bt.shape
    out = []
    for i in range(n + 1):
        seqs = np.concatenate([prompt_bt, generated_bt[:, :i]], axis=1) if i else prompt_bt
        aos = [adapter if adapters else None] * B
        lg, _ = first_token_logits(model, adapters, seqs, adapter_of_seq=aos, mode=mode)
        out.append(lg)
    return np.stack(out)
