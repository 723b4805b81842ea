"""compute-sanitizer target: one C1 cold start on 2 logical ranks of cuda:0 (device-side cross-rank readiness words,
peer copies, merges, pipelined prefill), checked against the oracle. PB_WAIT_TIMEOUT_S bounds a stall.

    PB_WAIT_TIMEOUT_S=120 compute-sanitizer --tool memcheck python tools/sanitize_2rank.py
"""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("PB_WAIT_TIMEOUT_S", "120")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import harness  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2503_17707_b200.api import Plan, RankEngine  # noqa: E402
from synth.configs import WORKLOADS  # noqa: E402

w = WORKLOADS["C1"]
plan = Plan(w.model, w.adapters, 2, policy="interleave", vocab_sliced=1, chunk_bytes=64 << 10, prefill_chunks=2)
base, ada = harness.build_host_images(plan)
toks = synth.tokens(w.batch, w.seq, w.model.vocab)
engs = [RankEngine(plan, r, base, ada, max_batch=w.batch, max_seq=w.seq) for r in range(2)]
for e in engs:
    e.wire_local(engs)
    e.invalidate()
for e in engs:
    e.enqueue(1, toks if e.rank == 0 else None, w.batch, w.seq, adapter_id=0)
tokens, logits = [e.wait(want_logits=True) for e in engs][0]
ol, ot = oracle.first_token_logits(w.model, w.adapters, toks, mode="bf16")
rel = float(np.abs(logits[0] - ol[0]).max() / np.abs(ol[0]).max())
for e in engs:
    e.close()
print(f"2-rank C1 cold start: token {int(tokens[0])} (oracle {int(ot[0])}), rel {rel:.2e}")
assert rel <= 1e-2
