"""Isolate the C3 (Llama-2-7B, 4 adapters) parity gap: multi-adapter microbatches vs one in-place adapter,
one vs two stages, each against the stored oracle (tests/golden/oracle_C3.npz, sequence b uses adapter b)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import harness  # noqa: E402
from paper_2503_17707_b200 import _binding as B  # noqa: E402
from paper_2503_17707_b200.api import Plan, RankEngine  # noqa: E402
from synth.configs import LLAMA2_7B, lora  # noqa: E402

gold = harness.load_golden("C3")
toks = gold["tokens"]
ol = gold["logits_bf16"].astype(np.float64)


def run(ads, n, toks_b, adapter_id, aos=None, policy="stage", k=1):
    plan = Plan(LLAMA2_7B, ads, n, policy=policy, chunk_bytes=128 << 20, prefill_chunks=k)
    base, ada = harness.build_host_images(plan)
    Bn, T = toks_b.shape
    multi = adapter_id == B.PB_MERGE_ALL
    engs = [RankEngine(plan, r, base, ada, max_batch=Bn, max_seq=T, multi_adapter=multi) for r in range(n)]
    for e in engs:
        e.wire_local(engs)
        e.invalidate()
    for e in engs:
        e.enqueue(1, toks_b if e.rank == 0 else None, Bn, T, adapter_id=adapter_id, adapter_of_seq=aos)
    t, l = [e.wait(want_logits=True) for e in engs][0]
    for e in engs:
        e.close()
    del base, ada
    torch.cuda.empty_cache()
    return t, l


def rel(l, b):
    return float(np.abs(l.astype(np.float64) - ol[b]).max() / np.abs(ol[b]).max())


out = {}
t, l = run(tuple(lora(16) for _ in range(4)), 1, toks, B.PB_MERGE_ALL, aos=[0, 1, 2, 3])
out["multi_n1"] = [rel(l[b], b) for b in range(4)]
np.save("gpurun_out/c3_multi_n1.npy", l)
for a in range(2):
    ads = tuple(lora(16) for _ in range(a + 1))
    t, l = run(ads, 1, toks[a:a + 1], a)
    out[f"inplace_adapter{a}_n1"] = rel(l[0], a)
    np.save(f"gpurun_out/c3_inplace{a}.npy", l)
t, l = run(tuple(lora(16) for _ in range(4)), 2, toks, B.PB_MERGE_ALL, aos=[0, 1, 2, 3])
out["multi_n2"] = [rel(l[b], b) for b in range(4)]
print(json.dumps(out))
