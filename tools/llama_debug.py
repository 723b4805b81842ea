"""Bisect a GPU-vs-oracle gap on Llama shapes: depth L and prompt length T sweeps at the Llama-2-7B width, each
cold start compared with the oracle computed on the spot (bf16-contract and exact modes)."""
import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import harness  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2503_17707_b200.api import Plan, RankEngine  # noqa: E402
from synth.configs import LLAMA2_7B, OPT_13B, lora  # noqa: E402


def run(model, ads, toks):
    plan = Plan(model, ads, 1, chunk_bytes=128 << 20)
    base, ada = harness.build_host_images(plan)
    Bn, T = toks.shape
    e = RankEngine(plan, 0, base, ada, max_batch=Bn, max_seq=T)
    e.invalidate()
    e.enqueue(1, toks, Bn, T, adapter_id=0 if ads else -1)
    t, l = e.wait(want_logits=True)
    e.close()
    return l


cases = [(LLAMA2_7B, 1, 16), (LLAMA2_7B, 1, 512), (LLAMA2_7B, 2, 512), (LLAMA2_7B, 4, 128), (LLAMA2_7B, 4, 512),
         (OPT_13B, 2, 512)]
for base_model, L, T in cases:
    m = dataclasses.replace(base_model, n_layers=L)
    ads = (lora(16),)
    toks = synth.tokens(1, T, m.vocab)
    g = run(m, ads, toks)[0].astype(np.float64)
    ob, _ = oracle.first_token_logits(m, ads, toks, mode="bf16")
    oe, _ = oracle.first_token_logits(m, ads, toks, mode="exact")
    ob, oe = ob[0], oe[0]
    r = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
    print(json.dumps({"arch": m.arch, "L": L, "T": T, "gpu_vs_bf16": r(g, ob), "gpu_vs_exact": r(g, oe),
                      "bf16_vs_exact": r(ob, oe)}), flush=True)
