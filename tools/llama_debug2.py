"""Where does the GPU leave the storage contract on a Llama-2-7B-width layer? Saves the GPU logits of 1-layer
cold starts (T = 16 / 512) and reports the bit-exact fraction of the merged q|k|v weights against the oracle's
correctly rounded merge."""
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
from oracle.numerics import bf16_bits_to_f64  # noqa: E402
from paper_2503_17707_b200.api import Plan, RankEngine  # noqa: E402
from synth.configs import LLAMA2_7B, lora  # noqa: E402

os.makedirs("gpurun_out/dbg", exist_ok=True)
for L, T in ((1, 16), (1, 512)):
    m = dataclasses.replace(LLAMA2_7B, n_layers=L)
    ads = (lora(16),)
    toks = synth.tokens(1, T, m.vocab)
    plan = Plan(m, ads, 1, chunk_bytes=128 << 20)
    base, ada = harness.build_host_images(plan)
    e = RankEngine(plan, 0, base, ada, max_batch=1, max_seq=T)
    e.invalidate()
    e.enqueue(1, toks, 1, T, adapter_id=0)
    t, lg = e.wait(want_logits=True)
    np.save(f"gpurun_out/dbg/llama7b_L{L}_T{T}.npy", lg)
    if T == 16:
        w = e.weights_bytes()
        ow = oracle.OracleWeights(m, ads)
        for (name, rows, cols, ho, layer, off) in plan.tensors():
            if name == "L0.qkv":
                g = w[off:off + rows * cols * 2].view(np.uint16).reshape(rows, cols)
                o = ow.merged_bits(name, 0)
                q = slice(0, 4096)
                v = slice(8192, 12288)
                print(json.dumps({"tensor": name, "exact_q": float((g[q] == o[q]).mean()),
                                  "exact_v": float((g[v] == o[v]).mean()), "exact_k": float((g[4096:8192] == o[4096:8192]).mean())}))
    e.close()
print("saved")
