#!/usr/bin/env python
"""How far apart can two correct implementations of the SAME storage contract be? (DESIGN.md §3 reading R1.)

The oracle's bf16 mode rounds at the contract's points with fp64 arithmetic in between; the GPU rounds at the same
points with fp32 accumulation in between. This tool (analysis only; imports oracle/ and synth/, never the product
path) runs, on the seeded Llama-2-7B-shaped model truncated to its first L layers:
  exact    : oracle fp64 forward (no storage rounding)
  contract : oracle 'bf16' mode (fp64 between the rounding points)
  c32      : the same contract with every product accumulated in fp32 (operands cast to float32 before each
             matmul / attention product — the GPU's arithmetic between the rounding points)
and prints rel(contract, exact) and rel(c32, contract) (||a-b||inf / ||b||inf over the last position's logits) as L
grows. If rel(c32, contract) tracks rel(contract, exact), the spread is the model's sensitivity to sub-ulp rounding
differences, not an error of either implementation.

    python tools/contract_sensitivity.py --layers 1,2,4,8,16,32 --seq 128
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import forward as OF  # noqa: E402
from oracle.numerics import bf16_bits_to_f64, rne_bf16, rne_f32  # noqa: E402
from synth.configs import WORKLOADS  # noqa: E402


def mm32(a, b):
    return (np.asarray(a, dtype=np.float32) @ np.asarray(b, dtype=np.float32)).astype(np.float64)


def attention32(q, k, v, H, KVH, hd, scale, R):
    T = q.shape[0]
    g = H // KVH
    out = np.zeros((T, H * hd))
    mask = np.triu(np.ones((T, T), dtype=bool), k=1)
    for h in range(H):
        kv = h // g
        S = mm32(q[:, h * hd:(h + 1) * hd], k[:, kv * hd:(kv + 1) * hd].T) * scale
        S = np.where(mask, -np.inf, S)
        S = S - S.max(axis=-1, keepdims=True)
        E = np.exp(S)
        P = R(E / E.sum(axis=-1, keepdims=True))
        out[:, h * hd:(h + 1) * hd] = mm32(P, v[:, kv * hd:(kv + 1) * hd])
    return out


def llama_c32(m, W, toks, layers):
    """The contract (oracle/forward.py 'bf16' rounding points) with fp32 accumulation of every product."""
    R, F = rne_bf16, rne_f32
    d, H, KVH, hd, f = m.d_model, m.n_heads, m.n_kv_heads, m.head_dim, m.d_ffn
    qd, kvd = H * hd, KVH * hd
    h = F(W("embed")[toks].copy())
    for l in layers:
        p = f"L{l}."
        x = R(OF.rms_norm(h, W(p + "ln1_g"), m.norm_eps))
        qkv = mm32(x, W(p + "qkv").T)
        q = R(OF.rope(qkv[:, :qd], H, hd, m.rope_theta))
        k = R(OF.rope(qkv[:, qd:qd + kvd], KVH, hd, m.rope_theta))
        v = R(qkv[:, qd + kvd:])
        a = R(attention32(q, k, v, H, KVH, hd, hd ** -0.5, R))
        h = F(h + mm32(a, W(p + "o").T))
        x = R(OF.rms_norm(h, W(p + "ln2_g"), m.norm_eps))
        gu = mm32(x, W(p + "gate_up").T)
        g, u = gu[:, :f], gu[:, f:]
        h = F(h + mm32(R(g / (1.0 + np.exp(-g)) * u), W(p + "down").T))
    y = R(OF.rms_norm(h[-1], W("final_g"), m.norm_eps))
    return F(mm32(W("lm_head"), y))


def opt_c32(m, W, toks, layers):
    """OPT (pre-LN, biases, learned positions, ReLU, tied head) under the contract with fp32 accumulation."""
    R, F = rne_bf16, rne_f32
    d, H, hd = m.d_model, m.n_heads, m.head_dim
    T = len(toks)
    h = F(W("embed")[toks] + W("pos")[np.arange(T) + 2])
    for l in layers:
        p = f"L{l}."
        x = R(OF.layer_norm(h, W(p + "ln1_g"), W(p + "ln1_b"), m.norm_eps))
        qkv = mm32(x, W(p + "qkv").T) + W(p + "qkv_b")
        q = R(qkv[:, :d] * hd ** -0.5)
        k = R(qkv[:, d:2 * d])
        v = R(qkv[:, 2 * d:])
        a = R(attention32(q, k, v, H, H, hd, 1.0, R))
        h = F(h + mm32(a, W(p + "o").T) + W(p + "o_b"))
        x = R(OF.layer_norm(h, W(p + "ln2_g"), W(p + "ln2_b"), m.norm_eps))
        u = R(np.maximum(mm32(x, W(p + "fc1").T) + W(p + "fc1_b"), 0.0))
        h = F(h + mm32(u, W(p + "fc2").T) + W(p + "fc2_b"))
    y = R(OF.layer_norm(h[-1], W("final_g"), W("final_b"), m.norm_eps))
    return F(mm32(W("embed"), y))


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--layers", default="1,2,4,8,16,32")
    ap.add_argument("--seq", type=int, default=128)
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    for L in [int(x) for x in args.layers.split(",")]:
        m = dataclasses.replace(w.model, n_layers=L)
        ow = oracle.OracleWeights(m, w.adapters)
        cache = {}   # merged bf16 BITS (2 B / element; fp64 copies are made per use)

        def W(name):
            if name not in cache:
                cache[name] = ow.merged_bits(name, 0)
            x = bf16_bits_to_f64(cache[name])
            return x.reshape(-1) if ow.tensors[name].rows == 1 else x

        toks = synth.tokens(1, args.seq, m.vocab)[0]
        ex = OF.forward_logits(m, W, toks, "exact")
        con = OF.forward_logits(m, W, toks, "bf16")
        c32 = (llama_c32 if m.arch == "llama" else opt_c32)(m, W, toks, range(L))
        print(json.dumps({"workload": args.workload, "layers": L, "seq": args.seq,
                          "rel_contract_vs_exact": rel(con, ex), "rel_c32_vs_contract": rel(c32, con),
                          "rel_c32_vs_exact": rel(c32, ex), "argmax": [int(np.argmax(x)) for x in (ex, con, c32)]}),
              flush=True)
        cache.clear()


if __name__ == "__main__":
    main()
