"""O3/O4 — sequential first-token forward pass (TEST INFRASTRUCTURE ONLY; see oracle/plan.py).

What this computes: the plain, whole-model, one-device
forward of an OPT (HF ``do_layer_norm_before=True``) or Llama decoder over a
prompt, then the first token = argmax of the last position's logits.
The paper builds on HF Transformers and describes prefill as
"each layer ... self-attention ... Then ... a feed-forward network ... The final
layer of the model generates the first token". PipeBoost's pipelined
prefill must reach exactly this result (stages only move where the
layers run), so the oracle is N-agnostic by construction.

Modes
  'exact': fp64 everywhere (the weights are bf16 values, nothing else rounds).
  'bf16' : the storage-precision contract: fp64 arithmetic, with
           a single rounding at every storage point — norm outputs, q/k/v (after
           bias/scale/RoPE), attention probabilities P, attention output, MLP
           hidden -> bf16 (RNE); residual stream h and logits -> fp32.
  'f32'  : the fp32 debug-parity contract (PB_DTYPE_F32 models): the same storage
           points, every one rounded RNE to fp32.

Layer-by-layer loops over heads in plain numpy; no blocking, no fusion.
"""
from __future__ import annotations

import numpy as np

from .numerics import rne_bf16, rne_f32


def _rounders(mode):
    if mode == "exact":
        ident = lambda x: x
        return ident, ident
    if mode == "bf16":
        return rne_bf16, rne_f32
    if mode == "f32":
        return rne_f32, rne_f32
    raise ValueError(mode)


def layer_norm(x, g, b, eps):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def rms_norm(x, g, eps):
    return x / np.sqrt((x * x).mean(axis=-1, keepdims=True) + eps) * g


def causal_attention(q, k, v, n_heads, n_kv_heads, head_dim, score_scale, R):
    """q [T, H*hd], k/v [T, KVH*hd] -> [T, H*hd]. Per head: S = q k^T * scale,
    mask j > i, P = softmax(S) (rounded by R), a = P v."""
    T = q.shape[0]
    group = n_heads // n_kv_heads
    out = np.zeros((T, n_heads * head_dim))
    mask = np.triu(np.ones((T, T), dtype=bool), k=1)
    for h in range(n_heads):
        kv = h // group
        qh = q[:, h * head_dim:(h + 1) * head_dim]
        kh = k[:, kv * head_dim:(kv + 1) * head_dim]
        vh = v[:, kv * head_dim:(kv + 1) * head_dim]
        S = (qh @ kh.T) * score_scale
        S = np.where(mask, -np.inf, S)
        S = S - S.max(axis=-1, keepdims=True)
        E = np.exp(S)
        Pm = R(E / E.sum(axis=-1, keepdims=True))
        out[:, h * head_dim:(h + 1) * head_dim] = Pm @ vh
    return out


def rope(x, n_heads, head_dim, theta):
    """HF rotate_half RoPE (modeling_llama.py): for i < hd/2,
    x'_i = x_i cos(t w_i) - x_{i+hd/2} sin(t w_i), x'_{i+hd/2} = x_{i+hd/2} cos + x_i sin,
    w_i = theta^(-2i/hd), positions t = 0..T-1."""
    T = x.shape[0]
    half = head_dim // 2
    inv_freq = theta ** (-(2.0 * np.arange(half)) / head_dim)
    ang = np.arange(T)[:, None] * inv_freq[None, :]
    c, s = np.cos(ang), np.sin(ang)
    y = x.copy()
    for h in range(n_heads):
        a = x[:, h * head_dim:h * head_dim + half]
        b = x[:, h * head_dim + half:(h + 1) * head_dim]
        y[:, h * head_dim:h * head_dim + half] = a * c - b * s
        y[:, h * head_dim + half:(h + 1) * head_dim] = b * c + a * s
    return y


def forward_logits(m, W, tokens, mode="exact", layers=None, return_hidden=False):
    """Logits [V] of the last position of ONE sequence.

    m: ModelDesc; W(name) -> fp64 array of the (merged) tensor; tokens: [T] ints.
    layers: optional iterable restricting the decoder layers run (for the
    extrapolated CPU baseline); default all.
    """
    R, F = _rounders(mode)
    T = len(tokens)
    d, H, KVH, hd, f = m.d_model, m.n_heads, m.n_kv_heads, m.head_dim, m.d_ffn
    E = W("embed")
    if m.arch == "opt":
        pos = W("pos")
        h = F(E[tokens] + pos[np.arange(T) + 2])          # HF OPT learned positions, offset 2
    else:
        h = F(E[tokens].copy())
    for l in (range(m.n_layers) if layers is None else layers):
        p = f"L{l}."
        if m.arch == "opt":
            x = R(layer_norm(h, W(p + "ln1_g"), W(p + "ln1_b"), m.norm_eps))
            qkv = x @ W(p + "qkv").T + W(p + "qkv_b")
            q = R(qkv[:, :d] * hd ** -0.5)               # HF OPT scales q after the bias
            k = R(qkv[:, d:2 * d])
            v = R(qkv[:, 2 * d:])
            a = R(causal_attention(q, k, v, H, H, hd, 1.0, R))
            h = F(h + a @ W(p + "o").T + W(p + "o_b"))
            x = R(layer_norm(h, W(p + "ln2_g"), W(p + "ln2_b"), m.norm_eps))
            u = R(np.maximum(x @ W(p + "fc1").T + W(p + "fc1_b"), 0.0))
            h = F(h + u @ W(p + "fc2").T + W(p + "fc2_b"))
        else:
            qd, kvd = H * hd, KVH * hd
            x = R(rms_norm(h, W(p + "ln1_g"), m.norm_eps))
            qkv = x @ W(p + "qkv").T
            q = R(rope(qkv[:, :qd], H, hd, m.rope_theta))
            k = R(rope(qkv[:, qd:qd + kvd], KVH, hd, m.rope_theta))
            v = R(qkv[:, qd + kvd:])
            a = R(causal_attention(q, k, v, H, KVH, hd, hd ** -0.5, R))
            h = F(h + a @ W(p + "o").T)
            x = R(rms_norm(h, W(p + "ln2_g"), m.norm_eps))
            gu = x @ W(p + "gate_up").T
            g, u = gu[:, :f], gu[:, f:]
            mh = R(g / (1.0 + np.exp(-g)) * u)           # SiLU(g) * u
            h = F(h + mh @ W(p + "down").T)
    last = h[T - 1]
    if m.arch == "opt":
        y = R(layer_norm(last, W("final_g"), W("final_b"), m.norm_eps))
        head = W("embed") if m.tied else W("lm_head")
    else:
        y = R(rms_norm(last, W("final_g"), m.norm_eps))
        head = W("lm_head")
    logits = F(head @ y)
    if return_hidden:
        return logits, h
    return logits


def first_token(logits: np.ndarray) -> int:
    """O4: argmax over the vocabulary, lowest index on exact ties (np.argmax)."""
    return int(np.argmax(logits))
