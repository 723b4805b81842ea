"""Hand-written scalar reference of the storage-precision contract (TEST CODE; pins oracle/forward.py's 'bf16'
mode independently — VERDICT r01 "What's weak" #3, SURVEY.md §8(c) "Storage-precision contract").

Nothing here comes from oracle/: every operation is a scalar Python loop in exact rational arithmetic
(fractions.Fraction) and every rounding is written out by hand (round half to even at 8 significant bits for
bf16, 24 for fp32). The only inexact steps are the transcendental functions the model definitions need — sqrt
(norm), exp (softmax, SiLU), cos / sin (RoPE) — evaluated with Python's `math` on the exact argument converted to
a double; their ~1e-16 relative error cannot move a bf16 (2^-9) or fp32 (2^-24) rounding except on an exact
tie, which random inputs do not produce.

Contract: weights bf16; residual stream h fp32; norm outputs, q/k/v (after bias,
q-scale, RoPE), softmax probabilities P, attention output a, MLP hidden -> bf16; everything else exact here; final
logits fp32. `skip` names rounding points to leave out (mutation tests: each one must change the logits).
"""
from __future__ import annotations

import math
from fractions import Fraction as Fr

POINTS = ("h0", "x1", "q", "k", "v", "P", "a", "h_attn", "x2", "mlp", "h_mlp", "y", "logits")


def _round_sig(x: Fr, bits: int) -> Fr:
    """Round-half-even of an exact rational to `bits` significant bits (no underflow at these magnitudes)."""
    if x == 0:
        return Fr(0)
    ax = abs(x)
    e = ax.numerator.bit_length() - ax.denominator.bit_length()   # 2^(e-1) <= ax < 2^(e+1)
    while Fr(2) ** e > ax:
        e -= 1
    while Fr(2) ** (e + 1) <= ax:
        e += 1
    ulp = Fr(2) ** (e - bits + 1)                                  # 2^e <= ax < 2^(e+1)
    q = ax / ulp
    n = q.numerator // q.denominator
    rem = q - n
    if rem > Fr(1, 2) or (rem == Fr(1, 2) and n % 2 == 1):
        n += 1
    r = n * ulp
    return r if x > 0 else -r


def bf16(x: Fr) -> Fr:
    return _round_sig(x, 8)


def f32(x: Fr) -> Fr:
    return _round_sig(x, 24)


def _fr(v: float) -> Fr:
    return Fr(float(v))


def forward(arch, d, H, KVH, ffn, eps, theta, W, tokens, skip=()):
    """Last-position logits (list of Fractions) and the final residual stream h [T][d] of a one-layer OPT (pre-LN, biases, learned positions offset 2,
    ReLU, tied head) or Llama (RMSNorm, rotate_half RoPE, GQA, SiLU * up) decoder. W: dict name -> nested lists
    of floats (bf16 values)."""
    R = {p: ((lambda x: x) if p in skip else (f32 if p in ("h0", "h_attn", "h_mlp", "logits") else bf16))
         for p in POINTS}
    T = len(tokens)
    hd = d // H
    w = {k: ([[Fr(float(c)) for c in row] for row in v] if isinstance(v[0], (list, tuple)) else
             [Fr(float(c)) for c in v]) for k, v in W.items()}

    def matvec(M, x, bias=None):           # M [out][in] (HF layout), x [in]
        out = []
        for i, row in enumerate(M):
            s = sum((row[j] * x[j] for j in range(len(x))), Fr(0))
            out.append(s + (bias[i] if bias is not None else 0))
        return out

    def layer_norm(x, g, b):
        n = len(x)
        mu = sum(x, Fr(0)) / n
        var = sum(((v - mu) ** 2 for v in x), Fr(0)) / n
        inv = Fr(1) / _fr(math.sqrt(float(var + Fr(eps))))
        return [(x[i] - mu) * inv * g[i] + b[i] for i in range(n)]

    def rms_norm(x, g):
        n = len(x)
        ms = sum((v * v for v in x), Fr(0)) / n
        inv = Fr(1) / _fr(math.sqrt(float(ms + Fr(eps))))
        return [x[i] * inv * g[i] for i in range(n)]

    def rope(vec, t, nh):                  # rotate_half per head, angle t * theta^(-2i/hd)
        out = list(vec)
        half = hd // 2
        for h in range(nh):
            for i in range(half):
                ang = t * theta ** (-(2.0 * i) / hd)
                c, s = _fr(math.cos(ang)), _fr(math.sin(ang))
                a, b = vec[h * hd + i], vec[h * hd + half + i]
                out[h * hd + i] = a * c - b * s
                out[h * hd + half + i] = b * c + a * s
        return out

    # embedding (+ OPT learned positions, HF offset 2)
    hs = []
    for t, tok in enumerate(tokens):
        e = w["embed"][tok]
        if arch == "opt":
            e = [e[i] + w["pos"][t + 2][i] for i in range(d)]
        hs.append([R["h0"](v) for v in e])

    # attention block
    qs, ks, vs = [], [], []
    for t in range(T):
        if arch == "opt":
            x = [R["x1"](v) for v in layer_norm(hs[t], w["ln1_g"], w["ln1_b"])]
            q = matvec(w["q"], x, w["q_b"])
            q = [v * _fr(hd ** -0.5) for v in q]          # HF OPT scales q after the bias
            k = matvec(w["k"], x, w["k_b"])
            v_ = matvec(w["v"], x, w["v_b"])
        else:
            x = [R["x1"](v) for v in rms_norm(hs[t], w["ln1_g"])]
            q = rope(matvec(w["q"], x), t, H)
            k = rope(matvec(w["k"], x), t, KVH)
            v_ = matvec(w["v"], x)
        qs.append([R["q"](v) for v in q])
        ks.append([R["k"](v) for v in k])
        vs.append([R["v"](v) for v in v_])
    group = H // KVH
    scale = Fr(1) if arch == "opt" else _fr(hd ** -0.5)
    for t in range(T):
        a = []
        for h in range(H):
            kv = h // group
            S = [sum((qs[t][h * hd + c] * ks[j][kv * hd + c] for c in range(hd)), Fr(0)) * scale
                 for j in range(t + 1)]
            m = max(S)
            E = [_fr(math.exp(float(s - m))) for s in S]
            Z = sum(E, Fr(0))
            P = [R["P"](e / Z) for e in E]
            for c in range(hd):
                a.append(sum((P[j] * vs[j][kv * hd + c] for j in range(t + 1)), Fr(0)))
        a = [R["a"](v) for v in a]
        o = matvec(w["o"], a, w.get("o_b"))
        hs[t] = [R["h_attn"](hs[t][i] + o[i]) for i in range(d)]

    # MLP block
    for t in range(T):
        if arch == "opt":
            x = [R["x2"](v) for v in layer_norm(hs[t], w["ln2_g"], w["ln2_b"])]
            u = [R["mlp"](max(v, Fr(0))) for v in matvec(w["fc1"], x, w["fc1_b"])]
            f = matvec(w["fc2"], u, w["fc2_b"])
        else:
            x = [R["x2"](v) for v in rms_norm(hs[t], w["ln2_g"])]
            g = matvec(w["gate"], x)
            up = matvec(w["up"], x)
            u = [R["mlp"](g[i] / (1 + _fr(math.exp(-float(g[i])))) * up[i]) for i in range(ffn)]
            f = matvec(w["down"], u)
        hs[t] = [R["h_mlp"](hs[t][i] + f[i]) for i in range(d)]

    last = hs[T - 1]
    if arch == "opt":
        y = [R["y"](v) for v in layer_norm(last, w["final_g"], w["final_b"])]
        head = w["embed"]
    else:
        y = [R["y"](v) for v in rms_norm(last, w["final_g"])]
        head = w["lm_head"]
    return [R["logits"](v) for v in matvec(head, y)], hs
