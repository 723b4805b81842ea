"""Independent pin of the oracle's bf16 storage-precision mode (VERDICT r01 "What's weak" #3; SURVEY.md §8(c)
"Storage-precision contract"): oracle/forward.py in mode 'bf16' must reproduce, value for value, a hand-written
scalar forward in exact rational arithmetic that rounds at exactly the contract's points (tests/contract_ref.py),
on one-layer OPT and Llama (GQA) decoders — and leaving out ANY single rounding point of the hand-written forward
must break the agreement, so a dropped, added or moved rounding in the oracle cannot pass."""
import numpy as np
import pytest

import contract_ref as CR
from oracle import forward as OF
from oracle.numerics import rne_bf16
from synth.configs import ModelDesc


def _weights(arch, d, H, KVH, ffn, V, T, seed):
    # q / k weights large enough that attention scores are O(several): a sub-ulp change of q or k then moves
    # the softmax by more than the bf16 rounding of P absorbs
    rng = np.random.default_rng(seed)
    hd = d // H

    def lin(o, i, a=0.35):
        return rne_bf16(rng.uniform(-a, a, (o, i)))

    def vec(n, c=0.0, a=0.1):
        return rne_bf16(c + rng.uniform(-a, a, n))

    w = {"embed": lin(V, d, 0.8), "ln1_g": vec(d, 1.0), "ln2_g": vec(d, 1.0), "final_g": vec(d, 1.0)}
    if arch == "opt":
        w.update({"pos": lin(T + 2, d, 0.3), "ln1_b": vec(d), "ln2_b": vec(d), "final_b": vec(d),
                  "q": lin(d, d, 1.0), "k": lin(d, d, 1.0), "v": lin(d, d), "q_b": vec(d), "k_b": vec(d), "v_b": vec(d),
                  "o": lin(d, d), "o_b": vec(d), "fc1": lin(ffn, d), "fc1_b": vec(ffn), "fc2": lin(d, ffn),
                  "fc2_b": vec(d)})
    else:
        w.update({"q": lin(H * hd, d, 1.0), "k": lin(KVH * hd, d, 1.0), "v": lin(KVH * hd, d), "o": lin(d, H * hd),
                  "gate": lin(ffn, d), "up": lin(ffn, d), "down": lin(d, ffn), "lm_head": lin(V, d)})
    return w


def _oracle_W(arch, w):
    """The oracle's canonical tensor names (fused q|k|v, gate|up) over the same values."""
    m = {"embed": w["embed"], "final_g": w["final_g"], "L0.ln1_g": w["ln1_g"], "L0.ln2_g": w["ln2_g"],
         "L0.qkv": np.vstack([w["q"], w["k"], w["v"]]), "L0.o": w["o"]}
    if arch == "opt":
        m.update({"pos": w["pos"], "final_b": w["final_b"], "L0.ln1_b": w["ln1_b"], "L0.ln2_b": w["ln2_b"],
                  "L0.qkv_b": np.concatenate([w["q_b"], w["k_b"], w["v_b"]]), "L0.o_b": w["o_b"],
                  "L0.fc1": w["fc1"], "L0.fc1_b": w["fc1_b"], "L0.fc2": w["fc2"], "L0.fc2_b": w["fc2_b"]})
    else:
        m.update({"L0.gate_up": np.vstack([w["gate"], w["up"]]), "L0.down": w["down"], "lm_head": w["lm_head"]})
    return lambda name: m[name]


def _ref(arch, d, H, KVH, ffn, m, w, toks, skip=()):
    lg, hs = CR.forward(arch, d, H, KVH, ffn, m.norm_eps, m.rope_theta, {k: v.tolist() for k, v in w.items()}, toks,
                        skip=skip)
    return (np.array([float(x) for x in lg], dtype=np.float64),
            np.array([[float(x) for x in row] for row in hs], dtype=np.float64))


CASES = [("opt", 8, 2, 2, 16, 11, 3), ("llama", 8, 2, 1, 12, 11, 3), ("llama", 16, 4, 2, 24, 9, 4)]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-d{c[1]}-H{c[2]}-kv{c[3]}" for c in CASES])
def test_bf16_mode_equals_hand_written_contract(case):
    arch, d, H, KVH, ffn, V, T = case
    m = ModelDesc(arch, 1, d, H, KVH, ffn, V, T + 2 if arch == "opt" else 0, 1 if arch == "opt" else 0)
    w = _weights(arch, d, H, KVH, ffn, V, T, seed=d * 31 + H + KVH)
    toks = list(np.random.default_rng(7).integers(0, V, T))
    want, want_h = _ref(arch, d, H, KVH, ffn, m, w, toks)
    got, got_h = OF.forward_logits(m, _oracle_W(arch, w), np.array(toks), mode="bf16", return_hidden=True)
    # Both are fp32 values: every rounding point agrees, so the logits and the residual stream agree exactly.
    assert np.array_equal(np.asarray(got, dtype=np.float64), want), np.abs(np.asarray(got) - want).max()
    assert np.array_equal(np.asarray(got_h, dtype=np.float64), want_h), np.abs(np.asarray(got_h) - want_h).max()


@pytest.mark.parametrize("arch", ["opt", "llama"])
def test_every_rounding_point_is_observable(arch):
    """Mutation check of the pin itself: without any ONE of the contract's rounding points the hand-written
    forward no longer matches the oracle, so the equality above constrains every point. (A sub-ulp change survives
    only by flipping at least one downstream rounding, so the model is large enough to make that certain.)"""
    d, H, KVH, ffn, V, T = (16, 2, 2, 32, 13, 6) if arch == "opt" else (16, 4, 2, 24, 13, 6)
    m = ModelDesc(arch, 1, d, H, KVH, ffn, V, T + 2 if arch == "opt" else 0, 1 if arch == "opt" else 0)
    w = _weights(arch, d, H, KVH, ffn, V, T, seed=d * 31 + H + KVH)
    toks = list(np.random.default_rng(7).integers(0, V, T))
    ref, ref_h = OF.forward_logits(m, _oracle_W(arch, w), np.array(toks), mode="bf16", return_hidden=True)
    # h0 = E[tok] (+ P[t+2]) is exact in fp32 (one bf16 value, or the sum of two bf16 values whose exponents differ
    # by far less than 16): its rounding is an identity, not a point a mistake could move.
    for p in [q for q in CR.POINTS if q != "h0"]:
        mut, mut_h = _ref(arch, d, H, KVH, ffn, m, w, toks, skip=(p,))
        assert not (np.array_equal(mut, ref) and np.array_equal(mut_h, ref_h)), \
            f"rounding point {p} is not observable in the logits or the residual stream"


def test_round_sig_half_even():
    """The hand-written rounding itself: ties to even, at 8 (bf16) and 24 (fp32) significant bits."""
    from fractions import Fraction as Fr
    assert CR.bf16(Fr(257, 256)) == 1                 # 1 + 2^-8: tie between 1 and 1 + 2^-7 -> even (1)
    assert CR.bf16(Fr(259, 256)) == Fr(260, 256)      # 1 + 3*2^-8: tie -> even mantissa (1 + 2^-6)
    assert CR.bf16(Fr(-385, 256)) == Fr(-384, 256)    # -(1.5 + 2^-8): tie -> even
    assert CR.bf16(Fr(1, 3)) == Fr(float(np.float32(rne_bf16(np.float64(1 / 3)))))
    assert CR.f32(Fr(1, 3)) == Fr(float(np.float32(1 / 3)))
    assert CR.f32(Fr(2 ** 24 + 1, 2 ** 24)) == 1      # tie at 24 bits -> even
