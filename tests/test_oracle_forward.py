"""Pins for the oracle forward pass (O3/O4).

* Third-party definition: HF transformers' OPTForCausalLM / LlamaForCausalLM on
  CPU, run in float64 with the same (merged) weights, must give the same logits
  as the oracle's 'exact' mode (the paper builds on HF Transformers).
* Closed forms: T=1 attention reduces to v Wo^T (+bo); all-zero blocks make the
  decoder the identity on h, so logits = norm_f(h0[T-1]) E^T.
* The bf16 storage-contract mode stays close to exact mode.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import OracleWeights, first_token_logits
from oracle import forward as OF
from oracle import plan as P
from synth.configs import TINY_LLAMA, TINY_LLAMA_F32, TINY_OPT, TINY_OPT_F32, lora


def hf_state_dict(m, W):
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x))
    sd = {}
    d = m.d_model
    if m.arch == "opt":
        pre = "model.decoder."
        sd[pre + "embed_tokens.weight"] = t(W("embed"))
        sd[pre + "embed_positions.weight"] = t(W("pos"))
        sd[pre + "final_layer_norm.weight"] = t(W("final_g"))
        sd[pre + "final_layer_norm.bias"] = t(W("final_b"))
        for l in range(m.n_layers):
            p, q = f"{pre}layers.{l}.", f"L{l}."
            qkv, qkvb = W(q + "qkv"), W(q + "qkv_b")
            for j, nm in enumerate(("q_proj", "k_proj", "v_proj")):
                sd[p + f"self_attn.{nm}.weight"] = t(qkv[j * d:(j + 1) * d])
                sd[p + f"self_attn.{nm}.bias"] = t(qkvb[j * d:(j + 1) * d])
            sd[p + "self_attn.out_proj.weight"] = t(W(q + "o"))
            sd[p + "self_attn.out_proj.bias"] = t(W(q + "o_b"))
            sd[p + "self_attn_layer_norm.weight"] = t(W(q + "ln1_g"))
            sd[p + "self_attn_layer_norm.bias"] = t(W(q + "ln1_b"))
            sd[p + "fc1.weight"] = t(W(q + "fc1"))
            sd[p + "fc1.bias"] = t(W(q + "fc1_b"))
            sd[p + "fc2.weight"] = t(W(q + "fc2"))
            sd[p + "fc2.bias"] = t(W(q + "fc2_b"))
            sd[p + "final_layer_norm.weight"] = t(W(q + "ln2_g"))
            sd[p + "final_layer_norm.bias"] = t(W(q + "ln2_b"))
        sd["lm_head.weight"] = t(W("embed"))
    else:
        hd = m.head_dim
        qd, kvd, f = m.n_heads * hd, m.n_kv_heads * hd, m.d_ffn
        sd["model.embed_tokens.weight"] = t(W("embed"))
        sd["model.norm.weight"] = t(W("final_g"))
        sd["lm_head.weight"] = t(W("lm_head"))
        for l in range(m.n_layers):
            p, q = f"model.layers.{l}.", f"L{l}."
            qkv = W(q + "qkv")
            sd[p + "self_attn.q_proj.weight"] = t(qkv[:qd])
            sd[p + "self_attn.k_proj.weight"] = t(qkv[qd:qd + kvd])
            sd[p + "self_attn.v_proj.weight"] = t(qkv[qd + kvd:])
            sd[p + "self_attn.o_proj.weight"] = t(W(q + "o"))
            sd[p + "input_layernorm.weight"] = t(W(q + "ln1_g"))
            sd[p + "post_attention_layernorm.weight"] = t(W(q + "ln2_g"))
            gu = W(q + "gate_up")
            sd[p + "mlp.gate_proj.weight"] = t(gu[:f])
            sd[p + "mlp.up_proj.weight"] = t(gu[f:])
            sd[p + "mlp.down_proj.weight"] = t(W(q + "down"))
    return sd


def hf_model(m):
    if m.arch == "opt":
        from transformers import OPTConfig, OPTForCausalLM
        cfg = OPTConfig(vocab_size=m.vocab, hidden_size=m.d_model, num_hidden_layers=m.n_layers,
                        ffn_dim=m.d_ffn, num_attention_heads=m.n_heads, max_position_embeddings=m.max_pos,
                        word_embed_proj_dim=m.d_model, do_layer_norm_before=True, dropout=0.0,
                        attention_dropout=0.0, activation_function="relu", enable_bias=True,
                        tie_word_embeddings=True)
        cfg._attn_implementation = "eager"
        return OPTForCausalLM(cfg)
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(vocab_size=m.vocab, hidden_size=m.d_model, intermediate_size=m.d_ffn,
                      num_hidden_layers=m.n_layers, num_attention_heads=m.n_heads,
                      num_key_value_heads=m.n_kv_heads, rms_norm_eps=m.norm_eps, rope_theta=m.rope_theta,
                      max_position_embeddings=4096, tie_word_embeddings=False, attention_bias=False,
                      mlp_bias=False, hidden_act="silu")
    cfg._attn_implementation = "eager"
    return LlamaForCausalLM(cfg)


@pytest.mark.parametrize("model", [TINY_OPT, TINY_LLAMA], ids=["opt", "llama"])
def test_oracle_matches_hf_transformers_fp64(model):
    ads = (lora(8),)
    ow = OracleWeights(model, ads)
    W = lambda n: ow.get(n, 0)
    toks = synth.tokens(1, 16, model.vocab)[0]
    ours = OF.forward_logits(model, W, toks, "exact")
    hf = hf_model(model).double().eval()
    missing, unexpected = hf.load_state_dict(hf_state_dict(model, W), strict=False)
    assert not unexpected
    assert all("rotary" in k or "inv_freq" in k for k in missing), missing
    with torch.no_grad():
        ref = hf(torch.from_numpy(toks.astype(np.int64))[None]).logits[0, -1].numpy()
    rel = np.abs(ours - ref).max() / np.abs(ref).max()
    assert rel < 1e-6, rel          # HF upcasts softmax to fp32: ~3e-8 observed
    assert OF.first_token(ours) == int(np.argmax(ref))


@pytest.mark.parametrize("model", [TINY_OPT_F32, TINY_LLAMA_F32], ids=["opt", "llama"])
def test_f32_oracle_matches_hf_transformers(model):
    """fp32 debug-parity models (the 1e-4 gate): the oracle's 'exact' mode on the fp32 weights equals HF in
    float64, and its 'f32' storage mode equals HF run natively in float32 (a third-party fp32 forward) to
    well inside 1e-4."""
    ads = (lora(8),)
    ow = OracleWeights(model, ads)
    W = lambda n: ow.get(n, 0)
    toks = synth.tokens(1, 16, model.vocab)[0]
    exact = OF.forward_logits(model, W, toks, "exact")
    f32 = OF.forward_logits(model, W, toks, "f32")
    hf = hf_model(model).double().eval()
    hf.load_state_dict(hf_state_dict(model, W), strict=False)
    x = torch.from_numpy(toks.astype(np.int64))[None]
    with torch.no_grad():
        ref64 = hf(x).logits[0, -1].numpy()
        ref32 = hf.float()(x).logits[0, -1].double().numpy()
    assert np.abs(exact - ref64).max() / np.abs(ref64).max() < 1e-6
    rel = np.abs(f32 - ref32).max() / np.abs(ref32).max()
    assert rel < 2e-5, rel
    assert 0 < np.abs(f32 - exact).max() / np.abs(exact).max() < 1e-5


def test_merge_moves_logits():
    # The adapter is not a no-op: skipping the merge changes the logits well
    # beyond the 1e-2 parity gate (so a GPU path that skipped a3 would fail).
    m = TINY_OPT
    ow = OracleWeights(m, (lora(8),))
    toks = synth.tokens(1, 16, m.vocab)[0]
    merged = OF.forward_logits(m, lambda n: ow.get(n, 0), toks, "exact")
    base = OF.forward_logits(m, lambda n: ow.get(n, None), toks, "exact")
    assert np.abs(merged - base).max() / np.abs(merged).max() > 2e-2


def test_t1_attention_closed_form():
    # T = 1: softmax over one key is 1, so the attention output is v itself and
    # the first residual update is h += v Wo^T + bo.
    m = TINY_OPT
    ow = OracleWeights(m, ())
    W = lambda n: ow.get(n, None)
    tok = np.array([7])
    _, h = OF.forward_logits(m, W, tok, "exact", layers=[0], return_hidden=True)
    h0 = W("embed")[7] + W("pos")[2]
    x = OF.layer_norm(h0, W("L0.ln1_g"), W("L0.ln1_b"), m.norm_eps)
    v = x @ W("L0.qkv")[2 * m.d_model:].T + W("L0.qkv_b")[2 * m.d_model:]
    h1 = h0 + v @ W("L0.o").T + W("L0.o_b")
    x2 = OF.layer_norm(h1, W("L0.ln2_g"), W("L0.ln2_b"), m.norm_eps)
    h2 = h1 + np.maximum(x2 @ W("L0.fc1").T + W("L0.fc1_b"), 0) @ W("L0.fc2").T + W("L0.fc2_b")
    assert np.allclose(h[0], h2, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("model", [TINY_OPT, TINY_LLAMA], ids=["opt", "llama"])
def test_zero_blocks_identity(model):
    ow = OracleWeights(model, ())
    def W(n):
        x = ow.get(n, None)
        if n.startswith("L"):
            sfx = n.split(".", 1)[1]
            if sfx not in ("ln1_g", "ln2_g", "ln1_b", "ln2_b"):
                return np.zeros_like(x)
        return x
    toks = synth.tokens(1, 12, model.vocab)[0]
    got = OF.forward_logits(model, W, toks, "exact")
    h0 = W("embed")[toks[-1]] + (W("pos")[len(toks) - 1 + 2] if model.arch == "opt" else 0)
    if model.arch == "opt":
        y = OF.layer_norm(h0, W("final_g"), W("final_b"), model.norm_eps)
        want = W("embed") @ y
    else:
        y = OF.rms_norm(h0, W("final_g"), model.norm_eps)
        want = W("lm_head") @ y
    assert np.allclose(got, want, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("model", [TINY_OPT, TINY_LLAMA], ids=["opt", "llama"])
def test_bf16_contract_close_to_exact(model):
    toks = synth.tokens(1, 16, model.vocab)
    ex, _ = first_token_logits(model, (lora(8),), toks, mode="exact")
    bf, _ = first_token_logits(model, (lora(8),), toks, mode="bf16")
    rel = np.abs(ex - bf).max() / np.abs(ex).max()
    assert 0 < rel < 1e-2, rel


def test_layernorm_rmsnorm_definitions():
    x = np.array([1.0, 2.0, 3.0, 6.0])
    y = OF.layer_norm(x, np.ones(4), np.zeros(4), 0.0)
    assert abs(y.mean()) < 1e-15 and abs((y ** 2).mean() - 1) < 1e-13
    z = OF.rms_norm(x, np.ones(4), 0.0)
    assert abs((z ** 2).mean() - 1) < 1e-13


def test_rope_is_rotation():
    # RoPE preserves each (i, i+hd/2) pair's norm and is the identity at t=0
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 2 * 8))
    y = OF.rope(x, 2, 8, 1e4)
    assert np.allclose(y[0], x[0])
    for h in range(2):
        a, b = x[:, h * 8:h * 8 + 4], x[:, h * 8 + 4:(h + 1) * 8]
        c, d = y[:, h * 8:h * 8 + 4], y[:, h * 8 + 4:(h + 1) * 8]
        assert np.allclose(a * a + b * b, c * c + d * d)
