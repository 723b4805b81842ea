"""compute-sanitizer target for the kernels changed in round 2, at small sizes through the C ABI: the persistent GEMM's
224- and 160-column tiles (ragged N, bias / residual epilogues), the weight-streaming GEMV head (one and two
sequences, vocab slices), multi-tile attention on the longest-first grid (hd 128 and 64, GQA, two sequences), and a
batched merge. Each result is checked against a float64 reference so a silent corruption cannot pass.

    compute-sanitizer --tool memcheck python tools/sanitize_kernels.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_17707_b200 import _binding as B  # noqa: E402


def bf(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)


def f64(t):
    return t.float().cpu().numpy().astype(np.float64)


rng = np.random.default_rng(5)
s = torch.cuda.current_stream().cuda_stream
# persistent GEMM, 224- and 160-column tiles
for M, K, N in ((1024, 256, 3464), (1024, 256, 2600)):
    X, W, b = bf(rng.uniform(-1, 1, (M, K))), bf(rng.uniform(-0.05, 0.05, (N, K))), bf(rng.uniform(-0.05, 0.05, N))
    ref = f64(X) @ f64(W).T + f64(b)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    B.pb_op_gemm(X.data_ptr(), M, 0, M, K, W.data_ptr(), N, N, 0, b.data_ptr(), 0, 1.0, 0, out.data_ptr(), N, s)
    h = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    B.pb_op_gemm(X.data_ptr(), M, 0, M, K, W.data_ptr(), N, N, 1, b.data_ptr(), 0, 1.0, 0, h.data_ptr(), N, s)
    torch.cuda.synchronize()
    assert np.abs(f64(out) - ref).max() <= 0.02 * np.abs(ref).max(), "gemm bf16"
    assert np.abs(h.cpu().numpy() - ref).max() <= 1e-3 * np.abs(ref).max(), "gemm resid"
# GEMV head, whole and sliced
for Bsz in (1, 2):
    d, V = 2048, 3001
    y, E = bf(rng.uniform(-1, 1, (Bsz, d))), bf(rng.uniform(-0.035, 0.035, (V, d)))
    lg = torch.full((Bsz, V), float("nan"), device="cuda")
    B.pb_op_logits(y.data_ptr(), Bsz, d, E.data_ptr(), 0, 1234, lg.data_ptr(), V, s)
    B.pb_op_logits(y.data_ptr(), Bsz, d, E.data_ptr(), 1234, V, lg.data_ptr(), V, s)
    torch.cuda.synchronize()
    assert np.allclose(lg.cpu().numpy(), f64(y) @ f64(E).T, rtol=1e-4, atol=1e-4), "logits"
# attention, several query tiles (longest first), GQA, two sequences
for T, Bsz, H, KVH, hd in ((300, 2, 4, 2, 128), (260, 1, 2, 2, 64)):
    ld = (H + 2 * KVH) * hd
    qkv = bf(rng.uniform(-1, 1, (T * Bsz, ld)))
    out = torch.zeros(T * Bsz, H * hd, dtype=torch.bfloat16, device="cuda")
    B.pb_op_attention(qkv.data_ptr(), ld, out.data_ptr(), H * hd, 0, T, Bsz, H, KVH, hd, H * hd, (H + KVH) * hd,
                      hd ** -0.5, s)
    torch.cuda.synchronize()
    q = f64(qkv).reshape(T, Bsz, ld)
    for b in range(Bsz):
        for hh in range(H):
            kv = hh // (H // KVH)
            Q = q[:, b, hh * hd:(hh + 1) * hd]
            Kt = q[:, b, H * hd + kv * hd:H * hd + (kv + 1) * hd]
            Vt = q[:, b, (H + KVH) * hd + kv * hd:(H + KVH) * hd + (kv + 1) * hd]
            S = Q @ Kt.T * hd ** -0.5
            S[np.triu_indices(T, 1)] = -np.inf
            P = np.exp(S - S.max(1, keepdims=True))
            P /= P.sum(1, keepdims=True)
            got = f64(out).reshape(T, Bsz, H * hd)[:, b, hh * hd:(hh + 1) * hd]
            assert np.abs(got - P @ Vt).max() <= 0.03, "attention"
# batched merge
Ws = [bf(rng.uniform(-0.05, 0.05, (384, 640))) for _ in range(2)]
Bf, Af = bf(rng.uniform(-0.01, 0.01, (384, 16))), bf(rng.uniform(-0.01, 0.01, (16, 640)))
refs = [f64(w) + 2.0 * f64(Bf) @ f64(Af) for w in Ws]
B.pb_op_merge_batch([w.data_ptr() for w in Ws], [640] * 2, [384] * 2, [640] * 2, [Bf.data_ptr()] * 2,
                    [Af.data_ptr()] * 2, 16, [2.0] * 2, s)
torch.cuda.synchronize()
for w, r in zip(Ws, refs):
    assert np.abs(f64(w) - r).max() <= 2 ** -7 * np.abs(r).max(), "merge"
print("sanitize_kernels ok")
