"""Kernel-level parity on the B200: each pb_op_* (the path's own kernels, through the C ABI)
against the oracle's definitions on seeded inputs, including ragged tails."""
import numpy as np
import pytest
import torch

from oracle import forward as OF
from oracle.merge import merge_bf16_bits
from oracle.numerics import bf16_bits_to_f64, bf16_ulp, f64_to_bf16_bits, rne_bf16
from paper_2503_17707_b200 import _binding as B
from gpu_util import dev_bf16, dev_f32, host_bits, need_gpu, ptr, stream

pytestmark = pytest.mark.gpu


def rbits(rng, shape, a):
    return f64_to_bf16_bits(rng.uniform(-a, a, size=shape))


@pytest.mark.parametrize("rows,cols,rank", [(256, 256, 8), (384, 640, 16), (200, 328, 16), (512, 512, 64),
                                            (128, 1024, 32), (1000, 136, 16), (2048, 2048, 16),
                                            # full-size targets: OPT-13B q|k|v|o (C4, r=64), Llama-2-70B q (C5a)
                                            (5120, 5120, 64), (8192, 8192, 16),
                                            # persistent grid: several tiles per CTA through the stage ring, ragged
                                            (20480, 5120, 64), (1100, 8200, 32), (130, 136, 64)])
def test_merge_within_one_ulp_of_correct_rounding(rows, cols, rank):
    need_gpu()
    rng = np.random.default_rng(rows * 7 + cols + rank)
    guard = 3
    full = rbits(rng, (rows + 2 * guard, cols), 0.035)
    Bm = rbits(rng, (rows, rank), 0.08)
    Am = rbits(rng, (rank, cols), 1 / np.sqrt(cols))
    s = 2.0
    W = dev_bf16(full)
    Bd, Ad = dev_bf16(Bm), dev_bf16(Am)
    region = ptr(W) + guard * cols * 2
    B.pb_op_merge(region, cols, rows, cols, ptr(Bd), ptr(Ad), rank, s, stream())
    torch.cuda.synchronize()
    got = host_bits(W)
    want = merge_bf16_bits(full[guard:guard + rows], Bm, Am, s)
    # rows outside the region are untouched (bit exact)
    assert np.array_equal(got[:guard], full[:guard]) and np.array_equal(got[guard + rows:], full[guard + rows:])
    g = bf16_bits_to_f64(got[guard:guard + rows])
    w = bf16_bits_to_f64(want)
    # Bound: 1 bf16 ulp of the correctly rounded value (final rounding) + the fp32 accumulation error of
    # W + s*sum_k B A, (r + 2) * 2^-24 * (|W| + s * sum_k |B||A|) — the latter only matters under
    # cancellation (W ~ -s*BA), where the result is tiny and its ulp finer than fp32's error on the terms.
    Wf = bf16_bits_to_f64(full[guard:guard + rows])
    mag = np.abs(Wf) + s * (np.abs(bf16_bits_to_f64(Bm)) @ np.abs(bf16_bits_to_f64(Am)))
    bound = bf16_ulp(w) + (rank + 2) * 2.0 ** -24 * mag
    assert np.all(np.abs(g - w) <= bound), (np.abs(g - w) / bound).max()
    assert (g == w).mean() > 0.95


@pytest.mark.parametrize("rank", [16, 64])
def test_merge_batch_jobs_in_one_launch(rank):
    """pb_op_merge_batch: several tensors of different (ragged) shapes merged by one persistent launch whose CTAs walk
    all jobs' tiles as one list; each job must equal the correctly rounded merge like a single-job launch."""
    need_gpu()
    rng = np.random.default_rng(rank)
    shapes = [(256, 384), (130, 1000), (2048, 2048), (64, 136), (1024, 512)]
    Ws, Bs, As, want, devs = [], [], [], [], []
    for (rows, cols) in shapes:
        W = rbits(rng, (rows, cols), 0.035)
        Bm = rbits(rng, (rows, rank), 0.08)
        Am = rbits(rng, (rank, cols), 1 / np.sqrt(cols))
        d = (dev_bf16(W), dev_bf16(Bm), dev_bf16(Am))
        devs.append(d)
        Ws.append(W)
        want.append(merge_bf16_bits(W, Bm, Am, 2.0))
        Bs.append(Bm)
        As.append(Am)
    B.pb_op_merge_batch([ptr(d[0]) for d in devs], [c for _, c in shapes], [r for r, _ in shapes],
                        [c for _, c in shapes], [ptr(d[1]) for d in devs], [ptr(d[2]) for d in devs], rank,
                        [2.0] * len(shapes), stream())
    torch.cuda.synchronize()
    for (rows, cols), d, W, Bm, Am, wnt in zip(shapes, devs, Ws, Bs, As, want):
        g = bf16_bits_to_f64(host_bits(d[0]))
        w = bf16_bits_to_f64(wnt)
        mag = np.abs(bf16_bits_to_f64(W)) + 2.0 * (np.abs(bf16_bits_to_f64(Bm)) @ np.abs(bf16_bits_to_f64(Am)))
        assert np.all(np.abs(g - w) <= bf16_ulp(w) + (rank + 2) * 2.0 ** -24 * mag), (rows, cols)
        assert (g == w).mean() > 0.95


def test_merge_zero_B_is_identity():
    need_gpu()
    rng = np.random.default_rng(5)
    Wb = rbits(rng, (256, 384), 0.05)
    W = dev_bf16(Wb)
    Bd = dev_bf16(np.zeros((256, 16), np.uint16))
    Ad = dev_bf16(rbits(rng, (16, 384), 0.1))
    B.pb_op_merge(ptr(W), 384, 256, 384, ptr(Bd), ptr(Ad), 16, 2.0, stream())
    torch.cuda.synchronize()
    assert np.array_equal(host_bits(W), Wb)


def _gemm_case(rng, M, K, N):
    X = rbits(rng, (M, K), 1.0)
    W = rbits(rng, (N, K), 0.05)
    bias = rbits(rng, (N,), 0.05)
    return X, W, bias


@pytest.mark.parametrize("M,K,N,m0,m1", [(128, 256, 768, 0, 128), (16, 256, 1024, 0, 16), (300, 512, 384, 0, 300),
                                         (256, 2048, 640, 128, 256), (200, 192, 136, 40, 170), (130, 688, 256, 0, 130),
                                         (1024, 1024, 3072, 0, 1024), (2048, 512, 8192, 0, 2000),
                                         (700, 1536, 1000, 100, 700),
                                         # persistent kernel with 192-column tiles and a ragged last tile
                                         (1024, 512, 3000, 0, 1024),
                                         # 224-column tiles (128 + 64 + 32-row weight boxes; the last tile's 64- and
                                         # 32-row boxes wholly past N) and 160-column tiles (128 + 32), ragged M
                                         (1500, 256, 2328, 0, 1500), (1100, 512, 2300, 100, 1100),
                                         # M <= 2: the weight-streaming GEMV (decode sizes), ragged N and K
                                         (1, 2048, 640, 0, 1), (2, 512, 136, 0, 2), (3, 688, 258, 1, 3)])
def test_gemm_bf16_epilogue(M, K, N, m0, m1):
    need_gpu()
    rng = np.random.default_rng(M + K + N)
    X, W, bias = _gemm_case(rng, M, K, N)
    out = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
    sc_cols = N // 3
    Xd, Wd, bd = dev_bf16(X), dev_bf16(W), dev_bf16(bias)   # keep references alive across the async launch
    B.pb_op_gemm(ptr(Xd), M, m0, m1, K, ptr(Wd), N, N, 0, ptr(bd), 0, 0.125, sc_cols, ptr(out), N, stream())
    torch.cuda.synchronize()
    ref = bf16_bits_to_f64(X) @ bf16_bits_to_f64(W).T + bf16_bits_to_f64(bias)
    ref[:, :sc_cols] *= 0.125
    got = bf16_bits_to_f64(host_bits(out))
    assert np.all(got[:m0] == 0) and np.all(got[m1:] == 0)
    r = ref[m0:m1]
    err = np.abs(got[m0:m1] - r)
    assert np.all(err <= bf16_ulp(r) + 1e-6 * np.abs(r).max()), err.max()


@pytest.mark.parametrize("M,K,N,f", [(192, 320, 256, 136), (1536, 1024, 2560, 2752), (2, 320, 256, 136),
                                     (1, 2048, 512, 330), (1024, 512, 3000, 136), (600, 256, 1000, 136),
                                     (1024, 512, 3464, 136), (1024, 512, 2600, 136)])
def test_gemm_relu_and_resid_and_silu(M, K, N, f):
    """Small shapes take the split-K kernel or the persistent 128x256 kernel at S = 1; the second case runs the
    persistent kernel over more tiles than SMs (both TMEM accumulators cycle); M <= 2 takes the GEMV; the last two
    take the persistent kernel's 192- and 128-column tiles (ragged N), the last two its 224- and 160-column tiles."""
    need_gpu()
    rng = np.random.default_rng(11 + M)
    X, W, bias = _gemm_case(rng, M, K, N)
    Xd, Wd, bd = dev_bf16(X), dev_bf16(W), dev_bf16(bias)
    ref = bf16_bits_to_f64(X) @ bf16_bits_to_f64(W).T + bf16_bits_to_f64(bias)
    # ReLU
    out = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
    B.pb_op_gemm(ptr(Xd), M, 0, M, K, ptr(Wd), N, N, 0, ptr(bd), 1, 1.0, 0, ptr(out), N, stream())
    torch.cuda.synchronize()
    r = np.maximum(ref, 0)
    assert np.all(np.abs(bf16_bits_to_f64(host_bits(out)) - r) <= bf16_ulp(r) + 1e-6)
    # residual fp32
    h0 = rng.standard_normal((M, N)).astype(np.float32)
    h = dev_f32(h0)
    B.pb_op_gemm(ptr(Xd), M, 0, M, K, ptr(Wd), N, N, 1, ptr(bd), 0, 1.0, 0, ptr(h), N, stream())
    torch.cuda.synchronize()
    assert np.allclose(h.cpu().numpy(), h0 + ref, rtol=1e-5, atol=1e-5)
    # SiLU(gate) * up with W = [gate; up]
    Wgu = rbits(rng, (2 * f, K), 0.05)
    out2 = torch.zeros((M, f), dtype=torch.bfloat16, device="cuda")
    Wgud = dev_bf16(Wgu)
    B.pb_op_gemm(ptr(Xd), M, 0, M, K, ptr(Wgud), 2 * f, f, 2, 0, 0, 1.0, 0, ptr(out2), f, stream())
    torch.cuda.synchronize()
    gu = bf16_bits_to_f64(X) @ bf16_bits_to_f64(Wgu).T
    g, u = gu[:, :f], gu[:, f:]
    r2 = g / (1 + np.exp(-g)) * u
    err = np.abs(bf16_bits_to_f64(host_bits(out2)) - r2)
    assert np.all(err <= 2 * bf16_ulp(r2) + 1e-5), err.max()


@pytest.mark.parametrize("rms", [False, True])
@pytest.mark.parametrize("d", [256, 2048, 4096, 5120, 8192, 9216])
def test_norm(rms, d):
    need_gpu()
    rng = np.random.default_rng(d + rms)
    rows = 37
    h = (rng.standard_normal((rows, d)) * 3 + 0.5).astype(np.float32)
    g = rbits(rng, (d,), 0.1) if False else f64_to_bf16_bits(1 + rng.uniform(-0.1, 0.1, d))
    b = f64_to_bf16_bits(rng.uniform(-0.02, 0.02, d))
    out = torch.zeros((rows, d), dtype=torch.bfloat16, device="cuda")
    hd_, gd, bd = dev_f32(h), dev_bf16(g), dev_bf16(b)
    B.pb_op_norm(ptr(hd_), rows, d, ptr(gd), 0 if rms else ptr(bd), 1e-5, ptr(out), stream())
    torch.cuda.synchronize()
    hf = h.astype(np.float64)
    ref = OF.rms_norm(hf, bf16_bits_to_f64(g), 1e-5) if rms else \
        OF.layer_norm(hf, bf16_bits_to_f64(g), bf16_bits_to_f64(b), 1e-5)
    err = np.abs(bf16_bits_to_f64(host_bits(out)) - ref)
    assert np.all(err <= bf16_ulp(ref) + 1e-6), err.max()


@pytest.mark.parametrize("T,Bsz,H,KVH,hd,t0,t1", [(16, 1, 4, 4, 64, 0, 16), (77, 2, 4, 2, 128, 0, 77),
                                                  (128, 1, 2, 2, 64, 64, 128), (40, 3, 2, 1, 32, 17, 40),
                                                  (300, 2, 4, 2, 128, 0, 300), (520, 1, 2, 1, 64, 256, 520),
                                                  (257, 1, 2, 2, 128, 129, 257), (384, 3, 2, 2, 64, 0, 384),
                                                  # one query position (decode steps): the SIMT decode kernel
                                                  (300, 2, 4, 2, 128, 299, 300), (129, 3, 4, 4, 64, 128, 129),
                                                  (1, 1, 2, 1, 128, 0, 1), (500, 1, 8, 2, 128, 499, 500),
                                                  (1000, 2, 4, 2, 64, 999, 1000),
                                                  (2000, 1, 8, 2, 128, 1999, 2000)])   # clusters of 1, 2, 4, 8 CTAs
def test_attention(T, Bsz, H, KVH, hd, t0, t1):
    """Tensor-core kernel for hd 64/128 (SIMT for 32) vs the oracle's exact causal attention. Bound: the final
    bf16 rounding (1 ulp, 2 allowed) plus the bf16 rounding of the probabilities fed to the PV product (relative
    2^-9 each, so |err| <= 2^-9 * sum_j P_j |v_j|; 2^-8 allowed). The tensor-core kernel rounds the NORMALISED
    probabilities (two passes), exactly where the storage contract rounds them: against the oracle's bf16-contract
    attention RNE_bf16(RNE_bf16(P) v) it must be bit-exact on >= 97 % of the outputs and otherwise off only by
    rounding flips of single probabilities (fp32 vs fp64 arithmetic), <= 1 ulp + 2^-8 * max_j P_j |v_j|."""
    need_gpu()
    rng = np.random.default_rng(T + H + hd)
    qd, kvd = H * hd, KVH * hd
    ld = qd + 2 * kvd
    qkv = rbits(rng, (T * Bsz, ld), 1.0)
    out = torch.zeros((T * Bsz, qd), dtype=torch.bfloat16, device="cuda")
    scale = hd ** -0.5
    qkvd = dev_bf16(qkv)
    B.pb_op_attention(ptr(qkvd), ld, ptr(out), qd, t0, t1, Bsz, H, KVH, hd, qd, qd + kvd, scale, stream())
    torch.cuda.synchronize()
    got = bf16_bits_to_f64(host_bits(out))
    x = bf16_bits_to_f64(qkv)
    for b in range(Bsz):
        rows = np.arange(T) * Bsz + b
        q, k, v = x[rows, :qd], x[rows, qd:qd + kvd], x[rows, qd + kvd:]
        ref = OF.causal_attention(q, k, v, H, KVH, hd, scale, lambda z: z)
        pv_abs = OF.causal_attention(q, k, np.abs(v), H, KVH, hd, scale, lambda z: z)
        g = got[rows]
        assert np.all(g[:t0] == 0)
        assert np.all(g[t1:] == 0)
        err = np.abs(g[t0:t1] - ref[t0:t1])
        bound = 2 * bf16_ulp(ref[t0:t1]) + 2.0 ** -8 * pv_abs[t0:t1] + 1e-6
        assert np.all(err <= bound), (err - bound).max()
        if hd in (64, 128):
            con = rne_bf16(OF.causal_attention(q, k, v, H, KVH, hd, scale, rne_bf16))[t0:t1]
            frac = float((g[t0:t1] == con).mean())
            # one query position over hundreds of keys (decode): every output sums that many rounded probabilities,
            # so a single fp32-vs-fp64 rounding flip anywhere in the row changes it — 0.95 there (measured 0.964 at
            # 500 keys), 0.97 for the prompt tiles, whose rows average far fewer keys
            assert frac >= (0.95 if t1 - t0 == 1 and T > 256 else 0.97), frac
            e2 = np.abs(g[t0:t1] - con)
            assert np.all(e2 <= 2 * bf16_ulp(con) + 2.0 ** -6 * np.abs(v).max() + 1e-6), e2.max()


@pytest.mark.parametrize("T,H,KVH,hd", [(1024, 40, 40, 128), (640, 16, 4, 64), (128, 32, 32, 64)])
def test_attention_deterministic_under_load(T, H, KVH, hd):
    """Two CTAs per SM share the tensor pipe and TMEM, and P is written over S in TMEM: repeated launches (with
    another launch in flight) must give the same bits every time — a race between the two softmax threads of a row,
    or between a CTA's PV and its next QK^T, would show up as run-to-run differences."""
    need_gpu()
    rng = np.random.default_rng(T + H)
    qd, kvd = H * hd, KVH * hd
    ld = qd + 2 * kvd
    qkv = dev_bf16(f64_to_bf16_bits(rng.standard_normal((T, ld)) * 1.3))
    outs = [torch.zeros((T, qd), dtype=torch.bfloat16, device="cuda") for _ in range(6)]
    for o in outs:
        B.pb_op_attention(ptr(qkv), ld, ptr(o), qd, 0, T, 1, H, KVH, hd, qd, qd + kvd, hd ** -0.5, stream())
    torch.cuda.synchronize()
    ref = host_bits(outs[0])
    for o in outs[1:]:
        assert np.array_equal(host_bits(o), ref)


@pytest.mark.parametrize("M,K,H,KVH,hd,B_,row0,split", [
    (2048, 1024, 8, 2, 128, 1, 0, 0),      # persistent 256-column tiles (C5a-like GQA), rope + plain v columns
    (600, 512, 4, 4, 128, 2, 0, 0),        # persistent, 2 sequences token-major, ragged last row tile
    (128, 2048, 4, 2, 128, 1, 0, 0),       # split-K cluster kernel (128-column tiles)
    (128, 512, 8, 8, 64, 4, 0, 2),         # split-K S=2, hd 64 (two heads per tile), 4 sequences
    (300, 256, 4, 2, 64, 1, 44, 0),        # microbatch offset: positions count from row0
    (2, 1024, 4, 2, 128, 2, 0, 0),         # GEMV (decode sizes): rotary CTAs pair rows i and i + hd/2
    (1, 512, 8, 2, 64, 1, 0, 0)])
def test_gemm_rope_single_rounding(M, K, H, KVH, hd, B_, row0, split):
    """Llama QKV: RoPE on the fp32 accumulator in the GEMM epilogue, then ONE bf16 rounding — the storage contract's
    q/k = RNE_bf16(rope(x W^T)). Against the oracle's rope (oracle/forward.py, HF rotate_half) of the exact product:
    within 1 ulp of the correctly rounded value everywhere and bit-exact on >= 97 % (fp32 accumulation only)."""
    need_gpu()
    rng = np.random.default_rng(M + K + hd)
    qd, kvd = H * hd, KVH * hd
    N = qd + 2 * kvd
    X = rbits(rng, (M, K), 1.0)
    W = rbits(rng, (N, K), 0.05)
    T = (M - row0 + B_ - 1) // B_
    out = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
    table = torch.empty(T * hd, dtype=torch.float32, device="cuda")
    Xd, Wd = dev_bf16(X), dev_bf16(W)
    B.pb_op_gemm_rope(ptr(Xd), M, row0, M, K, ptr(Wd), N, ptr(out), N, qd + kvd, hd, row0, B_, T, 1e4, ptr(table),
                      split, stream())
    torch.cuda.synchronize()
    prod = bf16_bits_to_f64(X) @ bf16_bits_to_f64(W).T
    got = bf16_bits_to_f64(host_bits(out))
    assert np.all(got[:row0] == 0)
    for b in range(B_):
        rows = row0 + np.arange(T) * B_ + b
        rows = rows[rows < M]
        p = prod[rows]
        ref = np.concatenate([OF.rope(p[:, :qd], H, hd, 1e4), OF.rope(p[:, qd:qd + kvd], KVH, hd, 1e4), p[:, qd + kvd:]],
                             axis=1)
        # positions of these rows are 0..len-1 (oracle rope numbers rows from 0)
        con = rne_bf16(ref)
        g = got[rows]
        assert np.all(np.abs(g - con) <= bf16_ulp(con) + 1e-6), np.abs(g - con).max()
        assert (g == con).mean() >= 0.97, (g == con).mean()


def test_rope():
    need_gpu()
    rng = np.random.default_rng(3)
    T, Bsz, H, KVH, hd = 50, 2, 4, 2, 128
    qd, kvd = H * hd, KVH * hd
    ld = qd + 2 * kvd
    x = rbits(rng, (T * Bsz, ld), 1.0)
    xd = dev_bf16(x)
    table = torch.empty(T * hd // 2 * 2, dtype=torch.float32, device="cuda")
    B.pb_op_rope(ptr(xd), ld, 0, T * Bsz, Bsz, T, H, KVH, hd, qd, 1e4, ptr(table), stream())
    torch.cuda.synchronize()
    got = bf16_bits_to_f64(host_bits(xd))
    xf = bf16_bits_to_f64(x)
    for b in range(Bsz):
        rows = np.arange(T) * Bsz + b
        rq = OF.rope(xf[rows, :qd], H, hd, 1e4)
        rk = OF.rope(xf[rows, qd:qd + kvd], KVH, hd, 1e4)
        for g, r in ((got[rows, :qd], rq), (got[rows, qd:qd + kvd], rk)):
            assert np.all(np.abs(g - r) <= bf16_ulp(r) + 1e-6)
        assert np.array_equal(got[rows, qd + kvd:], xf[rows, qd + kvd:])


def test_argmax_large_vocab_ties_across_slices():
    """The argmax kernel splits a row over a cluster of CTAs: an exact tie between two slices resolves to the lowest
    index, the maximum in the last (ragged) slice is found, and a NaN anywhere raises the flag."""
    need_gpu()
    rng = np.random.default_rng(4)
    V = 50272
    lg = rng.standard_normal((3, V)).astype(np.float32)
    lg[0, 40000] = lg[0, 7] = 50.0          # tie across slices
    lg[1, V - 1] = 60.0                     # last element of the ragged last slice
    lg[2, 25000] = 70.0
    toks = torch.zeros(3, dtype=torch.int32, device="cuda")
    nan = torch.zeros(1, dtype=torch.int32, device="cuda")
    lgd = dev_f32(lg)
    B.pb_op_argmax(ptr(lgd), 3, V, V, ptr(toks), ptr(nan), stream())
    torch.cuda.synchronize()
    assert toks.cpu().tolist() == [7, V - 1, 25000] and nan.item() == 0
    lg[1, 33333] = np.nan
    lgd = dev_f32(lg)
    B.pb_op_argmax(ptr(lgd), 3, V, V, ptr(toks), ptr(nan), stream())
    torch.cuda.synchronize()
    assert nan.item() == 1


@pytest.mark.parametrize("Bsz,V", [(16, 1000), (64, 5000), (100, 777)])
def test_logits_large_batch_tensor_cores(Bsz, V):
    """B >= 16 takes the tcgen05 GEMM (S = 1): within fp32-accumulation error of the exact product, and vocab
    slices of any width give the same bits as the whole head (pipelined equals sequential)."""
    need_gpu()
    rng = np.random.default_rng(Bsz + V)
    d = 1024
    y = rbits(rng, (Bsz, d), 1.0)
    E = rbits(rng, (V, d), 0.035)
    Ed, yd = dev_bf16(E), dev_bf16(y)
    whole = torch.full((Bsz, V), float("nan"), device="cuda")
    B.pb_op_logits(ptr(yd), Bsz, d, ptr(Ed), 0, V, ptr(whole), V, stream())
    sliced = torch.full((Bsz, V), float("nan"), device="cuda")
    cut = V // 3 + 5
    B.pb_op_logits(ptr(yd), Bsz, d, ptr(Ed), cut, V, ptr(sliced), V, stream())
    B.pb_op_logits(ptr(yd), Bsz, d, ptr(Ed), 0, cut, ptr(sliced), V, stream())
    torch.cuda.synchronize()
    ref = bf16_bits_to_f64(y) @ bf16_bits_to_f64(E).T
    mag = np.abs(bf16_bits_to_f64(y)) @ np.abs(bf16_bits_to_f64(E)).T
    got = whole.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(got - ref) <= 4 * np.sqrt(d) * 2.0 ** -24 * mag + 1e-30)
    assert np.array_equal(whole.cpu().numpy().view(np.uint32), sliced.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("Bsz", [1, 2])
def test_logits_small_batch_gemv_vocab_slices(Bsz):
    """One or two sequences: the head as the weight-streaming GEMV; vocab slices give the bits of the whole head
    (pipelined equals sequential) and the values of y . E^T."""
    need_gpu()
    rng = np.random.default_rng(40 + Bsz)
    d, V = 2048, 5003
    y = rbits(rng, (Bsz, d), 1.0)
    E = rbits(rng, (V, d), 0.035)
    Ed, yd = dev_bf16(E), dev_bf16(y)
    whole = torch.full((Bsz, V), float("nan"), device="cuda")
    B.pb_op_logits(ptr(yd), Bsz, d, ptr(Ed), 0, V, ptr(whole), V, stream())
    sliced = torch.full((Bsz, V), float("nan"), device="cuda")
    for v0, v1 in ((0, 1237), (1237, 4000), (4000, V)):
        B.pb_op_logits(ptr(yd), Bsz, d, ptr(Ed), v0, v1, ptr(sliced), V, stream())
    torch.cuda.synchronize()
    assert torch.equal(whole, sliced)
    ref = bf16_bits_to_f64(y) @ bf16_bits_to_f64(E).T
    assert np.allclose(whole.cpu().numpy(), ref, rtol=1e-5, atol=1e-5)


def test_logits_argmax_embed():
    need_gpu()
    rng = np.random.default_rng(9)
    Bsz, d, V = 3, 512, 1000
    y = rbits(rng, (Bsz, d), 1.0)
    E = rbits(rng, (V, d), 0.035)
    logits = torch.full((Bsz, V), float("nan"), device="cuda")
    Ed, yd = dev_bf16(E), dev_bf16(y)
    B.pb_op_logits(ptr(yd), Bsz, d, ptr(Ed), 100, 1000, ptr(logits), V, stream())
    B.pb_op_logits(ptr(yd), Bsz, d, ptr(Ed), 0, 100, ptr(logits), V, stream())
    torch.cuda.synchronize()
    ref = bf16_bits_to_f64(y) @ bf16_bits_to_f64(E).T
    assert np.allclose(logits.cpu().numpy(), ref, rtol=1e-5, atol=1e-5)
    # argmax with an exact tie: lowest index wins
    lg = np.asarray(ref, dtype=np.float32)
    lg[1, 10] = lg[1, 900] = lg[1].max() + 1
    toks = torch.zeros(Bsz, dtype=torch.int32, device="cuda")
    nan = torch.zeros(1, dtype=torch.int32, device="cuda")
    lgd = dev_f32(lg)
    B.pb_op_argmax(ptr(lgd), Bsz, V, V, ptr(toks), ptr(nan), stream())
    torch.cuda.synchronize()
    assert toks.cpu().tolist() == [int(np.argmax(r)) for r in lg] and nan.item() == 0
    lg[2, 5] = np.nan
    lgd2 = dev_f32(lg)
    B.pb_op_argmax(ptr(lgd2), Bsz, V, V, ptr(toks), ptr(nan), stream())
    torch.cuda.synchronize()
    assert nan.item() == 1
    # embedding (+ OPT positions, offset 2), token-major rows
    T = 7
    P = rbits(rng, (T + 2, d), 0.035)
    tok = rng.integers(0, V, size=T * Bsz).astype(np.int32)
    h = torch.zeros((T * Bsz, d), device="cuda")
    Pd, tokd = dev_bf16(P), torch.from_numpy(tok).cuda()
    B.pb_op_embed(ptr(Ed), ptr(Pd), ptr(tokd), ptr(h), d, 0, T * Bsz, Bsz, stream())
    torch.cuda.synchronize()
    want = bf16_bits_to_f64(E)[tok] + bf16_bits_to_f64(P)[np.arange(T * Bsz) // Bsz + 2]
    assert np.array_equal(h.cpu().numpy(), want.astype(np.float32))
