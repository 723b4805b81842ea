"""Bit-exact fraction of each path kernel against the storage contract (correct rounding of the fp64 value) at
Llama-2-7B layer shapes: how often does fp32 arithmetic on the GPU flip a bf16 rounding?"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import forward as OF  # noqa: E402
from oracle.numerics import bf16_bits_to_f64, f64_to_bf16_bits, rne_bf16, rne_f32  # noqa: E402
from paper_2503_17707_b200 import _binding as B  # noqa: E402


def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)


def host(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


s = torch.cuda.current_stream().cuda_stream
rng = np.random.default_rng(0)
out = {}
for M in (16, 512):
    K, N, F = 4096, 12288, 11008
    x = f64_to_bf16_bits(rng.standard_normal((M, K)))
    w = f64_to_bf16_bits(rng.uniform(-0.0346, 0.0346, (N, K)))
    o = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
    xd, wd = dev(x), dev(w)
    B.pb_op_gemm(xd.data_ptr(), M, 0, M, K, wd.data_ptr(), N, N, 0, 0, 0, 1.0, 0, o.data_ptr(), N, s)
    torch.cuda.synchronize()
    ref = rne_bf16(bf16_bits_to_f64(x) @ bf16_bits_to_f64(w).T)
    out[f"gemm_bf16_M{M}"] = float((bf16_bits_to_f64(host(o)) == ref).mean())
    # SiLU * up
    wg = f64_to_bf16_bits(rng.uniform(-0.0346, 0.0346, (2 * F, K)))
    o2 = torch.zeros((M, F), dtype=torch.bfloat16, device="cuda")
    wgd = dev(wg)
    B.pb_op_gemm(xd.data_ptr(), M, 0, M, K, wgd.data_ptr(), 2 * F, F, 2, 0, 0, 1.0, 0, o2.data_ptr(), F, s)
    torch.cuda.synchronize()
    gu = bf16_bits_to_f64(x) @ bf16_bits_to_f64(wg).T
    g, u = gu[:, :F], gu[:, F:]
    ref2 = rne_bf16(g / (1 + np.exp(-g)) * u)
    out[f"gemm_silu_M{M}"] = float((bf16_bits_to_f64(host(o2)) == ref2).mean())
    # residual (fp32)
    mh = f64_to_bf16_bits(rng.standard_normal((M, F)))
    wdn = f64_to_bf16_bits(rng.uniform(-0.0346, 0.0346, (K, F)))
    h0 = rng.standard_normal((M, K)).astype(np.float32)
    hd_ = torch.from_numpy(h0).cuda()
    mhd, wdnd = dev(mh), dev(wdn)
    B.pb_op_gemm(mhd.data_ptr(), M, 0, M, F, wdnd.data_ptr(), K, K, 1, 0, 0, 1.0, 0, hd_.data_ptr(), K, s)
    torch.cuda.synchronize()
    ref3 = rne_f32(h0.astype(np.float64) + bf16_bits_to_f64(mh) @ bf16_bits_to_f64(wdn).T)
    got3 = hd_.cpu().numpy().astype(np.float64)
    out[f"gemm_resid_M{M}_exact"] = float((got3 == ref3).mean())
    out[f"gemm_resid_M{M}_maxrel"] = float((np.abs(got3 - ref3) / (np.abs(ref3) + 1e-30)).max())
    # RMSNorm
    gam = f64_to_bf16_bits(rng.uniform(0.9, 1.1, K))
    on = torch.zeros((M, K), dtype=torch.bfloat16, device="cuda")
    gd = dev(gam)
    B.pb_op_norm(hd_.data_ptr(), M, K, gd.data_ptr(), None, 1e-5, on.data_ptr(), s)
    torch.cuda.synchronize()
    hh = got3
    ref4 = rne_bf16(OF.rms_norm(hh, bf16_bits_to_f64(gam), 1e-5))
    out[f"rmsnorm_M{M}"] = float((bf16_bits_to_f64(host(on)) == ref4).mean())
# attention at T = 16 / 512, 32 heads hd 128
for T in (16, 512):
    H, hd = 32, 128
    qkv = f64_to_bf16_bits(rng.standard_normal((T, 3 * H * hd)) * 1.3)
    o = torch.zeros((T, H * hd), dtype=torch.bfloat16, device="cuda")
    qd = dev(qkv)
    B.pb_op_attention(qd.data_ptr(), 3 * H * hd, o.data_ptr(), H * hd, 0, T, 1, H, H, hd, H * hd, 2 * H * hd,
                      hd ** -0.5, s)
    torch.cuda.synchronize()
    xq = bf16_bits_to_f64(qkv)
    con = rne_bf16(OF.causal_attention(xq[:, :H * hd], xq[:, H * hd:2 * H * hd], xq[:, 2 * H * hd:], H, H, hd,
                                       hd ** -0.5, rne_bf16))
    out[f"attention_T{T}"] = float((bf16_bits_to_f64(host(o)) == con).mean())
print(json.dumps(out, indent=1))
