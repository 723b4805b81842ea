import numpy as np, torch, sys
sys.path.insert(0, "tests")
from gpu_util import dev_bf16, host_bits, ptr, stream
from oracle.numerics import bf16_bits_to_f64, f64_to_bf16_bits
from paper_2503_17707_b200 import _binding as B
rng = np.random.default_rng(0)
for (M, K, N) in [(128, 64, 128), (128, 128, 128), (128, 256, 128), (128, 256, 256)]:
    X = f64_to_bf16_bits(rng.uniform(-1, 1, (M, K)))
    W = f64_to_bf16_bits(rng.uniform(-1, 1, (N, K)))
    out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    B.pb_op_gemm(ptr(dev_bf16(X)), M, 0, M, K, ptr(dev_bf16(W)), N, N, 1, 0, 0, 1.0, 0, ptr(out), N, stream())
    torch.cuda.synchronize()
    g = out.cpu().numpy().astype(np.float64)
    x, w = bf16_bits_to_f64(X), bf16_bits_to_f64(W)
    ref = x @ w.T
    err = np.abs(g - ref)
    print(f"M{M} K{K} N{N}: max err {err.max():.3g}  bad frac {(err > 1e-3).mean():.3f}")
    bad_rows = np.where((err > 1e-3).any(1))[0]; bad_cols = np.where((err > 1e-3).any(0))[0]
    print("  bad rows", bad_rows[:10], len(bad_rows), " bad cols", bad_cols[:10], len(bad_cols))
    # hypotheses
    for name, h in [("first kblock only", x[:, :64] @ w[:, :64].T),
                    ("last kblock only", x[:, -64:] @ w[:, -64:].T),
                    ("first 16 k", x[:, :16] @ w[:, :16].T)]:
        print(f"  {name}: {np.abs(g - h).max():.3g}")
    if K >= 128:
        for kb in range(K // 64):
            sl = slice(kb * 64, kb * 64 + 64)
            print(f"   kb{kb} corr", np.corrcoef((g).ravel(), (x[:, sl] @ w[:, sl].T).ravel())[0, 1])
    # per 16-k slice correlation within first kblock
    for ks in range(4):
        sl = slice(ks * 16, ks * 16 + 16)
        print(f"   kslice{ks} corr", round(np.corrcoef(g.ravel(), (x[:, sl] @ w[:, sl].T).ravel())[0, 1], 3))
