"""Sweep of the skinny split-K GEMM (M <= 128) over (S, NT) at the C2 projection shapes (OPT-1.3B, T = 128), next to
the plain split-K kernel the path used before (run with PB_SKINNY=0: "auto" is then that kernel). CUDA graph of 30 launches,
weights rotated through > 300 MB so they stream from HBM; one event pair around the graph. Prints a table and
one JSON line per shape with the best shape and the model's pick (gemm_skinny_shape via pb_op_gemm)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17707_b200 import _binding as B  # noqa: E402

SHAPES = [("qkv", 2048, 6144, 0), ("o", 2048, 2048, 1), ("fc1", 2048, 8192, 0), ("fc2", 8192, 2048, 1),
          ("l7_qkv", 4096, 12288, 0), ("l7_gate_up", 4096, 11008, 2), ("l7_down", 11008, 4096, 1)]


def bench(M, K, N, epi, fn, reps=30):
    rows = 2 * N if epi == 2 else N
    nbuf = max(2, int(300e6 // (rows * K * 2)) + 1)
    X = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    Ws = [(torch.randn(rows, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(nbuf)]
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)

    def go(i, st):
        fn(X.data_ptr(), M, 0, M, K, Ws[i % nbuf].data_ptr(), rows, N, epi, out.data_ptr(), N, st)

    cs = torch.cuda.Stream()
    for i in range(2):
        go(i, cs.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        for i in range(reps):
            go(i, cs.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / reps)
    return best, rows * K * 2 / best / 1e3


def main():
    M = int(os.environ.get("SWEEP_M", "128"))
    for name, K, N, epi in SHAPES:
        res = {}

        def skinny(S, NT):
            return lambda X, m, a, b, K, W, r, N, e, o, ldo, st: B.pb_op_gemm_skinny(
                X, m, a, b, K, W, r, N, e, 0, 0, 1.0, 0, o, ldo, S, NT, st)

        auto = lambda X, m, a, b, K, W, r, N, e, o, ldo, st: B.pb_op_gemm(  # noqa: E731
            X, m, a, b, K, W, r, N, e, 0, 0, 1.0, 0, o, ldo, st)
        res["auto"] = bench(M, K, N, epi, auto)
        if os.environ.get("PB_SKINNY") == "0":   # the plain split-K kernel's numbers only
            print(json.dumps({"shape": name, "M": M, "plain_kernel_us": round(res["auto"][0], 2),
                              "plain_kernel_gbs": round(res["auto"][1])}), flush=True)
            continue
        for S in (1, 2, 4, 8, 16):
            if K // 64 < 2 * S:
                continue
            for NT in (1, 2, 4):
                per = 64 if epi == 2 else 128
                ctas = -(-(-(-N // per)) // NT) * S
                if ctas > 148:
                    continue
                res[f"S{S}NT{NT}"] = bench(M, K, N, epi, skinny(S, NT))
        best = min((v[0], k) for k, v in res.items() if k != "auto")
        print(f"{name:10s} M{M} K{K} N{N}: " + " ".join(f"{k}={v[0]:.1f}us/{v[1]:.0f}GB/s" for k, v in res.items()),
              flush=True)
        print(json.dumps({"shape": name, "M": M, "K": K, "N": N, "epi": epi, "auto_us": round(res["auto"][0], 2),
                          "auto_gbs": round(res["auto"][1]), "best": best[1], "best_us": round(best[0], 2)}),
              flush=True)


if __name__ == "__main__":
    main()
