"""Split-K factor sweep of the plain split-K GEMM at the C2 (M = 128) shapes: 30 back-to-back launches with
programmatic dependent launch in one CUDA graph (as in the prefill), weights rotated through > 300 MB, one event
pair around the replay on the replaying stream. Prints us per launch and weight GB/s per (shape, S)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17707_b200 import _binding as B  # noqa: E402

SHAPES = [("qkv", 2048, 6144, 0), ("o", 2048, 2048, 1), ("fc1", 2048, 8192, 0), ("fc2", 8192, 2048, 1)]


def bench(M, K, N, epi, split, reps=30):
    nbuf = max(2, int(300e6 // (N * K * 2)) + 1)
    X = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    Ws = [(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(nbuf)]
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)
    B.pb_op_debug_gemm(None, 1)   # PDL on, no trace

    def go(i, st):
        B.pb_op_gemm_split(X.data_ptr(), M, 0, M, K, Ws[i % nbuf].data_ptr(), N, N, epi, 0, 0, 1.0, 0, out.data_ptr(),
                           N, split, st)

    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        for i in range(2):
            go(i, cs.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        for i in range(reps):
            go(i, cs.cuda_stream)
    B.pb_op_debug_gemm(None, 0)
    best = 1e9
    for _ in range(3):
        st = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / reps)
    return best, N * K * 2 / best / 1e3


for name, K, N, epi in SHAPES:
    res = {}
    for S in (0, 2, 4, 8):
        if S and K // 64 < 2 * S:
            continue
        us, gbs = bench(128, K, N, epi, S)
        res["auto" if S == 0 else f"S{S}"] = [round(us, 2), round(gbs)]
    print(json.dumps({"shape": name, "K": K, "N": N, "us_gbs": res}), flush=True)
