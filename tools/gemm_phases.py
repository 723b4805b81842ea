"""Where does a C2 (M = 128) projection's time go? Phase stamps (%globaltimer, pb_op_debug_gemm) of every CTA of the
split-K kernel, for back-to-back launches in a CUDA graph with programmatic dependent launch (as in the prefill),
weights rotated through > 300 MB so they stream from HBM. Per launch (the middle ones of the sequence), relative to
the previous launch's last CTA end: when CTAs enter, finish the prologue, pass the activation wait, see their first
stage land, finish the MMAs, pass the partial-exchange barrier, finish the epilogue. Prints one JSON line per shape.

    python tools/gemm_phases.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17707_b200 import _binding as B  # noqa: E402

SHAPES = [("qkv", 2048, 6144, 0), ("o", 2048, 2048, 1), ("fc1", 2048, 8192, 0), ("fc2", 8192, 2048, 1)]
PHASES = ["entry", "prologue", "x_wait", "loads_issued", "first_stage", "mma_done", "partials", "epilogue"]


def run(M, K, N, epi, reps=12, pdl=1):
    nbuf = max(2, int(300e6 // (N * K * 2)) + 1)
    X = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    Ws = [(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(nbuf)]
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)
    maxcta = 512
    tr = torch.zeros(reps, maxcta, 8, dtype=torch.int64, device="cuda")
    cs = torch.cuda.Stream()

    def go(i, st):
        B.pb_op_debug_gemm(tr[i].data_ptr(), pdl)
        B.pb_op_gemm(X.data_ptr(), M, 0, M, K, Ws[i % nbuf].data_ptr(), N, N, epi, 0, 0, 1.0, 0, out.data_ptr(), N, st)

    for i in range(2):
        go(i, cs.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        for i in range(reps):
            go(i, cs.cuda_stream)
    B.pb_op_debug_gemm(None, 0)
    g.replay()
    torch.cuda.synchronize()
    tr.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    g.replay()
    e1.record(cs)
    torch.cuda.synchronize()
    per_launch_us = e0.elapsed_time(e1) * 1e3 / reps
    t = tr.cpu().numpy().astype(np.float64)
    res = []
    for i in range(3, reps - 1):
        ctas = t[i][t[i][:, 0] > 0]
        prev = t[i - 1][t[i - 1][:, 0] > 0]
        ref = prev[:, 7].max()          # previous launch's last CTA done
        rel = (ctas - ref) / 1e3        # us
        res.append({p: [float(np.min(rel[:, k])), float(np.median(rel[:, k])), float(np.max(rel[:, k]))]
                    for k, p in enumerate(PHASES)})
        res[-1]["ctas"] = int(len(ctas))
    avg = {p: [float(np.mean([r[p][j] for r in res])) for j in range(3)] for p in PHASES}
    return per_launch_us, avg, res[0]["ctas"]


def main():
    for name, K, N, epi in SHAPES:
        for pdl in (1, 0):
            us, avg, ctas = run(128, K, N, epi, pdl=pdl)
            print(json.dumps({"shape": name, "K": K, "N": N, "pdl": pdl, "ctas": ctas, "graph_us_per_launch": round(us, 2),
                              "phases_us_vs_prev_end [min, median, max]": {p: [round(x, 2) for x in v]
                                                                        for p, v in avg.items()}}), flush=True)


if __name__ == "__main__":
    main()
