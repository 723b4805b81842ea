"""Vocabulary-head microbenchmark at one sequence (the cold start's first token): pb_op_logits on the C2 / C4 / C5a
head shapes, 20 launches back to back in a CUDA graph (heads of 206-524 MB stream from HBM each launch), one event
pair. PB_LOGITS_GEMV=0 selects the warp-per-row logits kernel instead of the weight-streaming GEMV (A/B)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_17707_b200 import _binding as B  # noqa: E402

SHAPES = {"C2": (50272, 2048), "C4": (50272, 5120), "C5a": (32000, 8192)}


def run(tag, bsz=1, reps=20):
    V, d = SHAPES[tag]
    E = (torch.randn(V, d, device="cuda") * 0.02).to(torch.bfloat16)
    y = torch.randn(bsz, d, device="cuda").to(torch.bfloat16)
    out = torch.empty(bsz, V, device="cuda", dtype=torch.float32)
    for _ in range(2):
        B.pb_op_logits(y.data_ptr(), bsz, d, E.data_ptr(), 0, V, out.data_ptr(), V,
                       torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cs = torch.cuda.current_stream().cuda_stream
        for _ in range(reps):
            B.pb_op_logits(y.data_ptr(), bsz, d, E.data_ptr(), 0, V, out.data_ptr(), V, cs)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    print(f"{tag}: B={bsz} V={V} d={d}: {us:7.1f} us  {V * d * 2 / us / 1e3:6.0f} GB/s", flush=True)


if __name__ == "__main__":
    for tag in (sys.argv[1:] or list(SHAPES)):
        run(tag)
