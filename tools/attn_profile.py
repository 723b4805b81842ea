"""Standalone tensor-core attention launches at prefill shapes (for ncu / timing): C5a (Llama-2-70B, T=2048,
64 heads, 8 KV heads, hd 128), C4 (OPT-13B, T=1024, 40 heads, hd 128), C2 (OPT-1.3B, T=128, 32 heads, hd 64).
Prints per-launch device time (CUDA events, 10 launches after warm-up) and achieved TFLOP/s on causal pairs."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2503_17707_b200 import _binding as B

SHAPES = {"C5a": (2048, 64, 8, 128), "C4": (1024, 40, 40, 128), "C2": (128, 32, 32, 64)}


def run(tag, reps=10):
    T, H, KVH, hd = SHAPES[tag]
    qd, kvd = H * hd, KVH * hd
    ld = qd + 2 * kvd
    qkv = (torch.randn(T, ld, device="cuda") * 0.5).to(torch.bfloat16)
    out = torch.empty(T, qd, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    go = lambda: B.pb_op_attention(qkv.data_ptr(), ld, out.data_ptr(), qd, 0, T, 1, H, KVH, hd, qd, qd + kvd,
                                   hd ** -0.5, s)
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        go()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    flops = 4.0 * (T * (T + 1) / 2) * H * hd
    print(f"{tag}: T={T} H={H} KVH={KVH} hd={hd}: {us:8.1f} us  {flops / us / 1e6:7.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    for tag in (sys.argv[1:] or list(SHAPES)):
        run(tag)
