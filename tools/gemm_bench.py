"""Microbenchmark of the prefill GEMM on the C2 (OPT-1.3B, T=128) projection shapes and larger M,
for several split-K factors. CUDA events around 30 back-to-back launches; weights > L2 rotated."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2503_17707_b200 import _binding as B

def bench(M, K, N, epi, split, reps=30):
    nbuf = max(2, int(300e6 // (N * K * 2 * (2 if epi == 2 else 1))) + 1)   # rotate weights so they come from HBM
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Ws = [torch.randn((2 * N if epi == 2 else N), K, device="cuda").to(torch.bfloat16) * 0.02 for _ in range(nbuf)]
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    def go(i):
        nonlocal s
        W = Ws[i % nbuf]
        B.pb_op_gemm_split(X.data_ptr(), M, 0, M, K, W.data_ptr(), W.shape[0], N, epi, 0, 0, 1.0, 0, out.data_ptr(), N,
                           split, s)
    for i in range(3): go(i)
    torch.cuda.synchronize()
    # capture the launches in a CUDA graph so host-side map encoding does not starve the GPU
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        s = cs.cuda_stream
        for i in range(reps): go(i)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    # per-launch CUDA events back to back (the way bench.py times kernels)
    s = torch.cuda.current_stream().cuda_stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i in range(reps):
        evs[i][0].record()
        go(i)
        evs[i][1].record()
    torch.cuda.synchronize()
    global LAST_EV_US
    LAST_EV_US = sum(x.elapsed_time(y) for x, y in evs) * 1e3 / reps
    wbytes = (2 * N if epi == 2 else N) * K * 2
    flops = 2 * M * (2 * N if epi == 2 else N) * K
    return us, wbytes / us / 1e3, flops / us / 1e6

if __name__ == "__main__":
  shapes = [("qkv", 128, 2048, 6144, 0), ("o", 128, 2048, 2048, 1), ("fc1", 128, 2048, 8192, 0), ("fc2", 128, 8192, 2048, 1),
            ("c4_qkv_M1024", 1024, 5120, 15360, 0), ("c4_o_M1024", 1024, 5120, 5120, 1),
            ("c4_fc1_M1024", 1024, 5120, 20480, 0), ("c4_fc2_M1024", 1024, 20480, 5120, 1),
            ("c5_fc1_M2048", 2048, 8192, 28672, 2), ("c3_qkv_M512", 512, 4096, 12288, 0)]
  import os
  only_big = os.environ.get("GEMM_BENCH_BIG")
  if os.environ.get("GEMM_BENCH_GEMV"):   # M = 1 (decode): the weight-streaming GEMV, split 0 only
      for name, M, K, N, epi in [("qkv", 1, 2048, 6144, 0), ("o", 1, 2048, 2048, 1), ("fc1", 1, 2048, 8192, 0),
                                 ("fc2", 1, 8192, 2048, 1), ("c4_fc1", 1, 5120, 20480, 0), ("c4_fc2", 1, 20480, 5120, 1),
                                 ("l70_gate_up", 1, 8192, 28672, 2)]:
          us, gbs, tf = bench(M, K, N, epi, 0)
          print(f"{name:14s} M{M} K{K} N{N}: graph {us:6.1f}us {gbs:5.0f}GB/s ev {LAST_EV_US:6.1f}us", flush=True)
      sys.exit(0)
  if os.environ.get("GEMM_BENCH_SMALLM"):   # is the activation (X) operand's L2 traffic what limits M = 128?
      for name, M0, K, N, epi in shapes[:4]:
          res = []
          for M in (16, 32, 64, 128):
              us, gbs, tf = bench(M, K, N, epi, 0)
              res.append(f"M{M}: {us:6.1f}us {gbs:5.0f}GB/s")
          print(f"{name:6s} K{K} N{N} auto split: " + " | ".join(res), flush=True)
      sys.exit(0)
  for name, M, K, N, epi in shapes:
      if only_big and M <= 128: continue
      res = []
      for split in ((0, 1, 2, 4, 8) if M <= 256 else ((0,) if only_big else (0, 1, 2))):
          if split and split > K // 64: continue
          us, gbs, tf = bench(M, K, N, epi, split)
          res.append(f"S={split}: graph {us:6.1f}us {gbs:5.0f}GB/s {tf:5.0f}TF ev {LAST_EV_US:6.1f}us")
      print(f"{name:14s} M{M} K{K} N{N}: " + " | ".join(res), flush=True)
