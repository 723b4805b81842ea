"""Fixed overhead vs streaming slope of the GEMM: time vs K at M=128 (graph-captured launches)."""
import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from gemm_bench import bench
for N in (8192, 2048):
    for S in (1, 2, 4):
        row = []
        for K in (128, 256, 512, 1024, 2048, 4096, 8192):
            if S > K // 64: continue
            us, gbs, tf = bench(128, K, N, 0, S)
            row.append(f"K{K}:{us:5.1f}")
        print(f"N{N} S{S}: " + " ".join(row), flush=True)
