"""Diagnostic: one C2 cold start on one GPU with the per-launch trace; prints when each layer's
chunks land vs when its kernels run."""
import os, sys, json
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("PB_LANDED_TIMING", "1")   # per-chunk landed timestamps
sys.path.insert(0, ".")
import numpy as np, torch
import harness, synth
from paper_2503_17707_b200 import _binding as B
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import WORKLOADS
w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
cb = int(sys.argv[2]) if len(sys.argv) > 2 else 32
plan = Plan(w.model, w.adapters, 1, chunk_bytes=cb << 20)
base, ada = harness.build_host_images(plan)
eng = RankEngine(plan, 0, base, ada, max_batch=w.batch, max_seq=w.seq)
B.pb_ctx_set_profiling(eng.ctx, 1)
toks = synth.tokens(w.batch, w.seq, w.model.vocab)
import time
for ep in range(1, 5):
    eng.invalidate()
    t0 = time.perf_counter()
    eng.enqueue(ep, toks, w.batch, w.seq, 0)
    t1 = time.perf_counter()
    eng.wait()
    t2 = time.perf_counter()
tl = eng.timeline()
print(f"host enqueue {1e3*(t1-t0):.2f} ms, total host {1e3*(t2-t0):.2f} ms; ttft {tl['ttft_ms']:.2f} ready {tl['t_ready_ms']:.2f} load_done {tl['load_done_ms']:.2f}")
tens = plan.tensors()
# per layer: last landed chunk time
dump = plan.dump().splitlines()
chunks = [l for l in dump if l.startswith("chunk ")]
land = tl["chunk_landed_ms"]
per_layer = {}
for ln in chunks:
    f = ln.split()
    cid = int(f[1]); kind = f[2]; tid = int(f[3].split("=")[1])
    if kind != "base":
        continue
    layer = tens[tid][4]
    per_layer[layer] = max(per_layer.get(layer, 0), land[cid])
tr = B.pb_kernel_trace(eng.ctx)
gem = [t for t in tr if t[0] in ("gemm", "attention", "norm")]
print("n trace", len(tr))
# layer kernels: 7 per layer in order (norm, gemm, attn, gemm, norm, gemm, gemm)
comp = [t for t in tr if t[0] in ("gemm", "attention", "norm", "embed", "logits", "argmax")]
print("embed", [t for t in tr if t[0] == "embed"])
for l in range(w.model.n_layers):
    ks = comp[1 + 7 * l: 1 + 7 * l + 7]
    print(f"L{l:2d} landed {per_layer.get(l, -1):7.2f}  compute {ks[0][1]:7.2f} -> {ks[-1][2]:7.2f}  ({ks[-1][2]-ks[0][1]:.3f} ms)")
print("tail", [t for t in tr if t[0] in ("logits", "argmax")], "non-layer ready", per_layer.get(-1))
merges = [t for t in tr if t[0] == "merge"]
print("merges first/last", merges[:2], merges[-2:])
