"""C3 timeline: per layer, when its chunks land, when its merges run, when its compute runs."""
import os, sys
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("PB_LANDED_TIMING", "1")   # per-chunk landed timestamps
sys.path.insert(0, ".")
import numpy as np, torch, harness, synth
from paper_2503_17707_b200 import _binding as B
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import WORKLOADS
w = WORKLOADS["C3"]
plan = Plan(w.model, w.adapters, 1, chunk_bytes=64 << 20)
base, ada = harness.build_host_images(plan)
eng = RankEngine(plan, 0, base, ada, max_batch=w.batch, max_seq=w.seq, multi_adapter=True)
toks = synth.tokens(w.batch, w.seq, w.model.vocab)
aos = [0, 1, 2, 3]
for ep in range(1, 4):
    B.pb_ctx_set_profiling(eng.ctx, 1 if ep == 3 else 0)
    eng.invalidate()
    eng.enqueue(ep, toks, w.batch, w.seq, adapter_id=-2, adapter_of_seq=aos)
    eng.wait()
tl = eng.timeline()
print(f"ttft {tl['ttft_ms']:.1f} ready {tl['t_ready_ms']:.1f} full {tl['t_full_ms']:.1f} load_done {tl['load_done_ms']:.1f}")
tr = B.pb_kernel_trace(eng.ctx)
merges = [t for t in tr if t[0] == "merge"]
comp = [t for t in tr if t[0] in ("gemm", "attention", "norm", "rope")]
print("merge launches", len(merges), "first", merges[:2], "last", merges[-2:])
per = len(merges) // 32
for l in (0, 1, 2, 10, 20, 30, 31):
    ms = merges[l * per:(l + 1) * per]
    print(f"L{l}: merges {ms[0][1]:.1f}->{ms[-1][2]:.1f} ({sum(t[2]-t[1] for t in ms):.2f} ms busy)")
print("compute first", comp[0], "last", comp[-1], "n", len(comp), "sum", sum(t[2]-t[1] for t in comp))
dump = plan.dump().splitlines()
tens = plan.tensors()
land = tl["chunk_landed_ms"]
lay = {}
for ln in dump:
    if ln.startswith("chunk ") and " base " in ln:
        f = ln.split(); cid = int(f[1]); tid = int(f[3].split("=")[1]); l = tens[tid][4]
        if land[cid] >= 0: lay[l] = max(lay.get(l, 0), land[cid])
print("landed", {l: round(lay[l], 1) for l in (0, 1, 2, 10, 20, 30, 31)})
