"""Is the in-step kernel slowdown a clock effect? Sample SM clock via NVML every ~0.5 ms during C2 cold
starts, with and without a background keep-alive kernel."""
import os, sys, threading, time, json
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ".")
import numpy as np, torch, pynvml
import harness, synth
from paper_2503_17707_b200 import _binding as B
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import WORKLOADS
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
w = WORKLOADS["C2"]
plan = Plan(w.model, w.adapters, 1, chunk_bytes=64 << 20)
base, ada = harness.build_host_images(plan)
eng = RankEngine(plan, 0, base, ada, max_batch=w.batch, max_seq=w.seq)
B.pb_ctx_set_profiling(eng.ctx, 1)
toks = synth.tokens(w.batch, w.seq, w.model.vocab)
samples = []
stop = False
def sampler():
    while not stop:
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
        time.sleep(0.0005)
def run(ep, keep=False):
    global stop, samples
    eng.invalidate()
    side = torch.cuda.Stream()
    if keep:
        with torch.cuda.stream(side):
            x = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
            for _ in range(200): y = x @ x   # ~ busy for the whole trial
    samples = []; stop = False
    t = threading.Thread(target=sampler); t.start()
    t0 = time.perf_counter()
    eng.cold_start(ep, toks, w.batch, w.seq, 0)
    stop = True; t.join()
    torch.cuda.synchronize()
    st = B.pb_kernel_stats(eng.ctx)
    clk = [c for (tt, c) in samples]
    return eng.timeline()["ttft_ms"], {k: round(v["total_ms"] / max(1, v["launches"]) * 1e3, 1) for k, v in st.items() if v["launches"]}, (min(clk), int(np.median(clk)), max(clk), len(clk))
for ep in range(1, 4):
    print("plain", run(ep))
for ep in range(4, 6):
    print("keepalive", run(ep, keep=True))
