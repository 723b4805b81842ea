#!/usr/bin/env python
"""bench.py — cold-start TTFT of the PipeBoost layer-sharded cold start on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU)

A step = one whole cold start: the weights buffer of every GPU is put in an
explicit cold state (0xFF, untimed), then plan-ordered H2D load of each GPU's shard -> LoRA merge ->
NVLink gather -> pipelined first-token prefill, until the first token is in host memory.
  value      = TTFT ms, device clock (t0 event before the first DMA -> token D2H complete), max over ranks
  e2e        = the same cold start timed by the host around the public API call (RankEngine.cold_start),
               barrier -> token in host memory; bytes moved H2D/D2H per step stated
  roofline   = dominant SM kernel class vs MEASURED_PEAKS.json: the GEMM class timed back to back as one CUDA graph
               of the step's projections (one event pair per replay; roofline.event_timed_frac = the same class
               with a CUDA-event pair around every launch of the warm prefill), other classes per-launch events
  pcie_roofline = the path's own bound: S / sum of measured concurrent H2D GB/s (TTFT >= that)
The CPU oracle (oracle/, the only other place it runs) is timed on rank 0 on a bounded sample.
Inputs (2.6 GB of weights at C2) are far larger than the 126 MB L2; weights are re-invalidated each step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

METRIC = "cold-start TTFT (ms) and aggregate load GB/s vs PCIe roofline at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--policy", default=None, choices=[None, "stage", "interleave"])
    ap.add_argument("--vocab-sliced", type=int, default=None)
    ap.add_argument("--chunk-mb", type=int, default=None,
                    help="DMA group / merge granularity; default 128 on one GPU (measured on B200, C2: 16/32/64/128/256 MB"
                         " -> 0.965/0.971/0.981/0.988/0.988 of the PCIe bound: every group boundary costs a landed-event"
                         " record on the saturated link), 64 with several GPUs (finer stage / gather interleave)")
    ap.add_argument("--prefill-chunks", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--cpu-sample-layers", type=int, default=0,
                    help="decoder layers the CPU oracle baseline runs (0 = the whole model when it fits ~30 s of "
                         "CPU work — C1, C2 — else 4 layers extrapolated linearly)")
    ap.add_argument("--ref-sample-layers", type=int, default=0,
                    help="--impl reference: decoder layers per step (0 = the whole model where one oracle pass is "
                         "~30 s of CPU work at most, else a 4-layer sample extrapolated to the model)")
    ap.add_argument("--host-alias", type=int, default=0,
                    help="host_alias_layers K: layer l is DMA'd from the host image of layer l mod K (DRAM-limited boxes)")
    ap.add_argument("--dist-backend", default="nccl", help="torch.distributed backend for barriers/handle exchange")
    ap.add_argument("--same-gpu", action="store_true", help="all ranks on cuda:0 (testing the N>1 path on one GPU)")
    ap.add_argument("--check-oracle", type=int, default=1,
                    help="1 (default): after the timed steps, one more (untimed) cold start whose first-token logits "
                         "are compared with the stored full-depth oracle (tests/golden/oracle_<workload>[_K<k>].npz, "
                         "written by tools/oracle_reference.py from oracle/ only); adds 'parity' to the line")
    args = ap.parse_args()
    # the same defaults on both arms (the reference arm reports this configuration too)
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    from synth.configs import WORKLOADS
    w = WORKLOADS[args.workload]
    if args.policy is None:
        args.policy = "stage" if (world == 1 or len(w.adapters) > 1) else "interleave"
    if args.vocab_sliced is None:
        args.vocab_sliced = 0 if world == 1 else 1
    if args.prefill_chunks is None:
        args.prefill_chunks = 1 if world == 1 else 2
    if args.chunk_mb is None:
        args.chunk_mb = 128 if world == 1 else 64
    return args


# ----------------------------------------------------------------------------------------------------
# CPU oracle timing (reported baseline; --impl reference)
# ----------------------------------------------------------------------------------------------------

class OracleSample:
    """The CPU oracle (merge + sequential forward, bf16 storage contract) on embed + `sample_layers` decoder layers +
    head of workload `w`. prepare() materialises the seeded weights (untimed: a CPU 'cold start' has no load step);
    run() times the merge and the forward once and returns (ms for all L layers, detail) — measured when the sample
    is the whole model, else extrapolated linearly in layers (labelled)."""

    def __init__(self, w, sample_layers: int):
        self.w = w
        self.nl = min(sample_layers, w.model.n_layers)

    def prepare(self):
        import oracle
        import synth
        w = self.w
        m, ads = w.model, w.adapters
        self.ls = list(range(self.nl))
        ow = oracle.OracleWeights(m, ads)
        names = [n for n in ow.tensors if not n.startswith("L") or int(n[1:].split(".")[0]) in self.ls]
        self.base = {n: ow.base_bits(n) for n in names}
        n_ad = len(ads)
        self.aos = [b % n_ad for b in range(w.batch)] if n_ad > 1 else [0 if n_ad else None] * w.batch
        self.used = sorted({a for a in self.aos if a is not None})
        self.facs = [at for at in ow.atensors if at.adapter in self.used and at.layer in self.ls]
        self.fac_bits = {at.name: ow.adapter_bits(at) for at in self.facs}
        self.toks = synth.tokens(w.batch, w.seq, m.vocab)
        self.ow = ow
        # fp64 copies of the weights no merge touches: the oracle's resident input data, widened once (untimed);
        # a merged tensor is widened again every step (part of the timed work)
        from oracle.numerics import bf16_bits_to_f64
        id2name = {t.id: n for n, t in ow.tensors.items()}
        self.touched = {id2name[at.base] for at in self.facs}
        self.base64 = {}
        for n, bits in self.base.items():
            if n not in self.touched:
                x = bf16_bits_to_f64(bits)
                self.base64[n] = x.reshape(-1) if ow.tensors[n].rows == 1 else x
        return self

    def run(self):
        from oracle import forward as OF
        from oracle.merge import merge_bf16_bits
        from oracle.numerics import bf16_bits_to_f64
        import threadpoolctl  # noqa: F401  (numpy BLAS threads = all cores by default)
        w, ow = self.w, self.ow
        m, ads = w.model, w.adapters
        L = m.n_layers
        id2name = {t.id: n for n, t in ow.tensors.items()}
        t0 = time.perf_counter()
        merged = {a: dict(self.base) for a in self.used} if self.used else {None: dict(self.base)}
        for a in self.used:
            by_target = {}
            for at in self.facs:
                if at.adapter == a:
                    by_target.setdefault((at.layer, at.target), {})[at.factor] = at
            for (l, tgt), f in by_target.items():
                name = id2name[f["A"].base]
                W = merged[a][name].copy()
                r0, rows = f["A"].row0, f["B"].rows
                W[r0:r0 + rows] = merge_bf16_bits(W[r0:r0 + rows], self.fac_bits[f["B"].name],
                                                  self.fac_bits[f["A"].name], ads[a].scale)
                merged[a][name] = W
        t_merge = time.perf_counter() - t0
        wf = {}

        def getter(a):
            def Wget(n):
                if n in self.base64:
                    return self.base64[n]
                if (a, n) not in wf:
                    x = bf16_bits_to_f64(merged[a][n])
                    wf[(a, n)] = x.reshape(-1) if ow.tensors[n].rows == 1 else x
                return wf[(a, n)]
            return Wget

        tc = time.perf_counter()
        for a in merged:   # the oracle computes in fp64: widening the merged tensors is part of its work
            for n in merged[a]:
                if n not in self.base64:
                    getter(a)(n)
        t_conv = time.perf_counter() - tc
        t1 = time.perf_counter()
        for b in range(w.batch):
            OF.forward_logits(m, getter(self.aos[b]), self.toks[b], "bf16", layers=[])
        t_head = time.perf_counter() - t1
        t2 = time.perf_counter()
        for b in range(w.batch):
            OF.forward_logits(m, getter(self.aos[b]), self.toks[b], "bf16", layers=self.ls)
        t_all = time.perf_counter() - t2
        nls = len(self.ls)
        if nls == L:   # the whole model: the measured time itself
            total_s = t_merge + t_conv + t_all
            per_layer = max(t_all - t_head, 0.0) / nls
        else:
            per_layer = max(t_all - t_head, 0.0) / nls
            total_s = t_head + L * (per_layer + (t_merge + t_conv) / nls)
        detail = {"sample_layers": nls, "layers": L, "merge_s_per_layer": t_merge / nls,
                  "fp64_widen_s_per_layer": t_conv / nls, "forward_s_per_layer": per_layer, "embed_head_s": t_head,
                  "measured_s": t_merge + t_conv + t_head + t_all}
        return total_s * 1e3, detail


def _forward_flops(w):
    return 2.0 * w.batch * w.seq * 2.0 * w.model.n_layers * (4 * w.model.d_model ** 2 + 3 * w.model.d_model *
                                                               w.model.d_ffn)


def default_sample_layers(w):
    """cpu_baseline (one run): the whole model when one oracle pass is ~30 s of CPU work at most (C1, C2: ~0.3 TFLOP
    of fp64), else 4 layers (extrapolated, labelled)."""
    return w.model.n_layers if _forward_flops(w) < 1.2e12 else 4


def reference_sample_layers(w):
    """--impl reference runs K + W steps (the driver's 20 + 5): each step a bounded sample, ~3-5 s of CPU work at C2
    (6 of 24 layers + embed/head, extrapolated linearly in layers and labelled), the whole model only when it is
    tiny (C1)."""
    return w.model.n_layers if _forward_flops(w) < 5e10 else min(6, w.model.n_layers)


def oracle_sample(w, sample_layers: int):
    return OracleSample(w, sample_layers).prepare().run()


def cpu_cores():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth.configs import WORKLOADS
    w = WORKLOADS[args.workload]
    sample = OracleSample(w, args.ref_sample_layers or reference_sample_layers(w)).prepare()
    vals, walls = [], []
    det = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        v, det = sample.run()
        if i >= args.warmup:
            vals.append(v)
            walls.append((time.perf_counter() - t0) * 1e3)
    val = statistics.mean(vals)
    extrap = det["sample_layers"] < det["layers"]
    desc = (f"{det['sample_layers']} of {det['layers']} layers + embed/head, B={w.batch} T={w.seq}"
            + (", extrapolated linearly in layers (value); ms_per_step = the sample actually run per step"
               if extrap else ", whole model every step (merge + forward; weights materialised once, untimed)"))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(walls),
            "extrapolated": extrap, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (bf16 storage contract)",
            "data": "synthetic (seeded splitmix64; HF init std 0.02)",
            "config": workload_config(w, args, 1),
            "cpu_baseline": {"value": val, "unit": "ms", "cores": cpu_cores(), "kind": "oracle", "sample": desc,
                             "detail": det},
            "e2e": {"value": val, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(w, args, n):
    return {"workload": f"{w.tag}: {w.note}, L={w.model.n_layers} d={w.model.d_model}, "
                        f"LoRA r={w.adapters[0].rank if w.adapters else 0} on {','.join(w.adapters[0].targets) if w.adapters else '-'}",
            "batch": w.batch, "seq_len": w.seq, "n_gpus": n,
            "policy": args.policy, "vocab_sliced": args.vocab_sliced, "chunk_mb": args.chunk_mb,
            "prefill_chunks": args.prefill_chunks, "host_alias_layers": args.host_alias,
            "l2": "inputs (whole model weights) larger than the 126 MB L2; device weights reset to 0xFF between steps",
            "parallelism": f"pp{n} (layer-sharded load, pipelined prefill)"}


# ----------------------------------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------------------------------

class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.lines = []

    def start(self):
        """Starts nvidia-smi sampling every 100 ms and returns once it is producing samples (its start-up takes up to
        ~1 s, longer than a short timed region), so every sample kept was taken inside the timed region."""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.time() + 10
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.02)
            self.lines.clear()   # samples from before the timed region
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
                pw.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        thr = max(pw) * 0.5 if pw else 0
        load = [s for s, w in zip(sm, pw) if w >= thr] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw)}


# ----------------------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------------------

def measure_h2d(nbytes=2 << 30, chunk=128 << 20):
    """Concurrent pinned H2D GB/s of this rank's GPU on the load's own lane shape: ONE stream, copies of the load's
    group size (chunk), 2 GiB, best of 4 after a warm-up (all ranks at once): the PCIe roofline constant."""
    import torch
    chunk = max(1 << 20, min(chunk, nbytes))
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    best = 0.0
    for r in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for off in range(0, nbytes, chunk):
                dev[off:off + chunk].copy_(host[off:off + chunk], non_blocking=True)
            e1.record(st)
        torch.cuda.synchronize()
        if r:
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del host, dev
    return best


def ncu_traffic(kernel_class, workload):
    """dram bytes (read + write) per launch of the kernel class at this workload, from the committed ncu --set full
    capture of that workload (None when there is none)."""
    p = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(workload, {}).get(kernel_class)


def load_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6534.5), d.get("bf16_tflops", 1664.9), d.get("bf16_tflops_sustained", 1389.1), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def time_merges(eng, plan, w, reps=3):
    """a3 merge kernel in the bench line: every adapted tensor of adapter 0 merged once more, warm,
    out of place into a rotating scratch region larger than the 126 MB L2 (the resident weights are not touched),
    the launches captured as one CUDA graph and timed with one CUDA-event pair per replay on the capture stream.
    Algorithmic work per launch: 4 B per W element (read + write) + the factors; 2*rows*cols*r
    flop. Returns the kernels[] entry (or None without adapters)."""
    import torch
    from paper_2503_17707_b200 import _binding as B
    if not w.adapters:
        return None
    pairs = {}
    layer_of = [t[4] for t in plan.tensors()]
    for (name, rows, cols, off, a, is_b, bt, r0) in plan.atensors():
        if a == 0:
            pairs.setdefault((bt, r0), {})["B" if is_b else "A"] = (rows, cols, off)
            pairs[(bt, r0)]["layer"] = layer_of[bt]
    jobs = [(f["B"][0], f["A"][1], f["A"][0], f["A"][2], f["B"][2], f["layer"]) for f in pairs.values()]
    if not jobs:
        return None
    biggest = max(r * c * 2 for r, c, _, _, _, _ in jobs)
    cap = max(320 << 20, 2 * biggest)
    scratch = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    ada = eng.adapters.data_ptr()
    scale = w.adapters[0].scale
    nbytes = flops = 0.0
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    # one launch per layer (<= 8 adapted tensors), as the cold start merges the adapted chunks of a DMA group
    by_layer = {}
    for j in jobs:
        by_layer.setdefault(j[5], []).append(j)
    launches = 0
    with torch.cuda.graph(g):
        cs = torch.cuda.current_stream()
        off = 0
        for lj in by_layer.values():
            for k in range(0, len(lj), 8):
                batch = lj[k:k + 8]
                Wp = []
                for rows, cols, rank, a_off, b_off, _ in batch:
                    sz = (rows * cols * 2 + 255) // 256 * 256
                    if off + sz > cap:
                        off = 0
                    Wp.append(scratch.data_ptr() + off)
                    off += sz
                    nbytes += 4.0 * rows * cols + 2.0 * rank * (rows + cols)
                    flops += 2.0 * rows * cols * rank
                B.pb_op_merge_batch(Wp, [j[1] for j in batch], [j[0] for j in batch], [j[1] for j in batch],
                                    [ada + j[4] for j in batch], [ada + j[3] for j in batch], batch[0][2],
                                    [scale] * len(batch), cs.cuda_stream)
                launches += 1
    g.replay()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.current_stream()
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = statistics.mean(ms)
    del g, scratch
    torch.cuda.empty_cache()
    return {"launches": launches, "avg_us": 1e3 * t / launches, "ms_per_step": t, "bytes": nbytes, "flops": flops,
            "timing": "warm re-merge of every adapted tensor of adapter 0 into a rotating scratch region (> L2), "
                      "one pb_op_merge_batch launch per layer (its adapted tensors), one CUDA graph, one event pair "
                      "per replay (mean of 3); not inside the cold start, where merges overlap the PCIe load on "
                      "their own stream"}


def time_gemms(eng, plan, w, stage, reps=3):
    """The GEMM class without per-launch timing events: the step's projections of this rank's stage (QKV, O, FC1 |
    gate_up, FC2 | down of every layer, in prefill order, on the resident weights, M = B*T rows, the prefill's kernel
    choice, epilogue and programmatic dependent launch) replayed back to back as one CUDA graph, one CUDA-event pair
    per replay on the capture stream; the launch's activations come from scratch buffers (the values do not change
    the work). A per-launch event pair in the warm replay adds ~5 us of event overhead per launch and cancels the
    programmatic-dependent-launch overlap the prefill runs with; both numbers are reported.
    Algorithmic work per launch as pb_kernel_stats counts it: 2*M*N_w*K flop; X + W + output bytes."""
    import torch
    from paper_2503_17707_b200 import _binding as B
    m = w.model
    opt = m.arch == "opt"
    M = w.batch * w.seq
    d, f, hd = m.d_model, m.d_ffn, m.head_dim
    tens = {t[0]: t for t in plan.tensors()}
    wp = eng.weights.data_ptr()
    kmax = max(d, f)
    X = torch.zeros((M, kmax), dtype=torch.bfloat16, device="cuda")
    nmax = max(tens["L0.qkv"][1], tens["L0." + ("fc1" if opt else "gate_up")][1], d)
    out = torch.zeros((M, nmax), dtype=torch.float32, device="cuda")
    table = torch.zeros(max(1, w.seq * hd // 2 * 8), dtype=torch.uint8, device="cuda") if not opt else None
    flops = nbytes = 0.0
    launches = 0
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    B.pb_op_debug_gemm(None, 1)   # programmatic dependent launch, as the prefill launches them
    try:
        with torch.cuda.graph(g):
            cs = torch.cuda.current_stream().cuda_stream
            for l in range(stage[0], stage[1]):
                L = f"L{l}."
                projs = [("qkv", 0), ("o", 1), ("fc1" if opt else "gate_up", 0 if opt else 2), ("fc2" if opt else "down", 1)]
                for name, epi in projs:
                    _, rows, K, _, _, off = tens[L + name]
                    N = rows // 2 if epi == 2 else rows
                    bias = wp + tens[L + name + "_b"][5] if opt and (L + name + "_b") in tens else 0
                    if name == "qkv" and not opt:
                        qd = m.n_heads * hd
                        B.pb_op_gemm_rope(X.data_ptr(), M, 0, M, K, wp + off, N, out.data_ptr(), N,
                                          qd + m.n_kv_heads * hd, hd, 0, w.batch, w.seq, m.rope_theta,
                                          table.data_ptr(), 0, cs)
                    else:
                        B.pb_op_gemm(X.data_ptr(), M, 0, M, K, wp + off, rows, N, epi, bias,
                                     1 if name == "fc1" else 0, 1.0 / hd ** 0.5 if name == "qkv" else 1.0,
                                     d if name == "qkv" else 0, out.data_ptr(), N, cs)
                    launches += 1
                    flops += 2.0 * M * rows * K
                    nbytes += 2.0 * M * K + 2.0 * rows * K + (8.0 if epi == 1 else 2.0) * M * N
    finally:
        B.pb_op_debug_gemm(None, 0)
    g.replay()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.current_stream()
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = statistics.mean(ms)
    del g, X, out
    torch.cuda.empty_cache()
    return {"launches": launches, "avg_us": 1e3 * t / launches, "ms_per_step": t, "bytes": nbytes, "flops": flops,
            "timing": "the stage's projections back to back as one CUDA graph (PDL, the prefill's kernels and "
                      "shapes, resident weights), one event pair per replay (mean of 3)"}


def self_launch(args):
    """`python bench.py --gpus N` with N > 1 outside torchrun: re-launch this command as N processes, one per GPU,
    through torch.distributed.run on 127.0.0.1 (the same launch line the driver uses), and exit with its code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    if args.same_gpu and args.dist_backend == "nccl":
        args.dist_backend = "gloo"   # NCCL refuses two ranks on one device; gloo carries the host-side plumbing
    import torch
    import torch.distributed as dist

    import harness
    import synth
    from paper_2503_17707_b200 import _binding as B
    from paper_2503_17707_b200.api import Plan, RankEngine, pinned_host
    from synth.configs import WORKLOADS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    dev = 0 if args.same_gpu else local
    if dev >= torch.cuda.device_count():
        sys.exit(f"bench.py: rank {rank} needs cuda:{dev} but {torch.cuda.device_count()} GPU(s) are visible "
                 f"(--same-gpu runs every rank on cuda:0 for testing)")
    init = {}   # init breakdown, excluded from t0 ("Load Model Ckpt" / "Init Meta")
    ti = time.perf_counter()
    torch.cuda.set_device(dev)
    torch.empty(1, device="cuda")
    init["cuda_context"] = (time.perf_counter() - ti) * 1e3
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(args.dist_backend)

    def barrier():
        if world > 1:
            dist.barrier()

    red_dev = "cuda" if args.dist_backend == "nccl" else "cpu"

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t)
        return t.item()

    w = WORKLOADS[args.workload]
    ti = time.perf_counter()
    plan = Plan(w.model, w.adapters, world, policy=args.policy, vocab_sliced=args.vocab_sliced,
                chunk_bytes=args.chunk_mb << 20, prefill_chunks=args.prefill_chunks, host_alias_layers=args.host_alias)
    init["plan"] = (time.perf_counter() - ti) * 1e3
    ti = time.perf_counter()
    S = plan.sizes.dev_weight_bytes + plan.sizes.dev_adapter_bytes   # bytes DMA'd per cold start (all ranks)

    # --- host images: one DRAM copy of the checkpoint shared by all GPU processes
    shm_paths = []
    if world == 1:
        base, ada = harness.build_host_images(plan)
    else:
        # base image and (4 KiB-aligned after it) the adapter image in ONE shared file, registered once: the copy
        # lane then streams from one registered host range (as harness.build_host_images does in one process)
        path = f"/dev/shm/pipeboost_{args.workload}_{os.getppid()}_img"
        off = (plan.sizes.host_base_bytes + 4095) // 4096 * 4096
        total = off + max(plan.sizes.host_adapter_bytes, 1)
        if local == 0:
            img = torch.from_file(path, shared=True, size=total, dtype=torch.uint8)
            harness.fill_host_images(plan, img.data_ptr(), img.data_ptr() + off)
        barrier()
        img = torch.from_file(path, shared=True, size=total, dtype=torch.uint8)
        torch.cuda.cudart().cudaHostRegister(img.data_ptr(), total, 0)
        shm_paths = [path]
        base, ada = img[:plan.sizes.host_base_bytes], img[off:off + max(plan.sizes.host_adapter_bytes, 1)]

    init["host_image_pin_fill"] = (time.perf_counter() - ti) * 1e3
    multi = len(w.adapters) > 1   # C3: several adapters share the base, one sequence per adapter (PB_MERGE_ALL)
    ti = time.perf_counter()
    eng = RankEngine(plan, rank, base, ada if plan.sizes.host_adapter_bytes else None, max_batch=w.batch,
                     max_seq=w.seq, multi_adapter=multi)
    init["device_alloc_and_ctx"] = (time.perf_counter() - ti) * 1e3
    adapter_id = B.PB_MERGE_ALL if multi else (0 if w.adapters else -1)
    aos = [b % len(w.adapters) for b in range(w.batch)] if multi else None
    if world > 1:
        blobs = [None] * world
        dist.all_gather_object(blobs, eng.export())
        eng.wire_ipc(blobs)
    toks = synth.tokens(w.batch, w.seq, w.model.vocab)

    barrier()
    h2d_gbs = measure_h2d(chunk=args.chunk_mb << 20)   # all ranks concurrently: the PCIe roofline constant
    barrier()
    agg_h2d = allsum(h2d_gbs)

    clocks = ClockSampler()
    ttft, e2e, ready, full, load_done, warm, launches = [], [], [], [], [], [], 0
    recv_gbs, load_gbs_rank, stage_span = [], [], []
    kstats = {}
    out_tokens = out_logits = None
    for step in range(args.warmup + args.steps):
        timed = step >= args.warmup
        eng.invalidate()
        if timed and step == args.warmup and rank == 0:
            clocks.start()
        barrier()
        torch.cuda.synchronize()
        th0 = time.perf_counter()
        eng.enqueue(3 * step + 1, toks if rank == 0 else None, w.batch, w.seq, adapter_id=adapter_id,
                    adapter_of_seq=aos)
        last = step == args.warmup + args.steps - 1
        res = eng.wait()
        th1 = time.perf_counter()
        barrier()
        torch.cuda.synchronize()
        tl = eng.timeline()
        if rank == 0:
            out_tokens = res[0]

        if timed:
            ttft.append(allmax(tl["ttft_ms"]))
            e2e.append(allmax((th1 - th0) * 1e3))
            ready.append(allmax(tl["t_ready_ms"]))
            full.append(allmax(tl["t_full_ms"]))
            load_done.append(allmax(tl["load_done_ms"]))
            # NVLink ingress of this rank over its receive window (t0 -> its T_full), summed over ranks
            recv_gbs.append(allsum(tl["recv_bytes"] / max(tl["t_full_ms"], 1e-6) / 1e6))
            load_gbs_rank.append(allmax(tl["load_bytes"] / max(tl["load_done_ms"], 1e-6) / 1e6))
            stage_span.append(allmax(max(0.0, tl["stage_end_ms"] - tl["stage_begin_ms"])))
            launches += int(allsum(tl["n_launches"]))
            # warm prefill on the now-resident weights, no per-kernel events: the pipelined prefill alone
            # (the single-GPU-resident regime after T_full), device clock t0 -> token D2H
            barrier()
            eng.replay_enqueue(3 * step + 2, toks if rank == 0 else None, w.batch, w.seq)
            eng.wait()
            barrier()
            warm.append(allmax(eng.timeline()["ttft_ms"]))
            if not args.no_profile:
                # Kernel timing: the same prefill kernels re-run on the now-resident weights, each bracketed by
                # CUDA events on its launching stream. (Inside the cold start the PCIe link is saturated and a
                # timing-event record costs ~20 us, which would swamp 5-50 us kernels.)
                B.pb_ctx_set_profiling(eng.ctx, 1)
                barrier()
                eng.replay_enqueue(3 * step + 3, toks if rank == 0 else None, w.batch, w.seq)
                eng.wait()
                B.pb_ctx_set_profiling(eng.ctx, 0)
                barrier()
                for k, v in B.pb_kernel_stats(eng.ctx).items():
                    a = kstats.setdefault(k, {"launches": 0, "total_ms": 0.0, "flops": 0.0, "bytes": 0.0})
                    for f in a:
                        a[f] += v[f]
    clk = clocks.stop() if rank == 0 else None
    gold = harness.load_golden(w.tag, args.host_alias) if args.check_oracle else None
    if args.check_oracle:   # parity: one more cold start, outside the timed region, its logits to the host
        ep_chk = 3 * (args.warmup + args.steps) + 1
        eng.invalidate()
        barrier()
        eng.enqueue(ep_chk, toks if rank == 0 else None, w.batch, w.seq, adapter_id=adapter_id, adapter_of_seq=aos)
        chk = eng.wait(want_logits=gold is not None)
        barrier()
        if rank == 0:
            out_tokens, out_logits = chk
    merge_k = time_merges(eng, plan, w) if (rank == 0 and not args.no_profile) else None
    # rank 0's stage: contiguous balanced stages, remainder to the lower ranks
    L_, base_, rem_ = w.model.n_layers, w.model.n_layers // world, w.model.n_layers % world
    gemm_k = time_gemms(eng, plan, w, (0, base_ + (1 if rem_ > 0 else 0)) if world > 1 else (0, L_)) \
        if (rank == 0 and not args.no_profile) else None
    # prefill tensor-core FLOPs per step over all ranks (each rank profiles its own stage) for T_comp
    my_flops = sum(kstats.get(k, {}).get("flops", 0.0) for k in ("gemm", "attention")) / max(1, args.steps)
    all_flops = allsum(my_flops)

    if rank == 0:
        hbm, bf16_burst, bf16_sus, peak_src = load_peaks()
        val = statistics.mean(ttft)
        # dominant SM kernel class over the timed steps
        roof = None
        kern = {}
        for k, a in kstats.items():
            if a["launches"] == 0:
                continue
            t = a["total_ms"] * 1e-3
            # binding resource = the larger of (flops / tensor peak) and (bytes / HBM peak)
            # GEMMs and attention are tensor-core contractions; the rest are memory / latency-bound row kernels
            tensor_bound = k in ("gemm", "attention") and a["flops"] / (bf16_sus * 1e12) > a["bytes"] / (hbm * 1e9)
            if tensor_bound:
                ach, peak, unit = a["flops"] / t / 1e12, bf16_sus, "TFLOP/s"
            else:
                ach, peak, unit = a["bytes"] / t / 1e9, hbm, "GB/s"
            kern[k] = {"launches": a["launches"] // max(1, args.steps), "avg_us": 1e3 * a["total_ms"] / a["launches"],
                       "ms_per_step": a["total_ms"] / args.steps, "achieved": ach, "unit": unit, "frac": ach / peak,
                       "tflops": a["flops"] / t / 1e12, "gbs": a["bytes"] / t / 1e9}
        if merge_k is not None:
            t = merge_k["ms_per_step"] * 1e-3
            ach = merge_k["bytes"] / t / 1e9
            kern["merge"] = {"launches": merge_k["launches"], "avg_us": merge_k["avg_us"],
                             "ms_per_step": merge_k["ms_per_step"], "achieved": ach, "unit": "GB/s",
                             "frac": ach / hbm, "tflops": merge_k["flops"] / t / 1e12, "gbs": ach,
                             "timing": merge_k["timing"]}
        if gemm_k is not None and "gemm" in kern:
            # the GEMM class timed back to back (no per-launch events): the same tensor-core / HBM choice as above
            t = gemm_k["ms_per_step"] * 1e-3
            gk = kern["gemm"]
            tensor_bound = gemm_k["flops"] / (bf16_sus * 1e12) > gemm_k["bytes"] / (hbm * 1e9)
            ach = gemm_k["flops"] / t / 1e12 if tensor_bound else gemm_k["bytes"] / t / 1e9
            gk["event_timed"] = {"avg_us": gk["avg_us"], "achieved": gk["achieved"], "frac": gk["frac"],
                                 "timing": "CUDA events per launch on the launching stream, warm re-run of the "
                                           "step's prefill (pb_prefill_replay) after each timed cold start"}
            # timed alone (a replay of at most ~1 s, not inside the long step): the burst bf16 peak applies
            gk.update({"avg_us": gemm_k["avg_us"], "ms_per_step": gemm_k["ms_per_step"] * gk["launches"] / max(1, gemm_k["launches"]),
                       "achieved": ach, "unit": "TFLOP/s" if tensor_bound else "GB/s",
                       "frac": ach / (bf16_burst if tensor_bound else hbm), "tflops": gemm_k["flops"] / t / 1e12,
                       "gbs": gemm_k["bytes"] / t / 1e9, "timing": gemm_k["timing"],
                       "peak": bf16_burst if tensor_bound else hbm,
                       "peak_kind": "burst bf16" if tensor_bound else "HBM copy"})
        # the dominant kernel of the step's critical path: the prefill classes (the merge overlaps the load)
        sm_kernels = {k: v for k, v in kern.items() if k not in ("signal", "merge")}
        if sm_kernels:
            dom = max(sm_kernels, key=lambda k: sm_kernels[k]["ms_per_step"])
            d = sm_kernels[dom]
            pk = d.get("peak", bf16_sus if d["unit"] == "TFLOP/s" else hbm)
            pkind = d.get("peak_kind", "sustained bf16" if d["unit"] == "TFLOP/s" else "HBM copy")
            roof = {"kernel": dom, "bound": "tensor" if d["unit"] == "TFLOP/s" else "hbm", "achieved": d["achieved"],
                    "peak": pk, "unit": d["unit"], "frac": d["achieved"] / pk,
                    "traffic": ncu_traffic(dom, w.tag),
                    "peak_source": f"{peak_src} ({pkind})",
                    "timing": d.get("timing", "CUDA events per launch on the launching stream, warm re-run of the "
                                              "step's prefill (pb_prefill_replay) after each timed cold start")}
            if "event_timed" in d:
                roof["event_timed_frac"] = d["event_timed"]["frac"]
        load_gbs = S / (statistics.mean(load_done) * 1e-3) / 1e9
        # the link's capability: the measured pinned copy rate, or the load's own rate where that was faster (with
        # host_alias_layers the load re-reads a few GB of host image and can beat the 2 GiB measurement)
        link_gbs = max(agg_h2d, load_gbs)
        t_pcie = S / (link_gbs * 1e9) * 1e3
        # roofline = max(T_pcie, T_nv, T_comp). T_nv: every GPU ingests (N-1)/N of S over NVLink
        # (900 GB/s per direction nominal, B200 NVLink 5); T_comp: the prefill FLOPs spread over N GPUs at the
        # measured sustained tensor peak (the serial chain is a scheduling hazard, not a bound).
        nv_peak = 900.0
        t_nv = ((world - 1) / world) * S / (nv_peak * 1e9) * 1e3 if world > 1 else 0.0
        t_comp = all_flops / (world * bf16_sus * 1e12) * 1e3
        bound = max(t_pcie, t_nv, t_comp)
        line = {
            "metric": METRIC, "value": val, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": val, "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded splitmix64 values, HF init std 0.02; random-init OPT/Llama shapes)",
            "config": workload_config(w, args, world),
            "e2e": {"value": statistics.mean(e2e), "unit": "ms", "h2d_bytes_per_step": int(S + toks.nbytes),
                    "d2h_bytes_per_step": int(4 * w.batch)},
            "gpu_launches": launches,
            "clocks": clk,
            "roofline": roof,
            "pcie_roofline": {"bound_ms": bound, "bound": ("pcie" if bound == t_pcie else
                                                            "nvlink" if bound == t_nv else "compute"),
                              "t_pcie_ms": t_pcie, "t_nv_ms": t_nv, "t_comp_ms": t_comp, "bytes": S,
                              "h2d_gbs_per_gpu_measured": h2d_gbs, "h2d_gbs_aggregate": agg_h2d,
                              "h2d_measured_on": f"one stream, {args.chunk_mb} MB copies (the load's lane and group size)",
                              "link_gbs_used": link_gbs,
                              "frac": bound / val, "load_gbs_aggregate": load_gbs,
                              "load_frac_of_measured_link": load_gbs / agg_h2d,
                              "load_gbs_per_gpu_max": statistics.mean(load_gbs_rank),
                              "nvlink_recv_gbs_aggregate": statistics.mean(recv_gbs) if world > 1 else 0.0,
                              "nvlink_peak_gbs_per_gpu": nv_peak if world > 1 else None,
                              "nvlink_bytes": int((world - 1) * S) if world > 1 else 0},
            "ttft_breakdown_ms": {"t_ready": statistics.mean(ready), "t_full": statistics.mean(full),
                                  "load_done": statistics.mean(load_done), "ttft_min": min(ttft),
                                  "ttft_median": statistics.median(ttft),
                                  "prefill_warm": statistics.mean(warm),
                                  "stage_span_max": statistics.mean(stage_span)},
            "kernels": kern,
            "init_breakdown_ms": dict(init, ctx_create=eng.timeline()["ctx_create_ms"],
                                      note="host wall clock, rank 0, before t0; not part of TTFT"),
            "first_tokens": [int(x) for x in out_tokens],
        }
        if args.check_oracle:
            if gold is None:
                line["parity"] = {"unavailable": f"no {os.path.relpath(harness.golden_path(w.tag, args.host_alias), HERE)}"}
            else:
                rep = harness.golden_parity(gold, out_logits, out_tokens)
                line["parity"] = {"rel": rep["max_rel"], "rel_exact": rep.get("max_rel_exact"),
                                  "token_ok": all(rep["token_ok"]), "token_exact_match": all(rep["token_exact_match"]),
                                  "min_margin": min(rep["margin"]), "gate": rep["gate"], "ok": rep["ok"],
                                  "oracle": os.path.relpath(harness.golden_path(w.tag, args.host_alias), HERE)}
        if not args.no_cpu_baseline:
            # whole model when it is ~30 s of CPU work at most (C1, C2: one fp64 forward ~2 x 0.3 TFLOP), else a
            # 4-layer sample extrapolated linearly
            nl = args.cpu_sample_layers or default_sample_layers(w)
            v, det = oracle_sample(w, nl)
            whole = det["sample_layers"] == det["layers"]
            line["cpu_baseline"] = {"value": v, "unit": "ms", "cores": cpu_cores(), "kind": "oracle",
                                    "sample": f"{det['sample_layers']} of {det['layers']} layers + embed/head, "
                                              f"B={w.batch} T={w.seq}"
                                              + (", whole model, timed once" if whole else
                                                 ", extrapolated linearly in layers"),
                                    "extrapolated": not whole, "detail": det}
        print(json.dumps(line), flush=True)
    barrier()
    eng.close()
    if world > 1:
        for p in shm_paths:
            if local == 0 and os.path.exists(p):
                os.unlink(p)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
