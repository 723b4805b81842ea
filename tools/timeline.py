"""Device timeline of a cold start and of the warm prefill, recorded with CUPTI through torch.profiler (kineto).

Nsight Systems is not installed in this image; CUPTI activity records give the same device-side facts: every
H2D copy (copy-engine lane), every kernel of the path (merge stream, compute stream; PDL overlap included) with
its start / end on the device clock. Writes a Chrome / Perfetto trace (gzip) and prints a JSON summary:
  * cold start: H2D GB/s over the load window, merges overlapped with the load, last byte landed -> first token
  * warm prefill (the single-GPU replay after T_full, CUDA graph): per kernel class count / total / mean
    duration, and the idle gaps between consecutive kernels of the compute stream (launch + dependency latency)

    python tools/timeline.py [--workload C2] [--out profiles/r02_timeline_C2_N1.json.gz]
"""
import argparse
import collections
import gzip
import json
import os
import shutil
import sys
import tempfile

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import harness  # noqa: E402
import synth  # noqa: E402
from paper_2503_17707_b200.api import Plan, RankEngine  # noqa: E402
from synth.configs import WORKLOADS  # noqa: E402

CLASSES = [("gemm", "gemm"), ("merge", "merge"), ("attention", "attention"), ("norm", "norm"), ("logits", "logits"),
           ("argmax", "argmax"), ("embed", "embed"), ("rope", "rope"), ("signal", "signal"), ("copy16", "copy"),
           ("feed_tokens", "tokens"), ("set_words", "words")]


def kclass(name):
    for pat, c in CLASSES:
        if pat in name:
            return c
    return "other"


def summarise(events, t_lo, t_hi):
    ks = [e for e in events if e.get("cat") == "kernel" and t_lo <= e["ts"] <= t_hi]
    cp = [e for e in events if e.get("cat") in ("gpu_memcpy", "gpu_memset") and t_lo <= e["ts"] <= t_hi]
    cls = collections.defaultdict(lambda: {"n": 0, "total_us": 0.0})
    for e in ks:
        c = cls[kclass(e["name"])]
        c["n"] += 1
        c["total_us"] += e["dur"]
    for c in cls.values():
        c["mean_us"] = c["total_us"] / max(1, c["n"])
    h2d = [e for e in cp if "HtoD" in e["name"]]
    out = {"kernels": dict(cls)}
    if h2d:
        t0 = min(e["ts"] for e in h2d)
        t1 = max(e["ts"] + e["dur"] for e in h2d)
        nbytes = sum(e.get("args", {}).get("bytes", 0) for e in h2d)
        out["h2d"] = {"copies": len(h2d), "bytes": nbytes, "window_us": t1 - t0,
                      "gbs": nbytes / max(t1 - t0, 1e-9) / 1e3}
    # compute-stream gaps: the stream carrying the gemm kernels
    gs = [e for e in ks if kclass(e["name"]) == "gemm"]
    if gs:
        stream = collections.Counter(e["args"].get("stream") for e in gs).most_common(1)[0][0]
        seq = sorted([e for e in ks if e["args"].get("stream") == stream], key=lambda e: e["ts"])
        gaps = [max(0.0, b["ts"] - (a["ts"] + a["dur"])) for a, b in zip(seq, seq[1:])]
        overl = [max(0.0, (a["ts"] + a["dur"]) - b["ts"]) for a, b in zip(seq, seq[1:])]
        out["compute_stream"] = {"kernels": len(seq), "span_us": seq[-1]["ts"] + seq[-1]["dur"] - seq[0]["ts"],
                                 "busy_us": sum(e["dur"] for e in seq), "gap_total_us": sum(gaps),
                                 "gap_mean_us": sum(gaps) / max(1, len(gaps)),
                                 "pdl_overlap_total_us": sum(overl)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--chunk-mb", type=int, default=128)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    plan = Plan(w.model, w.adapters, 1, chunk_bytes=args.chunk_mb << 20)
    base, ada = harness.build_host_images(plan)
    eng = RankEngine(plan, 0, base, ada, max_batch=w.batch, max_seq=w.seq)
    toks = synth.tokens(w.batch, w.seq, w.model.vocab)
    for ep in (1, 2):   # warm-up: module load, graph capture of the replay
        eng.invalidate()
        eng.cold_start(3 * ep, toks, adapter_id=0 if w.adapters else -1)
        eng.replay_enqueue(3 * ep + 1, toks, w.batch, w.seq)
        eng.wait()
    eng.invalidate()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        with torch.profiler.record_function("cold_start"):
            eng.cold_start(10, toks, adapter_id=0 if w.adapters else -1)
        torch.cuda.synchronize()
        with torch.profiler.record_function("warm_prefill"):
            eng.replay_enqueue(11, toks, w.batch, w.seq)
            eng.wait()
        torch.cuda.synchronize()
    tmp = tempfile.mktemp(suffix=".json")
    prof.export_chrome_trace(tmp)
    tr = json.load(open(tmp))
    ev = tr["traceEvents"] if isinstance(tr, dict) else tr
    marks = {e["name"]: e for e in ev if e.get("cat") == "user_annotation"}
    gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    cs, wp = marks.get("cold_start"), marks.get("warm_prefill")
    # device events are attributed to the phase whose host window launched them: cold start = everything before the
    # first device event of the warm phase's launches
    tl = eng.timeline()
    res = {"workload": args.workload, "ttft_ms": tl["ttft_ms"], "load_done_ms": tl["load_done_ms"]}
    if cs and wp:
        dev_ts = sorted(e["ts"] for e in gpu)
        split = wp["ts"]
        res["cold_start"] = summarise(gpu, dev_ts[0], split)
        res["warm_prefill"] = summarise(gpu, split, dev_ts[-1] + 1)
    out = args.out or f"gpurun_out/timeline_{args.workload}_N1.json.gz"
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(tmp, "rb") as fi, gzip.open(out, "wb") as fo:
        shutil.copyfileobj(fi, fo)
    os.unlink(tmp)
    res["trace"] = out
    print(json.dumps(res, indent=1))
    eng.close()


if __name__ == "__main__":
    main()
