"""f3 measurement — decode after the cold start, one B200.

    python tools/decode_bench.py [--workload C2] [--steps 32] [--batch 1]

Cold start (OPT-1.3B + LoRA by default), then `steps` greedy decode steps of the same batch; each step's device
time (t0 event -> new tokens in host memory, pb_timeline ttft_ms) against the step's HBM bound (every weight
byte read once: a decode step is weight streaming at M = batch rows). Also the replica mode (the same GPU after
T_full serving a new batch alone; identical here since N = 1, reported for the API path). One JSON line.
"""
import argparse
import json
import os
import statistics
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import harness  # noqa: E402
import synth  # noqa: E402
from paper_2503_17707_b200.api import Plan, RankEngine  # noqa: E402
from synth.configs import WORKLOADS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    w = WORKLOADS[a.workload]
    plan = Plan(w.model, w.adapters, 1, chunk_bytes=64 << 20)
    base, ada = harness.build_host_images(plan)
    toks = synth.tokens(a.batch, w.seq, w.model.vocab)
    eng = RankEngine(plan, 0, base, ada, max_batch=a.batch, max_seq=w.seq + a.steps + 1)
    eng.wire_local([eng])
    eng.invalidate()
    eng.cold_start(1, toks, adapter_id=0)
    ttft = eng.timeline()["ttft_ms"]
    step_ms, out = [], []
    for i in range(a.steps):
        eng.decode_enqueue(2 + i)
        t, _ = eng.wait()
        out.append(int(t[0]))
        step_ms.append(eng.timeline()["ttft_ms"])
    eng.set_replica(True)
    eng.replay_enqueue(100, toks, a.batch, w.seq)
    eng.wait()
    rep_ms = []
    for i in range(a.steps):
        eng.decode_enqueue(101 + i)
        t, _ = eng.wait()
        rep_ms.append(eng.timeline()["ttft_ms"])
    peaks = json.load(open(os.path.join(HERE, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(HERE, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    wbytes = plan.sizes.dev_weight_bytes
    bound_ms = wbytes / (peaks["hbm_gbs"] * 1e9) * 1e3
    med = statistics.median(step_ms[2:])
    line = {"metric": "f3 decode ms/token after the cold start", "workload": a.workload, "batch": a.batch,
            "prompt": w.seq, "steps": a.steps, "ttft_ms": ttft, "decode_ms_median": med,
            "decode_ms_min": min(step_ms), "replica_decode_ms_median": statistics.median(rep_ms[2:]),
            "hbm_bound_ms": bound_ms, "frac_of_hbm_bound": bound_ms / med, "tokens": out[:8],
            "note": "single GPU: each step is one CUDA graph (position read on the device); ~8 kernels per layer, "
                    "fixed per-kernel cost dominates at M = batch rows (DESIGN.md §5)"}
    print(json.dumps(line), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
