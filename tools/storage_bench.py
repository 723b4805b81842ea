"""f4 measurement — cold start with the checkpoint read from a FILE (pb_ctx_set_file_source) vs from the pinned
DRAM image the paper assumes, one B200.

    python tools/storage_bench.py [--workload C2] [--steps 3] [--dir /tmp]

The file is the host image in the canonical layout, written once (untimed). TTFT on the device clock
(t0 -> first token in host memory), mean of `steps` trials after one warm-up; the page cache is NOT dropped (no
root guarantee on the box), so with O_DIRECT the reads go to the device, without it they may hit the cache —
both are reported with the file system the directory is on. One JSON line.
"""
import argparse
import json
import os
import statistics
import subprocess
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
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--staging-mb", type=int, default=512)
    a = ap.parse_args()
    w = WORKLOADS[a.workload]
    plan = Plan(w.model, w.adapters, 1, chunk_bytes=64 << 20)
    base, ada = harness.build_host_images(plan)
    toks = synth.tokens(w.batch, w.seq, w.model.vocab)
    path = os.path.join(a.dir, f"pipeboost_ckpt_{a.workload}.bin")
    base.numpy().tofile(path)
    fs = subprocess.run(["df", "-T", a.dir], capture_output=True, text=True).stdout.splitlines()[-1].split()[1]
    eng = RankEngine(plan, 0, base, ada, max_batch=w.batch, max_seq=w.seq)
    eng.wire_local([eng])
    res = {}
    ep = 1
    for mode in ("pinned", "file", "pinned"):
        if mode == "file":
            eng.set_file_source(path, a.staging_mb << 20)
        else:
            eng.set_file_source(None)
        vals, toks_out = [], None
        for i in range(a.steps + 1):
            eng.invalidate()
            t, _ = eng.cold_start(ep, toks, adapter_id=0)
            ep += 1
            if i:
                vals.append(eng.timeline()["ttft_ms"])
            toks_out = [int(x) for x in t]
        res.setdefault(mode, []).append((statistics.mean(vals), toks_out))
    os.unlink(path)
    S = plan.sizes.host_base_bytes
    line = {"metric": "f4 cold-start TTFT from a checkpoint file vs pinned DRAM", "workload": a.workload,
            "bytes": S, "dir": a.dir, "fs": fs, "staging_mb": a.staging_mb,
            "ttft_ms_pinned": res["pinned"][0][0], "ttft_ms_file": res["file"][0][0],
            "ttft_ms_pinned_again": res["pinned"][1][0],
            "file_gbs_effective": S / (res["file"][0][0] * 1e-3) / 1e9,
            "first_tokens_equal": res["file"][0][1] == res["pinned"][0][1]}
    print(json.dumps(line), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
