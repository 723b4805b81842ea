#!/usr/bin/env python
"""Full-depth oracle first-token logits for the target workloads (TEST INFRASTRUCTURE; imports only oracle/ and
synth/ — never the product path).

    python tools/oracle_reference.py C4 [--host-alias K] [--modes bf16,exact] [--batch B --seq T]

Streams the model one tensor at a time (oracle.OracleWeights regenerates each tensor from the seeded generator
and merges its LoRA factors in fp64), runs the plain sequential forward (oracle/forward.py)
over the workload's prompt(s) and writes tests/golden/oracle_<tag>[_K<k>].npz:

  tokens            [B, T] int32   prompt (synth.tokens)
  adapter_of_seq    [B] int32      adapter used per sequence (-1 = none)
  logits_<mode>     [B, V] float32 last-position logits (bf16 mode: already fp32 values, stored exactly;
                                   exact mode: fp64 rounded to fp32, 6e-8 relative — far below the 1e-2 gate)
  argmax_<mode>     [B] int32      first token (lowest index on ties, O4)
  margin_<mode>     [B] float64    top-1 minus top-2 logit
  maxabs_<mode>     [B] float64    max |logit| (the denominator of the relative error)
  meta              json string    workload, host_alias_layers, modes, seconds per mode, cores

Every stored value comes from oracle/ (pipelining moves where layers run, not what they compute,
so the oracle's sequential forward is the reference for any N, policy or prompt chunking).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from synth.configs import WORKLOADS  # noqa: E402


def golden_path(tag: str, alias: int) -> str:
    return os.path.join(ROOT, "tests", "golden", f"oracle_{tag}" + (f"_K{alias}" if alias else "") + ".npz")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--host-alias", type=int, default=0)
    ap.add_argument("--modes", default="bf16,exact")
    ap.add_argument("--out", default=None)
    ap.add_argument("--append", action="store_true",
                    help="keep the modes already stored in the output file (e.g. run bf16 and exact as separate jobs)")
    ap.add_argument("--keep-logits", type=int, default=0,
                    help="store the full logit rows of the first N sequences only (argmax / margin / maxabs stay for "
                         "every sequence); with no modes to run, trims an existing file in place (C2p: 64 x 50272)")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.keep_logits and args.modes == "":
        path = args.out or golden_path(w.tag, args.host_alias)
        d = dict(np.load(path))
        meta = json.loads(str(d.pop("meta")))
        for k in list(d):
            if k.startswith("logits_"):
                d[k] = d[k][:args.keep_logits]
        meta["logits_rows_kept"] = args.keep_logits
        d["meta"] = np.array(json.dumps(meta))
        np.savez_compressed(path, **d)
        print("trimmed", path)
        return
    m = w.model
    toks = synth.tokens(w.batch, w.seq, m.vocab)
    n_ad = len(w.adapters)
    aos = [b % n_ad for b in range(w.batch)] if n_ad > 1 else [0 if n_ad else None] * w.batch
    out = {"tokens": toks, "adapter_of_seq": np.array([-1 if a is None else a for a in aos], dtype=np.int32)}
    meta = {"workload": w.tag, "note": w.note, "host_alias_layers": args.host_alias, "batch": w.batch,
            "seq": w.seq, "modes": [], "seconds": {}, "cores": os.cpu_count(),
            "source": "tools/oracle_reference.py (oracle.first_token_logits; imports oracle/ and synth/ only)"}
    path = args.out or golden_path(w.tag, args.host_alias)
    if args.append and os.path.exists(path):
        old = dict(np.load(path))
        assert np.array_equal(old["tokens"], toks), "stored prompt differs"
        prev = json.loads(str(old.pop("meta")))
        out.update({k: v for k, v in old.items() if k not in out})
        meta["modes"] = list(prev.get("modes", []))
        meta["seconds"] = dict(prev.get("seconds", {}))
    for mode in args.modes.split(","):
        t0 = time.time()
        lg, tk = oracle.first_token_logits(m, w.adapters, toks, adapter_of_seq=aos, mode=mode,
                                           host_alias_layers=args.host_alias)
        dt = time.time() - t0
        srt = np.sort(lg, axis=1)
        out[f"logits_{mode}"] = lg.astype(np.float32)[:args.keep_logits or None]
        out[f"argmax_{mode}"] = tk.astype(np.int32)
        out[f"margin_{mode}"] = (srt[:, -1] - srt[:, -2]).astype(np.float64)
        out[f"maxabs_{mode}"] = np.abs(lg).max(axis=1).astype(np.float64)
        meta["modes"].append(mode)
        meta["seconds"][mode] = dt
        print(json.dumps({"workload": w.tag, "mode": mode, "s": round(dt, 1), "argmax": tk.tolist()[:8],
                          "margin": out[f"margin_{mode}"].tolist()[:8]}), flush=True)
        out["meta"] = np.array(json.dumps(meta))
        np.savez_compressed(path, **out)       # after every mode: a long run keeps what it finished
    if "logits_bf16" in out and "logits_exact" in out:
        e = np.abs(out["logits_bf16"].astype(np.float64) - out["logits_exact"]).max(axis=1)
        print(json.dumps({"workload": w.tag, "bf16_vs_exact_rel": (e / out["maxabs_exact"]).tolist()[:8]}))
    print("wrote", path)


if __name__ == "__main__":
    main()
