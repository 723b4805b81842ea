"""Multi-process cold start (one process per rank, CUDA-IPC wiring exchanged with torch.distributed).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/mp_coldstart.py [--same-gpu] [--backend gloo]

With --same-gpu every rank uses cuda:0 (the GPU test box has one B200); rank 0 checks the first token and
logits against the CPU oracle and prints one JSON line.
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import harness
import synth
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--same-gpu", action="store_true")
ap.add_argument("--backend", default="gloo")
ap.add_argument("--workload", default="C1")
ap.add_argument("--policy", default="interleave")
ap.add_argument("--sliced", type=int, default=1)
ap.add_argument("--k", type=int, default=2)
args = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = 0 if args.same_gpu else int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(dev)
dist.init_process_group(args.backend)
w = WORKLOADS[args.workload]
plan = Plan(w.model, w.adapters, world, policy=args.policy, vocab_sliced=args.sliced, chunk_bytes=64 << 10,
            prefill_chunks=args.k)
dumps = [None] * world
dist.all_gather_object(dumps, plan.dump())
assert all(d == dumps[0] for d in dumps), "ranks disagree on the plan"
base, ada = harness.build_host_images(plan)
toks = synth.tokens(w.batch, w.seq, w.model.vocab)
eng = RankEngine(plan, rank, base, ada, max_batch=w.batch, max_seq=w.seq)
blobs = [None] * world
dist.all_gather_object(blobs, eng.export())
eng.wire_ipc(blobs)
results = []
for ep in (1, 2):
    eng.invalidate()
    dist.barrier()
    out = eng.cold_start(ep, toks if rank == 0 else None, w.batch, w.seq, adapter_id=0, want_logits=True)
    dist.barrier()
    results.append(out)
if rank == 0:
    import oracle
    ol, ot = oracle.first_token_logits(w.model, w.adapters, toks, mode="bf16")
    tokens, logits = results[-1]
    rel = float(np.abs(logits[0] - ol[0]).max() / np.abs(ol[0]).max())
    same = bool(np.array_equal(results[0][1].view(np.uint32), results[1][1].view(np.uint32)))
    print(json.dumps({"world": world, "tokens": tokens.tolist(), "oracle": ot.tolist(), "rel": rel,
                      "trials_identical": same, "ttft_ms": eng.timeline()["ttft_ms"]}), flush=True)
dist.barrier()
eng.close()
dist.destroy_process_group()
