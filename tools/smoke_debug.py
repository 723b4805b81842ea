import os, sys, faulthandler
os.environ["PB_DEBUG_ISSUER"] = "2"
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ".")
faulthandler.dump_traceback_later(25, exit=True)
import numpy as np, torch, harness, synth
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import WORKLOADS
w = WORKLOADS["C1"]
n = int(sys.argv[1])
plan = Plan(w.model, w.adapters, n, policy="interleave", vocab_sliced=1, chunk_bytes=64 << 10, prefill_chunks=2)
base, ada = harness.build_host_images(plan)
toks = synth.tokens(1, 16, w.model.vocab)
engs = [RankEngine(plan, r, base, ada, max_batch=1, max_seq=16) for r in range(n)]
for e in engs: e.wire_local(engs); e.invalidate()
for e in engs: e.enqueue(1, toks if e.rank == 0 else None, 1, 16, adapter_id=0)
print("enqueued", flush=True)
res = [e.wait(want_logits=True) for e in engs]
print("done", res[0][0], flush=True)
