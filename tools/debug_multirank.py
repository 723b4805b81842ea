import os, sys, time, faulthandler, threading
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("PB_DEBUG_ISSUER", "1")
sys.path.insert(0, ".")
import numpy as np, torch
import harness, synth
from paper_2503_17707_b200.api import Plan, RankEngine
from synth.configs import TINY_OPT, lora
faulthandler.dump_traceback_later(40, exit=False)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cb = int(sys.argv[2]) if len(sys.argv) > 2 else 32 << 10
pol = sys.argv[3] if len(sys.argv) > 3 else "interleave"
plan = Plan(TINY_OPT, (lora(8),), n, policy=pol, vocab_sliced=1, chunk_bytes=cb)
base, ada = harness.build_host_images(plan)
toks = synth.tokens(1, 16, TINY_OPT.vocab)
engs = [RankEngine(plan, r, base, ada, max_batch=1, max_seq=16) for r in range(n)]
for e in engs: e.wire_local(engs); e.invalidate()
print("chunks", plan.sizes.n_chunks, flush=True)
for e in engs: e.enqueue(1, toks if e.rank == 0 else None, 1, 16, 0)
print("enqueued", flush=True)
def dump():
    time.sleep(15)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for e in engs:
            w = e.workspace[:4 * 4096].view(torch.int32).cpu().numpy()
            nz = np.nonzero(w == 1)[0]
            zero = np.nonzero(w[:plan.sizes.n_chunks + 8] == 0)[0]
            print(f"rank {e.rank}: words==1: {len(nz)}; first zero words {zero[:20]}", flush=True)
threading.Thread(target=dump, daemon=True).start()
res = [e.wait(want_logits=True) for e in engs]
print("done", res[0][0], flush=True)
