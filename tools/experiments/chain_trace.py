"""Where does a layer-chain launch spend its time? (debug probe, one B200)

    python tools/chain_trace.py [--workload C2]          (sets PB_CHAIN=1 PB_CHAIN_TRACE=1)

Cold start + two warm replays of the bench workload with the per-item trace of chain.cu enabled, then, for one
launch of the last replay: per job, when its first item was claimed, when its activations were ready, when its
last unit was published; per-item mainloop (dependency met -> accumulator ready) and epilogue times.
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ["PB_CHAIN_TRACE"] = "1"
os.environ["PB_CHAIN"] = "1"
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import harness  # noqa: E402
import synth  # noqa: E402
from paper_2503_17707_b200 import _binding as B  # noqa: E402
from paper_2503_17707_b200.api import Plan, RankEngine  # noqa: E402
from synth.configs import WORKLOADS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--layer", type=int, default=10)
    a = ap.parse_args()
    w = WORKLOADS[a.workload]
    plan = Plan(w.model, w.adapters, 1, chunk_bytes=64 << 20)
    base, ada = harness.build_host_images(plan)
    toks = synth.tokens(1, w.seq, w.model.vocab)
    eng = RankEngine(plan, 0, base, ada, max_batch=1, max_seq=w.seq)
    eng.wire_local([eng])
    eng.invalidate()
    eng.cold_start(1, toks, adapter_id=0)
    for ep in (2, 3, 4):
        eng.replay_enqueue(ep, toks, 1, w.seq)
        eng.wait()
    L = w.model.n_layers
    tr, tr2 = B.pb_op_chain_trace(2 * L)
    slot = L + a.layer   # the replay graph's launches (captured after the cold start's L)
    t = tr[slot].astype(np.int64)
    used = t[:, 0] > 0
    meta = tr[slot][:, 5]
    job = ((meta >> np.uint64(40)) & np.uint64(0xFF)).astype(int)
    sm = (meta >> np.uint64(48)).astype(int)
    t0 = t[used, 0].min()
    out = {"workload": a.workload, "layer": a.layer, "items": int(used.sum()), "sms": int(len(set(sm[used])))}
    pub = t[:, 3] & ((1 << 62) - 1)
    fin = (tr[slot][:, 3] >> np.uint64(63)).astype(bool)
    for j in range(4):
        m = used & (job == j)
        if not m.any():
            continue
        rec = {"items": int(m.sum()),
               "first_claim_us": (t[m, 0].min() - t0) / 1e3,
               "last_claim_us": (t[m, 0].max() - t0) / 1e3,
               "dep_met_first_us": (t[m, 1][t[m, 1] > 0].min() - t0) / 1e3 if (t[m, 1] > 0).any() else None,
               "dep_met_last_us": (t[m, 1][t[m, 1] > 0].max() - t0) / 1e3 if (t[m, 1] > 0).any() else None}
        if j in (0, 2, 3):
            acc = t[m, 2]
            rec["mainloop_us_median"] = float(np.median(acc - t[m, 1])) / 1e3
            rec["epilogue_us_median"] = float(np.median(pub[m] - acc)) / 1e3
            rec["epilogue_us_median_finishing"] = float(np.median((pub[m] - acc)[fin[m]])) / 1e3
            mf = m & fin
            if (t[mf, 4] > 0).any():
                rec["fin_arrive_us"] = float(np.median(t[mf, 4] - t[mf, 2])) / 1e3
                rec["fin_first_stage_us"] = float(np.median(t[mf, 6] - t[mf, 4])) / 1e3
                rec["fin_reduce_us"] = float(np.median(t[mf, 7] - t[mf, 6])) / 1e3
                rec["fin_publish_us"] = float(np.median(pub[mf] - t[mf, 7])) / 1e3
                c2 = tr2[slot].astype(np.int64)[mf]
                rec["fin_chunks_us"] = [float(np.median(c2[:, i] - t[mf, 4])) / 1e3 for i in range(8)]
            mn = m & ~fin
            if mn.any() and (t[mn, 4] > 0).any():
                rec["nonfin_arrive_us"] = float(np.median(t[mn, 4] - t[mn, 2])) / 1e3
        rec["last_publish_us"] = (pub[m].max() - t0) / 1e3
        out[f"job{j}"] = rec
    out["total_us"] = (pub[used].max() - t0) / 1e3
    print(json.dumps(out, indent=1))
    np.save(os.path.join(HERE, "gpurun_out", "chain_trace.npy"), tr)
    eng.close()


if __name__ == "__main__":
    main()
