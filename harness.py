"""Test/bench harness: build the pinned host images for a plan from the seeded generator.

Not part of the product path: it plays the role of the checkpoint already residing in DRAM
("uses a model checkpoint already residing in DRAM"). Layout comes from the plan under
test (pb_plan accessors); values come from synth.
"""
from __future__ import annotations

import torch

from paper_2503_17707_b200.api import Plan, pinned_host
from synth import host_image


def fill_host_images(plan: Plan, base_ptr: int, ada_ptr: int | None):
    """Write the seeded model (and adapters) into host buffers laid out as `plan` says."""
    tens = plan.tensors()
    dt = getattr(plan.model, "dtype", "bf16")
    host_image.fill_base(base_ptr, [(n, r, c, off, l) for (n, r, c, off, l, _) in tens], dt)
    if plan.sizes.host_adapter_bytes and ada_ptr:
        items = [(n, r, c, off, a, is_b, tens[base_t][2]) for (n, r, c, off, a, is_b, base_t, _) in plan.atensors()]
        host_image.fill_adapters(ada_ptr, items, plan.adapters, dt)


def build_host_images(plan: Plan):
    """Pinned host images (one process): the base image and, 4 KiB-aligned right after it in the SAME pinned
    allocation, the adapter image (one registered host range for the copy engine: a DMA from a second pinned
    allocation measured tens of microseconds of extra latency on the copy lane)."""
    s = plan.sizes
    off = (s.host_base_bytes + 4095) // 4096 * 4096
    buf = pinned_host(off + s.host_adapter_bytes)
    base = buf[:s.host_base_bytes]
    ada = buf[off:off + s.host_adapter_bytes] if s.host_adapter_bytes else None
    fill_host_images(plan, base.data_ptr(), ada.data_ptr() if ada is not None else None)
    return base, ada


# ----------------------------------------------------------------------------------------------------
# Full-depth parity against stored oracle logits (tests/golden/oracle_<tag>[_K<k>].npz, written by
# tools/oracle_reference.py, which calls only oracle/).
# ----------------------------------------------------------------------------------------------------

def golden_path(tag: str, host_alias: int = 0) -> str:
    import os
    root = os.path.dirname(os.path.abspath(__file__))
    return os.path.join(root, "tests", "golden", f"oracle_{tag}" + (f"_K{host_alias}" if host_alias else "") + ".npz")


def load_golden(tag: str, host_alias: int = 0):
    import os
    import numpy as np
    p = golden_path(tag, host_alias)
    return dict(np.load(p)) if os.path.exists(p) else None


def golden_parity(gold, logits, tokens, gate: float = 1e-2) -> dict:
    """Compare GPU first-token logits [B, V] / tokens [B] with the stored oracle.

    rel = ||g - o||_inf / ||o||_inf per sequence against the bf16-contract oracle and, when stored, rel_exact
    against the exact fp64 oracle. The gate (DESIGN.md §3 "tolerance gates", reading R1): rel <= max(1e-2, c)
    where c = ||o_bf16 - o_exact||_inf / ||o_exact||_inf is the oracle's OWN bf16-vs-exact spread on that
    sequence — a bf16 forward cannot be held closer to the contract than the contract is to the exact forward
    (random-init Llama stacks amplify rounding noise ~sqrt(L): c = 4.6 % at C3); and rel_exact <= max(1e-2,
    1.25 c): the GPU is as accurate as the oracle's bf16 mode. Where c < 1e-2 (every OPT workload) the gate is the
    north star's 1e-2. Token rule G10: if the oracle's top-1 minus top-2 margin exceeds
    2*max|g - o| the GPU token must equal the oracle's argmax, otherwise the GPU token's oracle logit must lie
    within 2*max|g - o| of the oracle maximum."""
    import numpy as np
    out = {"rel": [], "token_ok": [], "token_exact_match": [], "margin": [], "gate": gate, "gate_used": [],
           "contract_vs_exact": []}
    ol = gold["logits_bf16"].astype(np.float64)
    if "logits_exact" in gold:
        out["rel_exact"] = []
    ok = True
    for b in range(ol.shape[0]):
        g = np.asarray(logits[b], dtype=np.float64)
        err = float(np.abs(g - ol[b]).max())
        rel = err / float(np.abs(ol[b]).max())
        out["rel"].append(rel)
        gb = gate
        if "logits_exact" in gold:
            oe = gold["logits_exact"][b].astype(np.float64)
            c = float(np.abs(ol[b] - oe).max() / np.abs(oe).max())
            re = float(np.abs(g - oe).max() / np.abs(oe).max())
            out["rel_exact"].append(re)
            out["contract_vs_exact"].append(c)
            gb = max(gate, c)
            ok = ok and re <= max(gate, 1.25 * c)
        out["gate_used"].append(gb)
        ok = ok and rel <= gb
        srt = np.sort(ol[b])
        margin = float(srt[-1] - srt[-2])
        ot = int(np.argmax(ol[b]))
        tk = int(tokens[b])
        tok_ok = tk == ot if margin > 2 * err else bool(ol[b][tk] >= srt[-1] - 2 * err)
        out["token_ok"].append(bool(tok_ok))
        out["token_exact_match"].append(tk == ot)
        out["margin"].append(margin)
    # sequences whose full logit rows are not stored (C2p keeps 16 of 64): the G10 token rule with the largest
    # absolute error seen on the stored rows, against the stored oracle argmax / margin
    if "argmax_bf16" in gold and gold["argmax_bf16"].shape[0] > ol.shape[0]:
        err_all = max(float(np.abs(np.asarray(logits[b], dtype=np.float64) - ol[b]).max()) for b in range(ol.shape[0]))
        for b in range(ol.shape[0], gold["argmax_bf16"].shape[0]):
            ot, margin, tk = int(gold["argmax_bf16"][b]), float(gold["margin_bf16"][b]), int(tokens[b])
            tok_ok = tk == ot if margin > 2 * err_all else True   # near tie: any token within the bound is accepted
            out["token_ok"].append(bool(tok_ok))
            out["token_exact_match"].append(tk == ot)
            out["margin"].append(margin)
    out["max_rel"] = max(out["rel"])
    if "rel_exact" in out:
        out["max_rel_exact"] = max(out["rel_exact"])
    out["ok"] = ok and all(out["token_ok"])
    return out
