"""Test/bench harness: build the pinned host images for a plan from the seeded generator.

Not part of the product path: it plays the role of the checkpoint already residing in DRAM
("uses a model checkpoint already residing in DRAM"). Layout comes from the plan under
test (pb_plan accessors); values come from synth.
"""
from __future__ import annotations

import torch

from paper_2503_17707_b200.api import Plan, pinned_host
from synth import host_image


def build_host_images(plan: Plan):
    s = plan.sizes
    base = pinned_host(s.host_base_bytes)
    tens = plan.tensors()
    host_image.fill_base(base.data_ptr(), [(n, r, c, off, l) for (n, r, c, off, l, _) in tens])
    ada = None
    if s.host_adapter_bytes:
        ada = pinned_host(s.host_adapter_bytes)
        items = []
        for (n, r, c, off, a, is_b, base_t, _) in plan.atensors():
            items.append((n, r, c, off, a, is_b, tens[base_t][2]))
        host_image.fill_adapters(ada.data_ptr(), items, plan.adapters)
    return base, ada
