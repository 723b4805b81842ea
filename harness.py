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
    """Pinned host images (one process)."""
    s = plan.sizes
    base = pinned_host(s.host_base_bytes)
    ada = pinned_host(s.host_adapter_bytes) if s.host_adapter_bytes else None
    fill_host_images(plan, base.data_ptr(), ada.data_ptr() if ada is not None else None)
    return base, ada
