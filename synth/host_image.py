"""Fill pinned host images in a given layout with seeded synthetic values.

The layout (names, shapes, host offsets) is supplied by the caller — it comes from the plan
being tested — so this module decides no placement and does no method arithmetic; it only
writes generator values at the offsets it is given.
"""
from __future__ import annotations

import synth


def fill_base(host_ptr: int, tensors, dtype: str = "bf16"):
    """tensors: iterable of (name, rows, cols, host_off, layer). Tensors sharing a host offset
    (host_alias_layers) are written once, by the first (lowest-layer) owner. dtype: 'bf16' | 'f32'."""
    seen = set()
    for name, rows, cols, off, layer in tensors:
        if off in seen:
            continue
        seen.add(off)
        c, a = synth.dist(synth.kind_of(name))
        synth.fill_into(host_ptr + off, rows * cols, synth.SEED_WEIGHTS, name, c, a, dtype)


def fill_adapters(host_ptr: int, atensors, adapters, dtype: str = "bf16"):
    """atensors: iterable of (name, rows, cols, off, adapter, is_B, fan_in)."""
    for name, rows, cols, off, a, is_B, fan_in in atensors:
        ad = adapters[a]
        c, w = synth.dist("lora_B" if is_B else "lora_A", fan_in=fan_in, rank=ad.rank, scale=ad.scale)
        synth.fill_into(host_ptr + off, rows * cols, synth.SEED_ADAPTER0 + a, name, c, w, dtype)
