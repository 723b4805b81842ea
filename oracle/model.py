"""Oracle weight provider (TEST INFRASTRUCTURE ONLY; see oracle/plan.py header).

Builds the model's weights on demand, one tensor at a time, from the seeded
generator in ``synth`` and the oracle's own tensor table (``oracle.plan``):
base values, then the LoRA merge (O2) of every adapted row range. Weights are
returned as fp64 arrays holding bf16 values. Streaming per tensor keeps a
70B-parameter model's oracle run within host RAM.

host_alias_layers = K > 0: layer l is backed by the host image
of layer (l mod K), so its base values are those of tensor "L{l mod K}.*".
Adapters are never aliased.
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

import synth

from . import plan as P
from .merge import merge_bf16_bits, merge_f32_values
from .numerics import bf16_bits_to_f64


class OracleWeights:
    def __init__(self, model, adapters, host_alias_layers: int = 0):
        self.model = model
        self.adapters = tuple(adapters)
        self.K = host_alias_layers
        pl = P.Plan(model, self.adapters, 1, P.PlanOpts(host_alias_layers=host_alias_layers))
        pl.stages = P.partition(model.n_layers, 1)
        P.build_tables(pl)
        self.tensors = {t.name: t for t in pl.tensors}
        self.atensors = pl.atensors
        # fp32 debug-parity models store fp32 values (float32 arrays) where bf16 models store bf16 bits
        self.dtype = getattr(model, "dtype", "bf16")

    def _source_name(self, name: str) -> str:
        t = self.tensors[name]
        if self.K > 0 and t.layer >= self.K:
            return f"L{t.layer % self.K}." + name.split(".", 1)[1]
        return name

    def base_bits(self, name: str) -> np.ndarray:
        t = self.tensors[name]
        return synth.base_values(self._source_name(name), t.rows, t.cols, self.dtype)

    def adapter_bits(self, at) -> np.ndarray:
        ad = self.adapters[at.adapter]
        _, _, out_f, in_f = P.target_geometry(self.model, at.target)
        return synth.adapter_values(at.adapter, at.name, at.factor, at.rows, at.cols,
                                    in_f, ad.rank, ad.scale, self.dtype)

    def merged_bits(self, name: str, adapter: int | None) -> np.ndarray:
        """bf16 bits (fp32 models: float32 values) of the base tensor with adapter `adapter` merged into
        every adapted row range (None: no merge)."""
        W = self.base_bits(name).copy()
        if adapter is None:
            return W
        t = self.tensors[name]
        ad = self.adapters[adapter]
        fac = {}
        for at in self.atensors:
            if at.adapter == adapter and at.base == t.id:
                fac.setdefault(at.target, {})[at.factor] = at
        for tgt, f in fac.items():
            A = self.adapter_bits(f["A"])
            B = self.adapter_bits(f["B"])
            r0 = f["A"].row0
            rows = B.shape[0]
            if self.dtype == "f32":
                W[r0:r0 + rows] = merge_f32_values(W[r0:r0 + rows], B, A, ad.scale)
            else:
                W[r0:r0 + rows] = merge_bf16_bits(W[r0:r0 + rows], B, A, ad.scale)
        return W

    def get(self, name: str, adapter: int | None) -> np.ndarray:
        """fp64 values of the (merged) tensor, shaped [rows, cols] (1-row tensors flattened)."""
        t = self.tensors[name]
        raw = self.merged_bits(name, adapter)
        x = raw.astype(np.float64) if self.dtype == "f32" else bf16_bits_to_f64(raw)
        return x.reshape(-1) if t.rows == 1 else x
