"""O2 — the merged-LoRA weight update (TEST INFRASTRUCTURE ONLY; see oracle/plan.py).

Definition followed:
  * P:L111-114 (§2.1): LoRA keeps W fixed and learns low-rank A, B of rank r.
  * P:L267-270 (§4.3.2): "the parameters of the LoRA adapter are merged back into
    the base model prior to inference, forming a full model".
  * North star / SURVEY.md §8(c) G1-G2:  W' = RNE_bf16( W + (alpha/r) * B @ A ),
    B is [out x r], A is [r x in] (Hu et al. convention).

Computed in fp64: every bf16*bf16 product is exact in fp64 and a sum of r <= 64
of them (each < 2^-8 in magnitude with 16 significant bits) is exact as well, so
the single final rounding gives the CORRECTLY ROUNDED merge.
"""
from __future__ import annotations

import numpy as np

from .numerics import bf16_bits_to_f64, f64_to_bf16_bits


def merge_f64(W: np.ndarray, B: np.ndarray, A: np.ndarray, scale: float) -> np.ndarray:
    """Exact W + scale * B @ A in fp64 (W, B, A given as fp64 values)."""
    return W + scale * (B @ A)


def merge_bf16_bits(W_bits: np.ndarray, B_bits: np.ndarray, A_bits: np.ndarray, scale: float) -> np.ndarray:
    """bf16 bits of RNE_bf16(W + scale * B @ A)."""
    W = bf16_bits_to_f64(W_bits)
    B = bf16_bits_to_f64(B_bits)
    A = bf16_bits_to_f64(A_bits)
    return f64_to_bf16_bits(merge_f64(W, B, A, scale))
