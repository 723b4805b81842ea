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

from .numerics import bf16_bits_to_f64, f64_to_bf16_bits, rne_f32


def merge_f64(W: np.ndarray, B: np.ndarray, A: np.ndarray, scale: float) -> np.ndarray:
    """Exact W + scale * B @ A in fp64 (W, B, A given as fp64 values)."""
    return W + scale * (B @ A)


def merge_bf16_bits(W_bits: np.ndarray, B_bits: np.ndarray, A_bits: np.ndarray, scale: float) -> np.ndarray:
    """bf16 bits of RNE_bf16(W + scale * B @ A)."""
    W = bf16_bits_to_f64(W_bits)
    B = bf16_bits_to_f64(B_bits)
    A = bf16_bits_to_f64(A_bits)
    return f64_to_bf16_bits(merge_f64(W, B, A, scale))


def merge_f32_values(W: np.ndarray, B: np.ndarray, A: np.ndarray, scale: float) -> np.ndarray:
    """fp32 debug-parity models (SURVEY.md §8(c) "Tolerances", 1e-4 gate): RNE_f32(W + scale * B @ A),
    W, B, A given as fp32 values. Each fp32*fp32 product is exact in fp64 (48 significant bits); the
    r-term sum rounds in fp64 (relative error < r * 2^-53), far below the one fp32 rounding at the end.
    Returned as a float32 array."""
    Wd, Bd, Ad = (np.asarray(x, dtype=np.float64) for x in (W, B, A))
    return rne_f32(merge_f64(Wd, Bd, Ad, scale)).astype(np.float32)
