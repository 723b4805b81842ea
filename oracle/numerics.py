"""Rounding helpers for the oracle (TEST INFRASTRUCTURE ONLY; see oracle/plan.py header).

Each helper is the textbook definition of the rounding it names, written with
numpy fp64 primitives:
  * rne_bf16(x): round-to-nearest-even of an fp64 value to the bfloat16 grid
    (8 significant bits, fp32 exponent range) — ONE rounding, straight from fp64.
  * rne_f32(x):  IEEE fp64 -> fp32 conversion (numpy's astype is RNE).
"""
from __future__ import annotations

import numpy as np


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def rne_bf16(x: np.ndarray) -> np.ndarray:
    """Correctly rounded (ties-to-even) bf16 value of fp64 x, returned as fp64."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                       # x = m * 2^e, 0.5 <= |m| < 1
    e = np.maximum(e, -125)                  # below 2^-126 the bf16 quantum stays 2^-133
    ulp = np.ldexp(1.0, e - 8)               # 8 significant bits
    r = np.rint(x / ulp) * ulp               # np.rint: half to even; x/ulp exact (power of 2)
    return np.where(np.isfinite(x), r, x)


def f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit pattern of rne_bf16(x) (x must already be on the bf16 grid or is rounded here)."""
    r = rne_bf16(x).astype(np.float32)       # exact: r is on the bf16 grid
    return (r.view(np.uint32) >> 16).astype(np.uint16)


def rne_f32(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def bf16_ulp(x: np.ndarray) -> np.ndarray:
    """Spacing of the bf16 grid at |x| (the unit a 1-ulp tolerance is measured in)."""
    x = np.abs(np.asarray(x, dtype=np.float64))
    _, e = np.frexp(np.where(x == 0, 1e-300, x))
    return np.ldexp(1.0, np.maximum(e, -125) - 8)
