"""Seeded synthetic inputs: the one module both the CPU
oracle and the CUDA harness draw inputs from.

It holds none of the method's arithmetic — only the counter-based value
generator (``synth.c``) and the table that maps a tensor *kind* to the value
distribution the survey fixes (HF ``init_std=0.02`` shapes). Names, shapes and
offsets of tensors are NOT decided here: each side builds its own tensor table
(the oracle in ``oracle/plan.py``, the product in ``pb_plan``) and asks this
module for the values of a named tensor.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libpbsynth.so")

SEED_WEIGHTS = 0x5EED0001
SEED_ADAPTER0 = 0x5EED0100
SEED_PROMPT0 = 0x5EED1000

SQRT3 = math.sqrt(3.0)
STD_INIT = 0.02


def build(force: bool = False) -> str:
    """Compile libpbsynth.so in place (gcc, OpenMP)."""
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", src, "-o", _SO])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.pbs_fill_bf16.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                    ctypes.c_char_p, ctypes.c_double, ctypes.c_double]
        L.pbs_fill_f32.argtypes = L.pbs_fill_bf16.argtypes
        L.pbs_fill_tokens.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_char_p,
                                      ctypes.c_int64]
        L.pbs_fnv1a64.argtypes = [ctypes.c_char_p]
        L.pbs_fnv1a64.restype = ctypes.c_uint64
        L.pbs_memset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64]
        _lib = L
    return _lib


# ---------------------------------------------------------------------------
# Distribution table (SURVEY.md §8(d) "Distributions")
# ---------------------------------------------------------------------------

def dist(kind: str, *, fan_in: int = 0, rank: int = 0, scale: float = 0.0):
    """(center, half-width a) of the uniform law for a tensor kind.

    kind: 'linear' | 'bias' | 'norm_g' | 'norm_b' | 'embed' | 'lora_A' | 'lora_B'.
    lora_A ~ U(-1/sqrt(in), 1/sqrt(in)); lora_B ~ U(-b, b) with b chosen so that
    RMS(s*B@A) = 0.25 * RMS(W) = 0.005 (a skipped merge then moves the logits).
    """
    if kind in ("linear", "bias", "embed"):
        return 0.0, SQRT3 * STD_INIT
    if kind == "norm_g":
        return 1.0, 0.1
    if kind == "norm_b":
        return 0.0, 0.02
    if kind == "lora_A":
        return 0.0, 1.0 / math.sqrt(fan_in)
    if kind == "lora_B":
        # var(BA) = r * (b^2/3) * (1/(3 in)) ; s*b*sqrt(r/in)/3 = 0.25*0.02
        return 0.0, 0.25 * STD_INIT * 3.0 * math.sqrt(fan_in / rank) / scale
    raise ValueError(kind)


def fill_bf16_into(ptr: int, n: int, seed: int, name: str, center: float, a: float, start: int = 0):
    lib().pbs_fill_bf16(ctypes.c_void_p(ptr), n, start, seed, name.encode(), center, a)


def fill_into(ptr: int, n: int, seed: int, name: str, center: float, a: float, dtype: str = "bf16"):
    """Write n generator values at ptr as bf16 (RNE) or fp32 (the fp32 debug-parity models)."""
    f = lib().pbs_fill_f32 if dtype == "f32" else lib().pbs_fill_bf16
    f(ctypes.c_void_p(ptr), n, 0, seed, name.encode(), center, a)


def values_bf16(name: str, shape, seed: int, center: float, a: float) -> np.ndarray:
    """bf16 bit patterns (uint16) of a named tensor, row-major."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.uint16)
    lib().pbs_fill_bf16(out.ctypes.data, n, 0, seed, name.encode(), center, a)
    return out.reshape(shape)


def values_f32(name: str, shape, seed: int, center: float, a: float) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float32)
    lib().pbs_fill_f32(out.ctypes.data, n, 0, seed, name.encode(), center, a)
    return out.reshape(shape)


def tokens(batch: int, seq: int, vocab: int) -> np.ndarray:
    """Prompt token ids [batch, seq]; prompt b uses seed 0x5EED1000+b."""
    out = np.empty((batch, seq), dtype=np.int32)
    for b in range(batch):
        row = np.empty(seq, dtype=np.int32)
        lib().pbs_fill_tokens(row.ctypes.data, seq, SEED_PROMPT0 + b, b"prompt", vocab)
        out[b] = row
    return out


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def kind_of(name: str) -> str:
    """Distribution kind of a base tensor from its table name (data spec only)."""
    sfx = name.split(".", 1)[1] if name.startswith("L") and "." in name else name
    if sfx in ("embed", "pos", "lm_head"):
        return "embed"
    if sfx in ("qkv", "o", "fc1", "fc2", "gate_up", "down"):
        return "linear"
    if sfx in ("qkv_b", "o_b", "fc1_b", "fc2_b"):
        return "bias"
    if sfx in ("ln1_g", "ln2_g", "final_g"):
        return "norm_g"
    if sfx in ("ln1_b", "ln2_b", "final_b"):
        return "norm_b"
    raise ValueError(name)


def base_values(name: str, rows: int, cols: int, dtype: str = "bf16") -> np.ndarray:
    """bf16 bits (uint16) — or fp32 values for dtype 'f32' — of a base tensor (seed 0x5EED0001)."""
    c, a = dist(kind_of(name))
    fn = values_f32 if dtype == "f32" else values_bf16
    return fn(name, (rows, cols), SEED_WEIGHTS, c, a)


def adapter_values(adapter: int, name: str, factor: str, rows: int, cols: int,
                   fan_in: int, rank: int, scale: float, dtype: str = "bf16") -> np.ndarray:
    """bf16 bits (uint16) — or fp32 values for dtype 'f32' — of a LoRA factor (seed 0x5EED0100 + adapter)."""
    c, a = dist("lora_A" if factor == "A" else "lora_B", fan_in=fan_in, rank=rank, scale=scale)
    fn = values_f32 if dtype == "f32" else values_bf16
    return fn(name, (rows, cols), SEED_ADAPTER0 + adapter, c, a)
