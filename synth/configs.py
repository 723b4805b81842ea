"""Workload shapes (BASELINE.json ``configs``; SURVEY.md §8 "Configs" / "Exact shapes").

Pure data: model hyper-parameters and adapter settings of the paper's workloads.
Both the oracle and the CUDA harness read these; neither side's arithmetic
lives here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Tuple


@dataclass(frozen=True)
class ModelDesc:
    arch: str            # 'opt' | 'llama'
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ffn: int
    vocab: int
    max_pos: int         # OPT learned positions table has max_pos + 2 rows (HF offset 2)
    tied: int            # OPT: lm_head tied to embed
    norm_eps: float = 1e-5
    rope_theta: float = 1e4
    dtype: str = "bf16"  # weights / LoRA factors: 'bf16' (the product path) or 'f32' (fp32 debug-parity gate)

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


@dataclass(frozen=True)
class AdapterDesc:
    rank: int
    alpha: float
    targets: Tuple[str, ...]   # subset of ('q','k','v','o','fc1','fc2') / ('q','k','v','o','gate','up','down')

    @property
    def scale(self) -> float:
        return self.alpha / self.rank


@dataclass(frozen=True)
class Workload:
    tag: str
    model: ModelDesc
    adapters: Tuple[AdapterDesc, ...]
    batch: int
    seq: int
    gpus: Tuple[int, ...]
    note: str = ""


OPT_ALL = ("q", "k", "v", "o", "fc1", "fc2")
LLAMA_ALL = ("q", "k", "v", "o", "gate", "up", "down")

TINY_OPT = ModelDesc("opt", 4, 256, 4, 4, 1024, 1024, 128, 1)
TINY_LLAMA = ModelDesc("llama", 4, 256, 4, 2, 688, 1000, 0, 0)      # GQA tiny shape (HF cross-check)
TINY_OPT_F32 = ModelDesc("opt", 4, 256, 4, 4, 1024, 1024, 128, 1, dtype="f32")
TINY_LLAMA_F32 = ModelDesc("llama", 4, 256, 4, 2, 688, 1000, 0, 0, dtype="f32")
OPT_1_3B = ModelDesc("opt", 24, 2048, 32, 32, 8192, 50272, 2048, 1)
LLAMA2_7B = ModelDesc("llama", 32, 4096, 32, 32, 11008, 32000, 0, 0)
OPT_13B = ModelDesc("opt", 40, 5120, 40, 40, 20480, 50272, 2048, 1)
LLAMA2_70B = ModelDesc("llama", 80, 8192, 64, 8, 28672, 32000, 0, 0)
OPT_66B = ModelDesc("opt", 64, 9216, 72, 72, 36864, 50272, 2048, 1)


def lora(rank: int, targets=("q", "v")) -> AdapterDesc:
    return AdapterDesc(rank, 2.0 * rank, tuple(targets))   # alpha = 2r  =>  s = 2 (exact)


WORKLOADS = {
    "C1": Workload("C1", TINY_OPT, (lora(8),), 1, 16, (2,), "tiny OPT, 2 shards"),
    # fp32 debug-parity run of C1 (SURVEY.md §8(c) "Tolerances": the 1e-4 gate; not timed)
    "C1f32": Workload("C1f32", TINY_OPT_F32, (lora(8),), 1, 16, (2,), "tiny OPT fp32, 2 shards"),
    "C2": Workload("C2", OPT_1_3B, (lora(16),), 1, 128, (1, 2, 4, 8), "OPT-1.3B + r16 q,v"),
    # paper-shaped secondary run of C2 (SURVEY.md §8(d) per-config inputs; "batch size of 64 ... 64 tokens")
    "C2p": Workload("C2p", OPT_1_3B, (lora(16),), 64, 64, (1, 2, 4, 8), "OPT-1.3B + r16 q,v, paper batch 64x64"),
    "C3": Workload("C3", LLAMA2_7B, tuple(lora(16) for _ in range(4)), 4, 512, (8,), "Llama-2-7B + 4 adapters"),
    "C4": Workload("C4", OPT_13B, (lora(64, OPT_ALL),), 1, 1024, (2, 4, 8), "OPT-13B + r64 all"),
    "C5a": Workload("C5a", LLAMA2_70B, (lora(16),), 1, 2048, (8,), "Llama-2-70B + r16"),
    "C5b": Workload("C5b", OPT_66B, (lora(16),), 1, 2048, (8,), "OPT-66B + r16"),
}
