"""O1 — the PipeBoost load planner, written step by step from the paper.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import anything under oracle/.

Paper passages this follows (P:L = line of PAPER.md):
  * P:L234-236 (§4.2.1 Base Model Loading): "splits the model checkpoint in DRAM
    into N parts, with each part corresponding to a GPU ... GPU 0 reads model
    A-0 while GPU 1 reads A-1"                              -> steps 1, 3
  * "the remaining portions of the model are progressively loaded"
    (here over NVLink; the north star replaces the paper's PCIe)  -> step 4
  * P:L244-245 (§4.2.2 LoRA Adapter Loading): "each adapter is partitioned, and
    the segmented parts are distributed across GPUs ... GPU 0 loads C-0, while
    GPU 1 loads B-1"                                          -> step 3 (adapters)
  * "GPU 0 which contains the first half portion of layers" -> step 1
  * P:L353-357 (Load Balance, Layer Contiguity)              -> step 1
  * P:L360-361 (§4.4.2, fig:ftpp_recovery(a)): "GPU 0 sequentially loads model
    segments 0, 1, 2 and 3, while GPU 3 loads 3, 0, 1 and 2"  -> step 4 rotation
Readings where the paper is silent are SURVEY.md §8(c) G5-G8 and DESIGN.md §3.

Plain Python lists and ints; no numpy, no cleverness.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Tuple

from synth.configs import AdapterDesc, ModelDesc

ALIGN = 4096
BF16 = 2


def elem_size(m: ModelDesc) -> int:
    """Bytes per weight / LoRA-factor element: 2 (bf16) or 4 (fp32 debug-parity path)."""
    return 4 if getattr(m, "dtype", "bf16") == "f32" else BF16

STAGE = "stage"
INTERLEAVE = "interleave"


class PartitionError(ValueError):
    pass


@dataclass(frozen=True)
class PlanOpts:
    policy: str = STAGE
    vocab_sliced: int = 0
    chunk_bytes: int = 32 << 20
    prefill_chunks: int = 1
    host_alias_layers: int = 0


@dataclass
class Tensor:
    id: int
    name: str
    rows: int
    cols: int
    layer: int          # -1 for non-layer tensors
    host_off: int = 0
    dev_off: int = 0
    es: int = BF16      # element size

    @property
    def bytes(self) -> int:
        return self.rows * self.cols * self.es


@dataclass
class ATensor:           # one LoRA factor of one adapter target
    id: int
    name: str
    rows: int
    cols: int
    layer: int
    adapter: int
    target: str
    factor: str         # 'A' ([r x in]) or 'B' ([out x r])
    base: int           # id of the base tensor it modifies
    row0: int           # first row of the base tensor it modifies
    off: int = 0        # host offset == device offset in the adapter region
    es: int = BF16

    @property
    def bytes(self) -> int:
        return self.rows * self.cols * self.es


@dataclass
class Chunk:
    id: int
    kind: str           # 'base' | 'adapter'
    tensor: int
    r0: int
    r1: int
    host_off: int
    dev_off: int
    bytes: int
    loader: int


@dataclass
class Plan:
    model: ModelDesc
    adapters: Tuple[AdapterDesc, ...]
    n_gpus: int
    opts: PlanOpts
    stages: List[Tuple[int, int]] = field(default_factory=list)
    tensors: List[Tensor] = field(default_factory=list)
    atensors: List[ATensor] = field(default_factory=list)
    chunks: List[Chunk] = field(default_factory=list)
    load: List[List[int]] = field(default_factory=list)
    recv: List[List[int]] = field(default_factory=list)
    own: List[int] = field(default_factory=list)
    host_base_bytes: int = 0
    host_adapter_bytes: int = 0
    dev_weight_bytes: int = 0
    # f1 re-plans only (replan below): original GPU id of each new rank, and the chunks each new rank
    # already holds (never re-transferred)
    survivors: Optional[List[int]] = None
    resident: Optional[List[List[int]]] = None


def round_up(x: int, a: int = ALIGN) -> int:
    return (x + a - 1) // a * a


# ---------------------------------------------------------------------------
# Step 1: partition (remainder rule S:L130)
# ---------------------------------------------------------------------------

def partition(n_layers: int, n_parts: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced stages; the first (L mod N) stages get one extra layer."""
    if n_parts < 1:
        raise ValueError("n_parts < 1")
    if n_parts > n_layers:
        raise PartitionError(f"{n_parts} parts > {n_layers} layers")
    base, rem = divmod(n_layers, n_parts)
    out, start = [], 0
    for g in range(n_parts):
        size = base + (1 if g < rem else 0)
        out.append((start, start + size))
        start += size
    return out


def balanced_slices(n: int, parts: int) -> List[Tuple[int, int]]:
    """Row slices of a vocab-sliced tensor: balanced, remainder to lower g (G5)."""
    base, rem = divmod(n, parts)
    out, start = [], 0
    for g in range(parts):
        size = base + (1 if g < rem else 0)
        out.append((start, start + size))
        start += size
    return out


# ---------------------------------------------------------------------------
# Step 2: tensor table (canonical order; offsets rounded up to 4 KiB)
# ---------------------------------------------------------------------------

def layer_tensor_shapes(m: ModelDesc):
    """(suffix, rows, cols) of one decoder layer, canonical order = the order the layer's forward
    consumes them (norm, qkv, o, norm, mlp), so a layer can start before its last bytes land.

    q,k,v are stored back to back as one [q;k;v] matrix and (Llama) gate,up as
    one [gate;up] matrix: the checkpoint layout is already the runtime layout, so
    the paper's "convert checkpoint to parameters" step is the identity.
    """
    d, f, hd = m.d_model, m.d_ffn, m.head_dim
    if m.arch == "opt":
        return [("ln1_g", 1, d), ("ln1_b", 1, d), ("qkv", 3 * d, d), ("qkv_b", 1, 3 * d), ("o", d, d),
                ("o_b", 1, d), ("ln2_g", 1, d), ("ln2_b", 1, d), ("fc1", f, d), ("fc1_b", 1, f),
                ("fc2", d, f), ("fc2_b", 1, d)]
    if m.arch == "llama":
        qkv_rows = (m.n_heads + 2 * m.n_kv_heads) * hd
        return [("ln1_g", 1, d), ("qkv", qkv_rows, d), ("o", d, m.n_heads * hd), ("ln2_g", 1, d),
                ("gate_up", 2 * f, d), ("down", d, f)]
    raise ValueError(m.arch)


def pre_tensor_shapes(m: ModelDesc):
    if m.arch == "opt":
        return [("embed", m.vocab, m.d_model), ("pos", m.max_pos + 2, m.d_model)]
    return [("embed", m.vocab, m.d_model)]


def post_tensor_shapes(m: ModelDesc):
    if m.arch == "opt":
        out = [("final_g", 1, m.d_model), ("final_b", 1, m.d_model)]
        if not m.tied:
            out.append(("lm_head", m.vocab, m.d_model))
        return out
    return [("final_g", 1, m.d_model), ("lm_head", m.vocab, m.d_model)]


def target_geometry(m: ModelDesc, target: str):
    """LoRA target -> (base suffix, first row, out_features, in_features) (G3)."""
    d, f, hd = m.d_model, m.d_ffn, m.head_dim
    if m.arch == "opt":
        table = {"q": ("qkv", 0, d, d), "k": ("qkv", d, d, d), "v": ("qkv", 2 * d, d, d),
                 "o": ("o", 0, d, d), "fc1": ("fc1", 0, f, d), "fc2": ("fc2", 0, d, f)}
    else:
        qd, kvd = m.n_heads * hd, m.n_kv_heads * hd
        table = {"q": ("qkv", 0, qd, d), "k": ("qkv", qd, kvd, d), "v": ("qkv", qd + kvd, kvd, d),
                 "o": ("o", 0, d, qd), "gate": ("gate_up", 0, f, d), "up": ("gate_up", f, f, d),
                 "down": ("down", 0, d, f)}
    return table[target]


def target_order(m: ModelDesc):
    return ("q", "k", "v", "o", "fc1", "fc2") if m.arch == "opt" else ("q", "k", "v", "o", "gate", "up", "down")


def build_tables(plan: Plan) -> None:
    m, K = plan.model, plan.opts.host_alias_layers
    L = m.n_layers
    names = [(n, r, c, -1) for (n, r, c) in pre_tensor_shapes(m)]
    for l in range(L):
        names += [(f"L{l}.{s}", r, c, l) for (s, r, c) in layer_tensor_shapes(m)]
    names += [(n, r, c, -1) for (n, r, c) in post_tensor_shapes(m)]

    dev = 0
    host = 0
    by_name = {}
    for i, (n, r, c, l) in enumerate(names):
        t = Tensor(i, n, r, c, l, es=elem_size(m))
        dev = round_up(dev)
        t.dev_off = dev
        dev += t.bytes
        if K > 0 and l >= K:
            # host_alias_layers: layer l is backed by the host image of layer l mod K
            t.host_off = by_name[f"L{l % K}." + n.split(".", 1)[1]].host_off
        else:
            host = round_up(host)
            t.host_off = host
            host += t.bytes
        by_name[n] = t
        plan.tensors.append(t)
    plan.dev_weight_bytes = round_up(dev)
    plan.host_base_bytes = round_up(host)

    off = 0
    aid = 0
    for a, ad in enumerate(plan.adapters):
        for l in range(L):
            for tgt in target_order(m):
                if tgt not in ad.targets:
                    continue
                base_sfx, row0, out_f, in_f = target_geometry(m, tgt)
                base = by_name[f"L{l}.{base_sfx}"]
                for factor, (r, c) in (("A", (ad.rank, in_f)), ("B", (out_f, ad.rank))):
                    at = ATensor(aid, f"A{a}.L{l}.{tgt}.{factor}", r, c, l, a, tgt, factor, base.id, row0,
                                 es=elem_size(m))
                    off = round_up(off)
                    at.off = off
                    off += at.bytes
                    plan.atensors.append(at)
                    aid += 1
    plan.host_adapter_bytes = round_up(off)


# ---------------------------------------------------------------------------
# Step 3: load assignment, pieces, chunks, per-GPU load lists
# ---------------------------------------------------------------------------

def layer_loader(plan: Plan, layer: int) -> int:
    if plan.opts.policy == STAGE:
        for g, (a, b) in enumerate(plan.stages):
            if a <= layer < b:
                return g
        raise AssertionError
    if plan.opts.policy == INTERLEAVE:
        return layer % plan.n_gpus
    raise ValueError(plan.opts.policy)


def pieces(plan: Plan, t: Tensor) -> List[Tuple[int, int, int]]:
    """(row0, row1, loader) pieces of a base tensor."""
    N = plan.n_gpus
    if t.layer >= 0:
        return [(0, t.rows, layer_loader(plan, t.layer))]
    if t.name in ("embed", "lm_head") and plan.opts.vocab_sliced:
        return [(a, b, g) for g, (a, b) in enumerate(balanced_slices(t.rows, N))]
    if t.name in ("embed", "pos"):
        return [(0, t.rows, 0)]
    return [(0, t.rows, N - 1)]          # final_g, final_b, lm_head (whole)


def rows_per_chunk(row_bytes: int, chunk_bytes: int) -> int:
    rpc = max(1, chunk_bytes // row_bytes)
    if rpc >= 128:
        rpc -= rpc % 128                  # keep 128-row merge tiles whole
    return rpc


def canonical_order(plan: Plan, base_chunks, ad_chunks):
    """Chunk ids in the canonical load order (G8): non-layer tensors before the first layer, then every adapter
    chunk (atensor order = host layout order), then the layers' base tensors and the remaining non-layer tensors,
    each tensor's chunks in row order. base_chunks / ad_chunks: tensor id -> chunk ids."""
    order, adapters_done = [], False
    for t in plan.tensors:
        if t.layer >= 0 and not adapters_done:
            for at in plan.atensors:
                order += [c if isinstance(c, int) else c.id for c in ad_chunks.get(at.id, [])]
            adapters_done = True
        order += [c if isinstance(c, int) else c.id for c in base_chunks.get(t.id, [])]
    return order


def build_chunks(plan: Plan) -> None:
    cb = plan.opts.chunk_bytes
    cid = 0
    per_tensor = {}
    for t in plan.tensors:
        row_bytes = t.cols * t.es
        rpc = rows_per_chunk(row_bytes, cb)
        lst = []
        for (p0, p1, g) in pieces(plan, t):
            r = p0
            while r < p1:
                r1 = min(p1, r + rpc)
                lst.append(Chunk(cid, "base", t.id, r, r1, t.host_off + r * row_bytes,
                                 t.dev_off + r * row_bytes, (r1 - r) * row_bytes, g))
                cid += 1
                r = r1
        per_tensor[t.id] = lst
        plan.chunks += lst
    per_atensor = {}
    for at in plan.atensors:
        row_bytes = at.cols * at.es
        rpc = rows_per_chunk(row_bytes, cb)
        g = layer_loader(plan, at.layer)   # part g of every adapter goes to the loader of those layers
        lst, r = [], 0
        while r < at.rows:
            r1 = min(at.rows, r + rpc)
            lst.append(Chunk(cid, "adapter", at.id, r, r1, at.off + r * row_bytes,
                             at.off + r * row_bytes, (r1 - r) * row_bytes, g))
            cid += 1
            r = r1
        per_atensor[at.id] = lst
        plan.chunks += lst

    # Per-GPU load list: the GPU's pieces in canonical table order, with ALL of
    # its adapter parts (in host layout order: adapter, layer, target, A then B)
    # right before the first layer tensor (G8: the paper is silent; the factors
    # are tiny, a GPU's parts of one adapter are contiguous in host and device
    # memory, so they cross PCIe as one DMA instead of one small DMA per layer,
    # and every adapted tensor can merge the moment its base rows land).
    N = plan.n_gpus
    plan.load = [[] for _ in range(N)]
    for cid in canonical_order(plan, per_tensor, per_atensor):
        plan.load[plan.chunks[cid].loader].append(cid)


# ---------------------------------------------------------------------------
# Step 4: receive lists (stage-needed first, then rotation (g+i) mod N)
# ---------------------------------------------------------------------------

def build_recv(plan: Plan) -> None:
    N = plan.n_gpus
    chunks = plan.chunks
    tens = plan.tensors
    plan.recv = []
    for g in range(N):
        a, b = plan.stages[g]
        need = []
        for c in chunks:
            if c.kind != "base" or c.loader == g:
                continue
            t = tens[c.tensor]
            if a <= t.layer < b:
                need.append(c.id)
        seen = set(need)
        rest = []
        for i in range(1, N):
            p = (g + i) % N
            for cid in plan.load[p]:
                c = chunks[cid]
                if c.kind == "base" and cid not in seen:
                    rest.append(cid)
                    seen.add(cid)
        plan.recv.append(need + rest)


def make_plan(model: ModelDesc, adapters, n_gpus: int, opts: PlanOpts = PlanOpts()) -> Plan:
    if n_gpus < 1:
        raise ValueError("n_gpus < 1")
    plan = Plan(model, tuple(adapters), n_gpus, opts)
    plan.stages = partition(model.n_layers, n_gpus)
    build_tables(plan)
    build_chunks(plan)
    build_recv(plan)
    # Step 5: adapter ownership own(g) = g mod A (G17); -1 without adapters.
    A = len(plan.adapters)
    plan.own = [(g % A) if A else -1 for g in range(n_gpus)]
    return plan


# ---------------------------------------------------------------------------
# f1 — recovery for model loading (§4.4.2)
# ---------------------------------------------------------------------------

def replan(plan: Plan, alive: Sequence[int], resident: Sequence[Sequence[int]]) -> Plan:
    """Re-plan the cold start over the GPUs that survived a crash during loading.

    alive[g] (0/1) for every GPU of `plan`; resident[g] = ids of the chunks GPU g already holds (landed,
    and merged where adapted). The paper's two principles and its worked example
    (GPUs 1 and 2 of 4 crash, GPU 0 keeps "0, 1, 2, 3", GPU 3 becomes "2, 3, 0, 1"):

    R1 survivors = alive GPUs in id order; m = their count (0 -> error; m > L -> PartitionError).
    R2 blocks    = partition(L, m): contiguous (Layer Contiguity), balanced (Load Balance).
    R3 blocks -> survivors: the assignment that maximises the bytes of each block's layer chunks its
       survivor already holds, over all m! assignments in lexicographic order (first maximum wins, so on a
       tie a lower GPU id keeps a lower block). New rank r = the survivor running block r
       (pipeline order = block order).
    R4 source of every chunk: the lowest new rank already holding it; else (missing everywhere) the rank
       whose block contains its layer; embed/pos -> rank 0, final norm / LM head -> rank m-1 (whole,
       vocab_sliced = 0). LoRA factor parts a rank's merges need and it does not hold are re-read from host
       by that rank (reading: a few KB per layer; the paper does not discuss adapters under recovery).
    R5 load list of rank r = chunks it sources and does not hold, canonical order (layer by layer, a
       layer's adapter parts first as in build_chunks) — its block's missing layers.
    R6 receive list of rank r = the base chunks its stage needs that it neither holds nor loads, in
       canonical order, then every other base chunk it lacks in rotation order of sources (r+i) mod m —
       "its block's missing segments first, then all remaining segments of the model".
    Already-held chunks are never loaded or received again.
    """
    N = plan.n_gpus
    if len(alive) != N or len(resident) != N:
        raise ValueError("alive / resident need one entry per GPU")
    surv = [g for g in range(N) if alive[g]]
    m = len(surv)
    if m == 0:
        raise ValueError("no surviving GPU")
    L = plan.model.n_layers
    blocks = partition(L, m)                                       # R2 (raises PartitionError)
    held = {g: set(resident[g]) for g in surv}
    tens, chunks = plan.tensors, plan.chunks

    def layer_of(c: Chunk) -> int:
        return tens[c.tensor].layer if c.kind == "base" else plan.atensors[c.tensor].layer

    def overlap(g: int, blk) -> int:
        a, b = blk
        return sum(c.bytes for c in chunks if c.kind == "base" and a <= layer_of(c) < b and c.id in held[g])

    best, best_perm = -1, None                                     # R3
    for perm in itertools.permutations(range(m)):
        tot = sum(overlap(surv[i], blocks[perm[i]]) for i in range(m))
        if tot > best:
            best, best_perm = tot, perm
    gpu_of_rank = [0] * m
    for i in range(m):
        gpu_of_rank[best_perm[i]] = surv[i]
    rank_held = [held[gpu_of_rank[r]] for r in range(m)]

    def block_rank(layer: int) -> int:
        for r, (a, b) in enumerate(blocks):
            if a <= layer < b:
                return r
        raise AssertionError(layer)

    def home_rank(c: Chunk) -> int:                                # rank that needs / would load chunk c
        l = layer_of(c)
        if l >= 0:
            return block_rank(l)
        return 0 if tens[c.tensor].name in ("embed", "pos") else m - 1

    new = Plan(plan.model, plan.adapters, m, replace(plan.opts, vocab_sliced=0))
    new.stages = blocks
    new.tensors, new.atensors = tens, plan.atensors
    new.host_base_bytes, new.host_adapter_bytes = plan.host_base_bytes, plan.host_adapter_bytes
    new.dev_weight_bytes = plan.dev_weight_bytes
    new.survivors = gpu_of_rank
    # R4: sources of base chunks
    src = {}
    for c in chunks:
        if c.kind == "base":
            holders = [r for r in range(m) if c.id in rank_held[r]]
            src[c.id] = min(holders) if holders else home_rank(c)
    # LoRA factor parts a rank needs for the merges of the base chunks it loads, and does not hold
    need_ad = [set() for _ in range(m)]
    for c in chunks:
        if c.kind == "base" and c.id not in rank_held[src[c.id]]:
            r = src[c.id]
            for at in plan.atensors:
                if at.base == c.tensor:
                    for ac in chunks:
                        if ac.kind == "adapter" and ac.tensor == at.id and ac.id not in rank_held[r]:
                            need_ad[r].add(ac.id)
    for c in chunks:
        if c.kind == "adapter":
            loaders = [r for r in range(m) if c.id in need_ad[r]]
            holders = [r for r in range(m) if c.id in rank_held[r]]
            src[c.id] = loaders[0] if loaders else (min(holders) if holders else home_rank(c))
    new.chunks = [replace(c, loader=src[c.id]) for c in chunks]
    # R5: load lists in the canonical order of build_chunks (G8: adapter parts, then the layers' base tensors)
    base_by_tensor = {}
    ad_chunks = {}
    for c in chunks:
        (base_by_tensor if c.kind == "base" else ad_chunks).setdefault(c.tensor, []).append(c.id)
    order = canonical_order(plan, base_by_tensor, ad_chunks)
    new.load = [[] for _ in range(m)]
    for cid in order:
        c = chunks[cid]
        if c.kind == "base":
            r = src[cid]
            if cid not in rank_held[r]:
                new.load[r].append(cid)
        else:
            for r in range(m):
                if cid in need_ad[r]:
                    new.load[r].append(cid)
    # R6: receive lists
    have = [set(rank_held[r]) | set(new.load[r]) for r in range(m)]
    new.recv = []
    for r in range(m):
        a, b = blocks[r]
        lst, seen = [], set()
        for cid in order:
            c = chunks[cid]
            if c.kind != "base" or cid in have[r]:
                continue
            l = tens[c.tensor].layer
            if (a <= l < b) or (l < 0 and home_rank(c) == r):
                lst.append(cid)
                seen.add(cid)
        for k in range(1, m):
            p = (r + k) % m
            for cid in order:
                c = chunks[cid]
                if c.kind == "base" and src[cid] == p and cid not in have[r] and cid not in seen:
                    lst.append(cid)
                    seen.add(cid)
        new.recv.append(lst)
    new.resident = [sorted(rank_held[r]) for r in range(m)]
    A = len(plan.adapters)
    new.own = [(r % A) if A else -1 for r in range(m)]
    return new


# ---------------------------------------------------------------------------
# Canonical text dump (compared byte for byte with pb_plan_dump)
# ---------------------------------------------------------------------------

def dump(plan: Plan) -> str:
    m, o = plan.model, plan.opts
    out = ["pipeboost-plan 1",
           f"model arch={m.arch} layers={m.n_layers} d_model={m.d_model} heads={m.n_heads} "
           f"kv_heads={m.n_kv_heads} d_ffn={m.d_ffn} vocab={m.vocab} max_pos={m.max_pos} tied={m.tied} "
           f"dtype={getattr(m, 'dtype', 'bf16')}",
           f"gpus {plan.n_gpus} policy={o.policy} vocab_sliced={o.vocab_sliced} chunk_bytes={o.chunk_bytes} "
           f"prefill_chunks={o.prefill_chunks} host_alias_layers={o.host_alias_layers}"]
    for a, ad in enumerate(plan.adapters):
        out.append(f"adapter {a} rank={ad.rank} alpha={float(ad.alpha):.6f} targets={','.join(t for t in target_order(m) if t in ad.targets)}")
    for g, (a, b) in enumerate(plan.stages):
        out.append(f"stage {g} layers=[{a},{b})")
    for t in plan.tensors:
        out.append(f"tensor {t.id} {t.name} rows={t.rows} cols={t.cols} layer={t.layer} "
                   f"host_off={t.host_off} dev_off={t.dev_off} bytes={t.bytes}")
    for at in plan.atensors:
        out.append(f"atensor {at.id} {at.name} rows={at.rows} cols={at.cols} layer={at.layer} "
                   f"base={at.base} row0={at.row0} off={at.off} bytes={at.bytes}")
    for c in plan.chunks:
        out.append(f"chunk {c.id} {c.kind} tensor={c.tensor} rows=[{c.r0},{c.r1}) host_off={c.host_off} "
                   f"dev_off={c.dev_off} bytes={c.bytes} loader={c.loader}")
    for g in range(plan.n_gpus):
        out.append(f"load {g}:" + "".join(f" {x}" for x in plan.load[g]))
    for g in range(plan.n_gpus):
        out.append(f"recv {g}:" + "".join(f" {x}" for x in plan.recv[g]))
    for g in range(plan.n_gpus):
        out.append(f"own {g} adapter={plan.own[g]}")
    if plan.survivors is not None:
        for g in range(plan.n_gpus):
            out.append(f"replan rank {g} gpu={plan.survivors[g]} resident:" + "".join(f" {x}" for x in plan.resident[g]))
    out.append(f"sizes host_base={plan.host_base_bytes} host_adapter={plan.host_adapter_bytes} "
               f"dev_weights={plan.dev_weight_bytes} dev_adapters={plan.host_adapter_bytes}")
    out.append("end")
    return "\n".join(out) + "\n"
