"""Pins for the oracle planner (O1) against what the paper fixes.

Every test names the passage it checks. None of them re-types the planner's
formulas: they check the paper's worked examples, exhaustive enumeration, and
structural invariants.
"""
import itertools
import random

import pytest

from oracle import plan as P
from synth.configs import AdapterDesc, ModelDesc, TINY_OPT, TINY_LLAMA, OPT_1_3B, LLAMA2_70B, lora, OPT_ALL


def tiny(L=4, arch="opt"):
    if arch == "opt":
        return ModelDesc("opt", L, 64, 2, 2, 128, 96, 16, 1)
    return ModelDesc("llama", L, 64, 4, 2, 96, 80, 0, 0)


def segment_of(plan, chunk):
    """Map a chunk to the pipeline segment (stage) it belongs to: layer tensors by
    their layer; leading non-layer tensors to segment 0, trailing to N-1."""
    c = plan.chunks[chunk]
    if c.kind == "adapter":
        t = plan.atensors[c.tensor]
        layer = t.layer
    else:
        layer = plan.tensors[c.tensor].layer
    if layer < 0:
        name = plan.tensors[c.tensor].name
        return 0 if name in ("embed", "pos") else plan.n_gpus - 1
    for g, (a, b) in enumerate(plan.stages):
        if a <= layer < b:
            return g
    raise AssertionError


def acquisition_segments(plan, g):
    """Order in which GPU g acquires segments: own load list (PCIe), then recv (NVLink)."""
    seq = []
    for cid in plan.load[g] + plan.recv[g]:
        if plan.chunks[cid].kind != "base":
            continue
        s = segment_of(plan, cid)
        if not seq or seq[-1] != s:
            seq.append(s)
    return seq


# --- Step 1: partition -----------------------------------------------------

def test_partition_spec_example():
    # S:L135 [DERIVED]: (30 layers, 4) -> [8, 8, 7, 7]
    st = P.partition(30, 4)
    assert [b - a for a, b in st] == [8, 8, 7, 7]


def test_partition_paper_first_half():
    # "GPU 0 which contains the first half portion of layers" (N=2)
    assert P.partition(24, 2) == [(0, 12), (12, 24)]


def test_partition_error():
    with pytest.raises(P.PartitionError):
        P.partition(3, 4)


@pytest.mark.parametrize("L", range(1, 13))
def test_partition_bruteforce(L):
    # P:L353-357 Load Balance + Layer Contiguity. Enumerate every contiguous split
    # into N non-empty parts: ours minimises the largest part, differs by <=1, and
    # is the unique balanced split with the larger parts first (remainder rule).
    for N in range(1, min(L, 6) + 1):
        ours = [b - a for a, b in P.partition(L, N)]
        best = None
        balanced = []
        for cuts in itertools.combinations(range(1, L), N - 1):
            bounds = (0,) + cuts + (L,)
            sizes = [bounds[i + 1] - bounds[i] for i in range(N)]
            mx = max(sizes)
            best = mx if best is None else min(best, mx)
            if mx - min(sizes) <= 1:
                balanced.append(sizes)
        assert max(ours) == best
        assert max(ours) - min(ours) <= 1
        nonincreasing = [s for s in balanced if all(s[i] >= s[i + 1] for i in range(N - 1))]
        assert nonincreasing == [ours]


# --- Steps 3/4: paper worked examples ---------------------------------------

def test_rotation_fig_ftpp_recovery_a():
    # "GPU 0 sequentially loads model segments 0, 1, 2 and 3, while
    # GPU 3 loads 3, 0, 1 and 2. GPUs 1 and 2 follow a similar pattern."
    plan = P.make_plan(tiny(4), (), 4, P.PlanOpts(policy=P.STAGE, chunk_bytes=4096))
    assert acquisition_segments(plan, 0) == [0, 1, 2, 3]
    assert acquisition_segments(plan, 1) == [1, 2, 3, 0]
    assert acquisition_segments(plan, 2) == [2, 3, 0, 1]
    assert acquisition_segments(plan, 3) == [3, 0, 1, 2]


def test_base_split_two_gpus():
    # "GPU 0 reads model A-0 while GPU 1 reads A-1" — disjoint halves.
    plan = P.make_plan(tiny(4), (), 2, P.PlanOpts())
    segs0 = {segment_of(plan, c) for c in plan.load[0]}
    segs1 = {segment_of(plan, c) for c in plan.load[1]}
    assert segs0 == {0} and segs1 == {1}
    # "model A-1 is loaded onto GPU 0, and model A-0 is loaded onto GPU 1"
    assert {segment_of(plan, c) for c in plan.recv[0]} == {1}
    assert {segment_of(plan, c) for c in plan.recv[1]} == {0}


def test_adapter_parts_two_gpus():
    # GPU 0 serves adapter B (id 0), GPU 1 adapter C (id 1);
    # "GPU 0 loads C-0, while GPU 1 loads B-1" (and each its own part).
    B, C = lora(4), lora(4)
    plan = P.make_plan(tiny(4), (B, C), 2, P.PlanOpts())
    def parts(g):
        out = set()
        for cid in plan.load[g]:
            c = plan.chunks[cid]
            if c.kind == "adapter":
                at = plan.atensors[c.tensor]
                out.add((at.adapter, segment_of(plan, cid)))
        return out
    assert parts(0) == {(0, 0), (1, 0)}      # B-0, C-0
    assert parts(1) == {(0, 1), (1, 1)}      # B-1, C-1
    assert plan.own == [0, 1]


# --- invariants -------------------------------------------------------------

def check_invariants(plan):
    N = plan.n_gpus
    ids = [c.id for c in plan.chunks]
    assert ids == list(range(len(ids)))
    # exactly once: the multiset union of load lists is every chunk (north star)
    allload = sorted(x for g in range(N) for x in plan.load[g])
    assert allload == ids
    for g in range(N):
        for cid in plan.load[g]:
            assert plan.chunks[cid].loader == g
    base = {c.id for c in plan.chunks if c.kind == "base"}
    for g in range(N):
        own = {c for c in plan.load[g] if plan.chunks[c].kind == "base"}
        rc = plan.recv[g]
        assert len(rc) == len(set(rc))
        assert own.isdisjoint(rc)
        assert own | set(rc) == base            # union of shards is the whole model
    # chunks tile each tensor's rows exactly once; offsets consistent & in bounds
    rows = {}
    for c in plan.chunks:
        rows.setdefault((c.kind, c.tensor), []).append((c.r0, c.r1))
        if c.kind == "base":
            t = plan.tensors[c.tensor]
            rb = t.cols * 2
            assert c.dev_off == t.dev_off + c.r0 * rb and c.host_off == t.host_off + c.r0 * rb
            assert c.dev_off + c.bytes <= plan.dev_weight_bytes
            assert c.host_off + c.bytes <= plan.host_base_bytes
        else:
            t = plan.atensors[c.tensor]
            assert c.dev_off + c.bytes <= plan.host_adapter_bytes
        assert c.bytes == (c.r1 - c.r0) * t.cols * 2
    for (kind, tid), rs in rows.items():
        t = plan.tensors[tid] if kind == "base" else plan.atensors[tid]
        rs.sort()
        assert rs[0][0] == 0 and rs[-1][1] == t.rows
        for (a, b), (c, d) in zip(rs, rs[1:]):
            assert b == c
    # tensors: aligned, non-overlapping on device
    prev_end = 0
    for t in plan.tensors:
        assert t.dev_off % 4096 == 0 and t.dev_off >= prev_end
        prev_end = t.dev_off + t.bytes
    # first-segment partition: the first chunk each GPU loads comes from its own loader set
    # and stages are a contiguous balanced cover
    assert plan.stages[0][0] == 0 and plan.stages[-1][1] == plan.model.n_layers


@pytest.mark.parametrize("arch", ["opt", "llama"])
@pytest.mark.parametrize("policy", [P.STAGE, P.INTERLEAVE])
@pytest.mark.parametrize("sliced", [0, 1])
def test_invariants_sweep(arch, policy, sliced):
    rng = random.Random(1234)
    for _ in range(12):
        L = rng.randint(1, 9)
        N = rng.randint(1, min(L, 5))
        A = rng.randint(0, 3)
        ads = tuple(lora(rng.choice([1, 4, 8]), rng.choice([("q", "v"), ("q",), ("o", "k")])) for _ in range(A))
        cb = rng.choice([4096, 8192, 65536, 1 << 20])
        plan = P.make_plan(tiny(L, arch), ads, N, P.PlanOpts(policy=policy, vocab_sliced=sliced, chunk_bytes=cb))
        check_invariants(plan)


def test_interleave_assignment_and_recv_priority():
    plan = P.make_plan(tiny(8), (lora(4),), 4, P.PlanOpts(policy=P.INTERLEAVE))
    for c in plan.chunks:
        if c.kind == "base":
            t = plan.tensors[c.tensor]
            if t.layer >= 0:
                assert c.loader == t.layer % 4
    # stage g's own layers that others load come first in recv, in layer order
    for g in range(4):
        a, b = plan.stages[g]
        head = []
        for cid in plan.recv[g]:
            lay = plan.tensors[plan.chunks[cid].tensor].layer
            if a <= lay < b:
                head.append(cid)
            else:
                break
        needed = [c.id for c in plan.chunks if c.kind == "base" and c.loader != g
                  and a <= plan.tensors[c.tensor].layer < b]
        assert head == needed


def test_vocab_slices_balanced():
    m = tiny(4)
    plan = P.make_plan(m, (), 3, P.PlanOpts(vocab_sliced=1))
    emb = [c for c in plan.chunks if c.kind == "base" and plan.tensors[c.tensor].name == "embed"]
    per = {}
    for c in emb:
        per[c.loader] = per.get(c.loader, 0) + (c.r1 - c.r0)
    assert sorted(per) == [0, 1, 2] and sum(per.values()) == m.vocab
    assert max(per.values()) - min(per.values()) <= 1 and per[0] >= per[2]


def test_host_alias_layers():
    m = tiny(8)
    plan = P.make_plan(m, (), 2, P.PlanOpts(host_alias_layers=2))
    byname = {t.name: t for t in plan.tensors}
    for l in range(8):
        assert byname[f"L{l}.qkv"].host_off == byname[f"L{l % 2}.qkv"].host_off
    assert len({t.dev_off for t in plan.tensors}) == len(plan.tensors)
    full = P.make_plan(m, (), 2, P.PlanOpts())
    assert plan.host_base_bytes < full.host_base_bytes
    assert plan.dev_weight_bytes == full.dev_weight_bytes


def test_real_shapes_parameter_counts():
    # SURVEY.md §8 "Exact shapes" (HF meta-device counts): OPT-1.3B 1.3158 B params, Llama-2-70B 68.9766 B
    for m, want in ((OPT_1_3B, 1.3158e9), (LLAMA2_70B, 68.9766e9)):
        plan = P.make_plan(m, (), 1, P.PlanOpts())
        n = sum(t.rows * t.cols for t in plan.tensors)
        assert abs(n - want) / want < 1e-4


def test_chunk_rows_multiple_of_128():
    plan = P.make_plan(OPT_1_3B, (lora(16),), 2, P.PlanOpts(chunk_bytes=8 << 20))
    for c in plan.chunks:
        t = plan.tensors[c.tensor] if c.kind == "base" else plan.atensors[c.tensor]
        if c.r1 != t.rows:
            n = c.r1 - c.r0
            assert n % 128 == 0 or n * t.cols * 2 <= 8 << 20
