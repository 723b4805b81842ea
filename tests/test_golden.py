"""The paper's worked examples (tests/golden/*.txt, each citing its passage) against the oracle planner and
the C++ planner behind the C ABI. The fixtures are transcriptions of the paper's text, never outputs of the
code under test."""
import os

import numpy as np
import pytest

from oracle import plan as P
from paper_2503_17707_b200 import _binding as B
from synth.configs import ModelDesc, lora

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_fixture(name):
    """{key: value} and {(key, idx): [ints]} from a fixture (# lines are citations)."""
    out = {}
    for ln in open(os.path.join(GOLDEN, name)):
        ln = ln.strip()
        if not ln or ln.startswith("#"):
            continue
        head, _, rest = ln.partition(":")
        if _:
            parts = head.split()
            vals = rest.split()
            key = (parts[0], int(parts[1])) if len(parts) > 1 else parts[0]
            out[key] = vals
        else:
            k, v = ln.split(None, 1)
            out[k] = int(v)
    return out


def tiny(L):
    return ModelDesc("opt", L, 64, 2, 2, 128, 96, 16, 1)


def layer_of(plan, cid):
    c = plan.chunks[cid]
    return plan.atensors[c.tensor].layer if c.kind == "adapter" else plan.tensors[c.tensor].layer


def seg(stages, layer):
    for g, (a, b) in enumerate(stages):
        if a <= layer < b:
            return g
    return None


def c_dump(model, adapters, n, opts: P.PlanOpts):
    p = B.pb_plan_create(model, adapters, n, B.plan_opts(opts.policy, opts.vocab_sliced, opts.chunk_bytes,
                                                          opts.prefill_chunks, opts.host_alias_layers))
    try:
        return B.pb_plan_dump(p)
    finally:
        B.pb_plan_free(p)


def test_golden_loading_two_gpus():
    f = load_fixture("loading_P234_239.txt")
    opts = P.PlanOpts(policy=P.STAGE)
    plan = P.make_plan(tiny(f["layers"]), (), f["gpus"], opts)
    for g in range(f["gpus"]):
        segs = {seg(plan.stages, layer_of(plan, c)) for c in plan.load[g] if layer_of(plan, c) >= 0}
        assert segs == {int(x) for x in f[("load", g)]}
        got = {seg(plan.stages, layer_of(plan, c)) for c in plan.recv[g] if layer_of(plan, c) >= 0}
        assert got == {int(x) for x in f[("receive", g)]}
    assert c_dump(plan.model, (), f["gpus"], opts) == P.dump(plan)


def test_golden_adapter_parts():
    f = load_fixture("adapters_P242_245.txt")
    ads = tuple(lora(4) for _ in range(f["adapters"]))
    opts = P.PlanOpts(policy=P.STAGE)
    plan = P.make_plan(tiny(f["layers"]), ads, f["gpus"], opts)
    for g in range(f["gpus"]):
        assert plan.own[g] == int(f[("serves", g)][0])
        parts = set()
        for cid in plan.load[g]:
            c = plan.chunks[cid]
            if c.kind == "adapter":
                parts.add(f"{plan.atensors[c.tensor].adapter}-{seg(plan.stages, layer_of(plan, cid))}")
        assert parts == set(f[("parts", g)])
    assert c_dump(plan.model, ads, f["gpus"], opts) == P.dump(plan)


def acquisition(plan, g, block=None):
    """Segments in the order GPU g acquires them: its own loads (or, for a re-plan, its block), then receives."""
    seq = []
    lists = plan.load[g] + plan.recv[g]
    if block is not None:
        seq = list(range(*block))
        lists = plan.recv[g]
    for cid in lists:
        l = layer_of(plan, cid)
        if plan.chunks[cid].kind != "base" or l < 0:
            continue
        if l not in seq:
            seq.append(l)
    return seq


def test_golden_rotation_four_gpus():
    f = load_fixture("rotation_P360_361.txt")
    plan = P.make_plan(tiny(f["layers"]), (), f["gpus"], P.PlanOpts(policy=P.STAGE, chunk_bytes=4096))
    for g in range(f["gpus"]):
        assert acquisition(plan, g) == [int(x) for x in f[("order", g)]]


@pytest.mark.parametrize("impl", ["oracle", "cabi"])
def test_golden_recovery_after_two_crashes(impl):
    """f1: GPUs 1 and 2 of 4 crash during loading."""
    f = load_fixture("recovery_P363_365.txt")
    N, L = f["gpus"], f["layers"]
    model = tiny(L)
    opts = P.PlanOpts(policy=P.STAGE, chunk_bytes=4096)
    plan = P.make_plan(model, (lora(4),), N, opts)
    crashed = {int(x) for x in f["crashed"]}
    alive = [0 if g in crashed else 1 for g in range(N)]
    held_segments = {g: {int(x) for x in f[("held", g)]} for g in range(N) if g not in crashed}
    resident = [[] for _ in range(N)]
    for g, segs in held_segments.items():   # a GPU holds every chunk (base + adapter parts) of its segments
        resident[g] = [c.id for c in plan.chunks if layer_of(plan, c.id) in segs]
    rp = P.replan(plan, alive, resident)
    if impl == "cabi":
        h = B.pb_plan_create(model, (lora(4),), N, B.plan_opts("stage", 0, 4096, 1, 0))
        mask = np.zeros((N, len(plan.chunks)), dtype=np.uint8)
        for g in range(N):
            mask[g, resident[g]] = 1
        hr = B.pb_plan_replan(h, alive, mask)
        try:
            assert B.pb_plan_dump(hr) == P.dump(rp)
            assert [B.pb_plan_gpu_of_rank(hr, r) for r in range(2)] == rp.survivors
        finally:
            B.pb_plan_free(hr)
            B.pb_plan_free(h)
    for r, g in enumerate(rp.survivors):
        assert acquisition(rp, r, block=rp.stages[r]) == [int(x) for x in f[("order", g)]]
        assert list(range(*rp.stages[r])) == [int(x) for x in f[("ready", g)]]
        held = set(resident[g])
        assert not held & set(rp.load[r]) and not held & set(rp.recv[r])   # nothing re-transferred


def test_golden_first_half():
    f = load_fixture("first_half_P262.txt")
    st = P.partition(f["layers"], f["gpus"])
    for g in range(f["gpus"]):
        assert list(st[g]) == [int(x) for x in f[("stage", g)]]


def test_golden_partition_spec():
    f = load_fixture("partition_S130.txt")
    st = P.partition(f["layers"], f["gpus"])
    assert [b - a for a, b in st] == [int(x) for x in f["sizes"]]
