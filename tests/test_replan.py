"""f1 — recovery for model loading: the oracle re-planner against what the
paper fixes, and the C++ pb_plan_replan against the oracle (bit-exact dumps).

Pins (besides the paper's worked example in tests/test_golden.py):
  * Load Balance + Layer Contiguity: blocks contiguous, sizes differ by <= 1;
  * no re-transfer: a chunk a survivor holds is in none of its lists; every base chunk is held, loaded
    or received exactly once per rank (the union is the whole model);
  * every chunk no survivor holds is loaded by exactly one rank — the one whose block needs it;
  * optimality of the block assignment, by an independent enumeration over assignments written with
    per-layer byte counts (not the oracle's loop);
  * a single survivor takes the whole model; all survivors holding nothing = a fresh plan's load set.
"""
import itertools
import random

import numpy as np
import pytest

from oracle import plan as P
from paper_2503_17707_b200 import _binding as B
from synth.configs import AdapterDesc, ModelDesc


def rand_case(rng):
    arch = rng.choice(["opt", "llama"])
    L = rng.randint(2, 9)
    H = rng.choice([2, 4])
    hd = rng.choice([16, 32])
    m = ModelDesc(arch, L, H * hd, H, H if arch == "opt" else rng.choice([1, 2]), rng.choice([64, 96]),
                  rng.randint(40, 200), 16 if arch == "opt" else 0, rng.choice([0, 1]) if arch == "opt" else 0,
                  dtype=rng.choice(["bf16", "f32"]))
    ads = tuple(AdapterDesc(rng.choice([4, 8]), 2.0 * 8, ("q", "v")) for _ in range(rng.randint(0, 2)))
    N = rng.randint(2, min(L, 6))
    opts = P.PlanOpts(policy=rng.choice([P.STAGE, P.INTERLEAVE]), vocab_sliced=rng.choice([0, 1]),
                      chunk_bytes=rng.choice([2048, 8192, 1 << 20]))
    plan = P.make_plan(m, ads, N, opts)
    alive = [rng.random() < 0.6 for _ in range(N)]
    if not any(alive):
        alive[rng.randrange(N)] = True
    # what each GPU holds at the crash: a prefix of its load list (landed + merged) and a prefix of its recv list
    resident = []
    for g in range(N):
        k1 = rng.randint(0, len(plan.load[g]))
        k2 = rng.randint(0, len(plan.recv[g]))
        resident.append(sorted(set(plan.load[g][:k1] + plan.recv[g][:k2])))
    return plan, [int(a) for a in alive], resident, opts


def c_replan_dump(plan, opts, alive, resident):
    h = B.pb_plan_create(plan.model, plan.adapters, plan.n_gpus,
                         B.plan_opts(opts.policy, opts.vocab_sliced, opts.chunk_bytes, opts.prefill_chunks,
                                     opts.host_alias_layers))
    mask = np.zeros((plan.n_gpus, len(plan.chunks)), dtype=np.uint8)
    for g in range(plan.n_gpus):
        mask[g, resident[g]] = 1
    hr = B.pb_plan_replan(h, alive, mask)
    try:
        return B.pb_plan_dump(hr)
    finally:
        B.pb_plan_free(hr)
        B.pb_plan_free(h)


def layer_of(plan, c):
    return plan.atensors[c.tensor].layer if c.kind == "adapter" else plan.tensors[c.tensor].layer


def test_replan_cabi_matches_oracle_sweep():
    rng = random.Random(11)
    for _ in range(120):
        plan, alive, resident, opts = rand_case(rng)
        if sum(alive) > plan.model.n_layers:
            continue
        rp = P.replan(plan, alive, resident)
        assert c_replan_dump(plan, opts, alive, resident) == P.dump(rp)


def test_replan_invariants_and_optimality():
    rng = random.Random(5)
    for _ in range(150):
        plan, alive, resident, _ = rand_case(rng)
        rp = P.replan(plan, alive, resident)
        m = sum(alive)
        assert rp.n_gpus == m and sorted(rp.survivors) == [g for g in range(plan.n_gpus) if alive[g]]
        sizes = [b - a for a, b in rp.stages]
        assert rp.stages[0][0] == 0 and rp.stages[-1][1] == plan.model.n_layers
        assert all(rp.stages[i][1] == rp.stages[i + 1][0] for i in range(m - 1)) and max(sizes) - min(sizes) <= 1
        base = [c.id for c in plan.chunks if c.kind == "base"]
        for r, g in enumerate(rp.survivors):
            held = set(resident[g])
            assert set(rp.resident[r]) == held
            ld, rv = rp.load[r], rp.recv[r]
            assert len(set(ld)) == len(ld) and len(set(rv)) == len(rv)
            assert not held & set(ld) and not held & set(rv) and not set(ld) & set(rv)
            got = [c for c in base if c in held or c in ld or c in rv]
            assert got == base                                     # whole model, each chunk once
            a, b = rp.stages[r]
            for cid in ld:                                         # loads: its block (or its end tensors)
                c = plan.chunks[cid]
                l = layer_of(plan, c)
                assert (a <= l < b) or (l < 0 and c.kind == "base")
        # every chunk no survivor holds is loaded by exactly one rank
        all_held = set().union(*(set(resident[g]) for g in rp.survivors))
        for cid in base:
            n_load = sum(cid in rp.load[r] for r in range(m))
            assert n_load == (0 if cid in all_held else 1), cid
        # optimality, enumerated independently: bytes held per (gpu, layer)
        per = {}
        for g in rp.survivors:
            for cid in resident[g]:
                c = plan.chunks[cid]
                if c.kind == "base" and plan.tensors[c.tensor].layer >= 0:
                    per[(g, plan.tensors[c.tensor].layer)] = per.get((g, plan.tensors[c.tensor].layer), 0) + c.bytes
        def score(assign):   # assign[r] = gpu of block r
            return sum(per.get((assign[r], l), 0) for r in range(m) for l in range(*rp.stages[r]))
        best = max(score(a) for a in itertools.permutations(rp.survivors))
        assert score(rp.survivors) == best


def test_replan_single_survivor_and_nothing_held():
    m = ModelDesc("llama", 6, 64, 4, 2, 96, 80, 0, 0)
    plan = P.make_plan(m, (AdapterDesc(8, 16.0, ("q", "v")),), 3, P.PlanOpts(chunk_bytes=4096))
    rp = P.replan(plan, [0, 1, 0], [[], plan.load[1], []])
    assert rp.stages == [(0, 6)] and rp.survivors == [1] and rp.recv == [[]]
    assert set(rp.load[0]) | set(plan.load[1]) == {c.id for c in plan.chunks}
    rp = P.replan(plan, [1, 1, 1], [[], [], []])
    fresh = P.make_plan(m, plan.adapters, 3, P.PlanOpts(chunk_bytes=4096, policy=P.STAGE))
    assert [sorted(x) for x in rp.load] == [sorted(x) for x in fresh.load]
    with pytest.raises(ValueError):
        P.replan(plan, [0, 0, 0], [[], [], []])


def test_replan_errors_cabi():
    m = ModelDesc("opt", 2, 64, 2, 2, 128, 96, 16, 1)
    h = B.pb_plan_create(m, (), 2, B.plan_opts("stage", 0, 4096, 1, 0))
    n = B.pb_plan_sizes(h).n_chunks
    try:
        with pytest.raises(B.PBError) as e:
            B.pb_plan_replan(h, [0, 0], np.zeros((2, n), np.uint8))
        assert e.value.status == B.PB_EINVAL
        hr = B.pb_plan_replan(h, [1, 1], np.zeros((2, n), np.uint8))
        with pytest.raises(B.PBError) as e:
            B.pb_plan_replan(hr, [1, 1], np.zeros((2, n), np.uint8))
        assert e.value.status == B.PB_EUNSUPPORTED
        B.pb_plan_free(hr)
    finally:
        B.pb_plan_free(h)
