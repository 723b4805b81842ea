"""pb_plan (C++, through the C ABI) vs the oracle planner: bit-exact text dumps.

North star: "The GPU path must match the oracle bit-exactly for the plan".
The sweep spans both architectures, both load policies, vocab slicing, several
chunk sizes, 0..3 adapters with different target sets and ranks, host layer
aliasing and N in 1..8, plus the real model shapes of every config.
"""
import random

import pytest

from oracle import plan as OP
from paper_2503_17707_b200 import _binding as B
from synth.configs import WORKLOADS, AdapterDesc, ModelDesc, TINY_LLAMA, TINY_OPT, lora


def c_dump(model, adapters, n, policy, sliced, cb, k=1, alias=0):
    p = B.pb_plan_create(model, adapters, n, B.plan_opts(policy, sliced, cb, k, alias))
    try:
        return B.pb_plan_dump(p)
    finally:
        B.pb_plan_free(p)


def o_dump(model, adapters, n, policy, sliced, cb, k=1, alias=0):
    return OP.dump(OP.make_plan(model, adapters, n, OP.PlanOpts(policy, sliced, cb, k, alias)))


@pytest.mark.parametrize("tag", ["C1", "C1f32"])
def test_dump_c1_matches(tag):
    w = WORKLOADS[tag]
    for n, policy, sliced, cb in [(2, "stage", 0, 32 << 20), (2, "interleave", 1, 4 << 10), (4, "stage", 1, 64 << 10)]:
        a = c_dump(w.model, w.adapters, n, policy, sliced, cb)
        b = o_dump(w.model, w.adapters, n, policy, sliced, cb)
        assert a == b, (tag, n, policy)
    if tag == "C1f32":   # 4-byte elements: twice the bytes of the bf16 plan, same tensor table
        assert "dtype=f32" in a


@pytest.mark.parametrize("tag", ["C2", "C3", "C4", "C5a", "C5b"])
@pytest.mark.parametrize("policy", ["stage", "interleave"])
def test_dump_real_configs(tag, policy):
    w = WORKLOADS[tag]
    for n in (1, 2, 8):
        for sliced in (0, 1):
            assert c_dump(w.model, w.adapters, n, policy, sliced, 64 << 20) == \
                o_dump(w.model, w.adapters, n, policy, sliced, 64 << 20), (tag, n, sliced)


def test_dump_random_sweep():
    rng = random.Random(7)
    for it in range(150):
        arch = rng.choice(["opt", "llama"])
        L = rng.randint(1, 10)
        H = rng.choice([1, 2, 4])
        hd = rng.choice([8, 16, 32])
        kvh = H if arch == "opt" else rng.choice([h for h in (1, 2, 4) if H % h == 0])
        m = ModelDesc(arch, L, H * hd, H, kvh, rng.choice([16, 48, 96]), rng.randint(8, 300),
                      rng.randint(1, 40) if arch == "opt" else 0, rng.choice([0, 1]) if arch == "opt" else 0,
                      dtype=rng.choice(["bf16", "bf16", "f32"]))
        tg = ("q", "k", "v", "o", "fc1", "fc2") if arch == "opt" else ("q", "k", "v", "o", "gate", "up", "down")
        ads = tuple(AdapterDesc(rng.choice([1, 3, 8, 16, 64]), rng.choice([1.0, 2.5, 16.0]),
                                tuple(t for t in tg if rng.random() < 0.5) or ("q",))
                    for _ in range(rng.randint(0, 3)))
        n = rng.randint(1, min(L, 8))
        pol = rng.choice(["stage", "interleave"])
        sl = rng.choice([0, 1])
        cb = rng.choice([2, 100, 4096, 5000, 1 << 16, 1 << 22])
        alias = rng.choice([0, 0, 1, 2, 3])
        assert c_dump(m, ads, n, pol, sl, cb, 1, alias) == o_dump(m, ads, n, pol, sl, cb, 1, alias), it


def test_partition_error_status():
    with pytest.raises(B.PBError) as e:
        B.pb_plan_create(TINY_OPT, (), 5, B.plan_opts())
    assert e.value.status == B.PB_EPARTITION


def test_invalid_arguments():
    with pytest.raises(B.PBError) as e:
        B.pb_plan_create(TINY_OPT, (lora(65),), 2, B.plan_opts())
    assert e.value.status == B.PB_EUNSUPPORTED
    with pytest.raises(B.PBError) as e:
        B.pb_plan_create(TINY_OPT, (AdapterDesc(4, 8.0, ("gate",)),), 2, B.plan_opts())
    assert e.value.status == B.PB_EINVAL
    with pytest.raises(B.PBError) as e:
        B.pb_plan_create(TINY_OPT, (), 0, B.plan_opts())
    assert e.value.status == B.PB_EINVAL


def test_tensor_accessors_match_oracle_table():
    w = WORKLOADS["C1"]
    p = B.pb_plan_create(w.model, w.adapters, 2, B.plan_opts())
    o = OP.make_plan(w.model, w.adapters, 2, OP.PlanOpts())
    s = B.pb_plan_sizes(p)
    assert s.n_tensors == len(o.tensors) and s.n_chunks == len(o.chunks)
    for i, t in enumerate(o.tensors):
        c = B.pb_plan_tensor(p, i)
        assert (c.name.decode(), c.rows, c.cols, c.layer, c.host_off, c.dev_off) == \
            (t.name, t.rows, t.cols, t.layer, t.host_off, t.dev_off)
    for i, t in enumerate(o.atensors):
        c = B.pb_plan_atensor(p, i)
        assert (c.name.decode(), c.rows, c.cols, c.off, c.base_tensor, c.base_row0) == \
            (t.name, t.rows, t.cols, t.off, t.base, t.row0)
    B.pb_plan_free(p)
