"""f2 — epoch-based adapter scheduling: the oracle (oracle/epoch.py) against the paper / SPEC, and the native
scheduler (pb_epoch_*) against the oracle decision for decision.

Pins: SPEC lora-scheduler examples, FIFO within a queue, conservation of requests
(S:L364), the starvation guard, and the paper's purpose — grouping by adapter needs no more switches
than serving in arrival order ("epoch batching never increases per-stage merges") on streams with the
paper's Fig. 9 setting (two adapters, switch probability 0.2)."""
import random

import pytest

from oracle.epoch import EpochScheduler, eager_switches
from paper_2503_17707_b200 import _binding as B


def test_spec_examples():
    # "epoch expired, queues {B: 5, C: 3}, active B -> switch to C"
    s = EpochScheduler(2, epoch_ms=10)
    for i in range(5):
        s.enqueue(0, i)
    for i in range(3):
        s.enqueue(1, 100 + i)
    s.set_active(0, 0.0)
    a, sw, ids = s.next_batch(5.0, 1)
    assert (a, sw, ids) == (0, False, [0])          # epoch not expired: keep the active adapter
    a, sw, ids = s.next_batch(10.0, 2)
    assert (a, sw, ids) == (1, True, [100, 101])
    # "epoch expired, only B non-empty, active B -> no switch"
    s = EpochScheduler(2, epoch_ms=10)
    s.enqueue(0, 1)
    s.enqueue(0, 2)
    s.set_active(0, 0.0)
    assert s.next_batch(20.0, 1) == (0, False, [1])
    # "queues {B:2, C:2, D:2}, active B, two successive expirations -> C then D"
    s = EpochScheduler(3, epoch_ms=1)
    for a in range(3):
        s.enqueue(a, 10 * a)
        s.enqueue(a, 10 * a + 1)
    s.set_active(0, 0.0)
    assert s.next_batch(1.0, 1)[0] == 1
    assert s.next_batch(2.0, 1)[0] == 2


def test_fifo_conservation_and_no_mixed_batches():
    rng = random.Random(3)
    s = EpochScheduler(3, epoch_ms=4.0)
    sent = {a: [] for a in (-1, 0, 1, 2)}
    got = {a: [] for a in (-1, 0, 1, 2)}
    t, rid = 0.0, 0
    for step in range(400):
        for _ in range(rng.randint(0, 3)):
            a = rng.choice([-1, 0, 1, 2])
            s.enqueue(a, rid)
            sent[a].append(rid)
            rid += 1
        a, sw, ids = s.next_batch(t, 4)
        if a is not None:
            got[a] += ids                                   # one adapter per batch by construction
        t += rng.uniform(0.5, 2.0)
    while True:
        a, sw, ids = s.next_batch(t, 4)
        if a is None:
            break
        got[a] += ids
        t += 1.0
    for a in sent:
        assert got[a] == sent[a]                            # FIFO within each queue, nothing lost


def test_starvation_guard():
    s = EpochScheduler(3, epoch_ms=1.0, starvation_epochs=2)
    s.set_active(0, 0.0)
    s.enqueue(2, 99)
    for i in range(50):
        s.enqueue(0, i)
        s.enqueue(1, 1000 + i)
    seen = []
    t = 0.0
    for _ in range(12):
        a, sw, ids = s.next_batch(t, 1)
        seen.append(a)
        t += 1.0
    assert 2 in seen[:6]                                    # served within a bounded number of epochs


def test_fewer_switches_than_eager():
    """P:L561-565 / Fig. 9: two adapters, switch probability 0.2 between consecutive requests; requests arrive
    faster than they are served, so queues build up and epochs batch them."""
    for seed in range(20):
        rng = random.Random(seed)
        arrivals, a = [], 0
        for _ in range(300):
            if rng.random() < 0.2:
                a = 1 - a
            arrivals.append(a)
        s = EpochScheduler(2, epoch_ms=5.0)
        switches, t, k = 0, 0.0, 0
        s.set_active(arrivals[0], 0.0)
        while True:
            for _ in range(2):                              # 2 arrivals per batch slot
                if k < len(arrivals):
                    s.enqueue(arrivals[k], k)
                    k += 1
            a_, sw, ids = s.next_batch(t, 2)
            if a_ is None and k >= len(arrivals):
                break
            switches += int(sw)
            t += 1.0
        assert switches <= eager_switches(arrivals), seed


def test_native_scheduler_matches_oracle():
    for seed in range(30):
        rng = random.Random(100 + seed)
        A = rng.randint(0, 4)
        ep = rng.choice([0.5, 2.0, 7.0])
        K = rng.randint(1, 4)
        o, n = EpochScheduler(A, ep, K), B.EpochScheduler(A, ep, K)
        if rng.random() < 0.5:
            a0 = rng.randint(-1, A - 1)
            o.set_active(a0, 0.0)
            n.set_active(a0, 0.0)
        t, rid = 0.0, 0
        for step in range(300):
            for _ in range(rng.randint(0, 3)):
                a = rng.randint(-1, A - 1)
                o.enqueue(a, rid)
                n.enqueue(a, rid)
                rid += 1
            mb = rng.randint(1, 4)
            assert o.next_batch(t, mb) == n.next_batch(t, mb), (seed, step)
            t += rng.uniform(0.1, 3.0)


def test_native_errors():
    with pytest.raises(B.PBError):
        B.EpochScheduler(2, 0.0)
    s = B.EpochScheduler(1, 1.0)
    with pytest.raises(B.PBError):
        s.enqueue(5, 1)
    assert s.next_batch(0.0, 4) == (None, False, [])
