"""f2 — epoch-based adapter scheduling (TEST INFRASTRUCTURE ONLY; see oracle/plan.py header).

Written from the paper's §4.3.2 and SPEC's lora-scheduler:
  1. "classifies requests and groups those belonging to the same adapter into the same queue"
     -> one FIFO queue per adapter, plus one for base-model requests (adapter -1).
  2. "prioritizes the scheduling of batches corresponding to the currently activated adapter"
     -> while the epoch lasts, batches come from the active adapter's queue.
  3. "At regular intervals, PipeBoost switches adapters to serve requests from other batches"
     -> when the epoch has expired and another queue is non-empty, switch to the next non-empty queue in
        round-robin order; if the active queue is empty, switch at once (nothing to prioritise).
  4. Starvation guard: a queue that stayed non-empty and inactive over more than K epoch
     expirations is scheduled next, before round-robin.
Round-robin order: adapter ids ascending with the base queue (-1) first, wrapping around.
Plain Python lists; the stage-by-stage application of a switch is the GPU's pb_switch_adapter.
"""
from __future__ import annotations

from collections import deque
from typing import List, Optional, Tuple


class EpochScheduler:
    def __init__(self, n_adapters: int, epoch_ms: float, starvation_epochs: int = 3):
        if n_adapters < 0 or not epoch_ms > 0 or starvation_epochs < 1:
            raise ValueError("bad scheduler config")
        self.order = list(range(-1, n_adapters))            # round-robin order
        self.q = {a: deque() for a in self.order}
        self.epoch_ms = epoch_ms
        self.K = starvation_epochs
        self.active: Optional[int] = None
        self.epoch_start = 0.0
        self.waited = {a: 0 for a in self.order}           # expirations survived non-empty and inactive

    def set_active(self, adapter: Optional[int], now_ms: float = 0.0) -> None:
        """The adapter the stages currently hold (e.g. the one the cold start merged); starts an epoch."""
        self.active = adapter
        self.epoch_start = now_ms

    def enqueue(self, adapter: int, request_id: int) -> None:
        if adapter not in self.q:
            raise ValueError(f"unknown adapter {adapter}")
        self.q[adapter].append(request_id)

    def _next_after(self, a: Optional[int]) -> Optional[int]:
        """First non-empty queue after `a` in round-robin order, `a` itself excluded."""
        n = len(self.order)
        start = 0 if a is None else self.order.index(a) + 1
        for i in range(n):
            b = self.order[(start + i) % n]
            if b != a and self.q[b]:
                return b
        return None

    def next_batch(self, now_ms: float, max_batch: int) -> Tuple[Optional[int], bool, List[int]]:
        """(adapter, switch_needed, request ids) of the batch to run now; (None, False, []) when all queues are empty."""
        if not any(self.q.values()):
            return None, False, []
        target = self.active
        if self.active is None or not self.q[self.active]:
            target = self._next_after(self.active)               # nothing left to prioritise: move on now
            self.epoch_start = now_ms
        elif now_ms - self.epoch_start >= self.epoch_ms:         # epoch expired
            for a in self.order:
                if a != self.active and self.q[a]:
                    self.waited[a] += 1
            starved = [a for a in self.order if a != self.active and self.q[a] and self.waited[a] > self.K]
            if starved:
                target = max(starved, key=lambda a: (self.waited[a], -self.order.index(a)))
            else:
                nxt = self._next_after(self.active)
                target = nxt if nxt is not None else self.active
            self.epoch_start = now_ms
        switched = target != self.active
        self.active = target
        self.waited[target] = 0
        ids = [self.q[target].popleft() for _ in range(min(max_batch, len(self.q[target])))]
        return target, switched, ids


def eager_switches(adapters_in_arrival_order) -> int:
    """SPEC eager_switch_baseline: serve strictly in arrival order, switching whenever the next
    request's adapter differs from the active one."""
    n, active = 0, None
    for a in adapters_in_arrival_order:
        if active is not None and a != active:
            n += 1
        active = a
    return n
