// epoch.cpp — f2 epoch-based adapter scheduling (§4.3.2; SPEC lora-scheduler S:L340-405), host side.
// Per-adapter FIFO queues (plus the base-model queue, adapter -1); batches come from the active adapter while
// its epoch lasts; on expiry the next non-empty queue in round-robin order (ids ascending, base first) takes
// over, a queue left waiting over more than K expirations first (starvation guard); an empty active queue
// hands over at once. The decision tells the caller whether the stages must switch (pb_switch_adapter) before
// the batch. Same algorithm as oracle/epoch.py (decisions compared in tests/test_epoch.py).
#include <algorithm>
#include <deque>
#include <vector>

#include "../../include/pipeboost.h"
#include "errors.hpp"

struct pb_epoch {
    std::vector<std::deque<int64_t>> q;   // index = adapter + 1 (0 = base model)
    std::vector<int64_t> waited;
    double epoch_ms = 0, epoch_start = 0;
    int32_t K = 3;
    int32_t active = -2;                  // -2: none yet (index active + 1)
};

namespace {
bool any_nonempty(const pb_epoch* e) {
    for (auto& d : e->q)
        if (!d.empty()) return true;
    return false;
}
// first non-empty queue after `a` (round-robin over indices 0..n-1), a itself excluded; -2 if none
int32_t next_after(const pb_epoch* e, int32_t a) {
    const int32_t n = (int32_t)e->q.size();
    const int32_t start = a == -2 ? 0 : a + 2;   // index of a is a + 1
    for (int32_t i = 0; i < n; ++i) {
        const int32_t idx = (start + i) % n, b = idx - 1;
        if (b != a && !e->q[idx].empty()) return b;
    }
    return -2;
}
}  // namespace

extern "C" pb_status pb_epoch_create(int32_t n_adapters, double epoch_ms, int32_t starvation_epochs, pb_epoch** out) {
    if (!out) return pb::fail(PB_EINVAL, "pb_epoch_create: null out");
    if (n_adapters < 0 || !(epoch_ms > 0) || starvation_epochs < 1)
        return pb::fail(PB_EINVAL, "pb_epoch_create: n_adapters >= 0, epoch_ms > 0, starvation_epochs >= 1");
    auto* e = new pb_epoch();
    e->q.resize(n_adapters + 1);
    e->waited.assign(n_adapters + 1, 0);
    e->epoch_ms = epoch_ms;
    e->K = starvation_epochs;
    *out = e;
    return PB_OK;
}

extern "C" pb_status pb_epoch_set_active(pb_epoch* e, int32_t adapter, double now_ms) {
    if (!e) return pb::fail(PB_EINVAL, "pb_epoch_set_active: null scheduler");
    if (adapter < -1 || adapter + 1 >= (int32_t)e->q.size()) return pb::fail(PB_EINVAL, "adapter %d out of range", adapter);
    e->active = adapter;
    e->epoch_start = now_ms;
    return PB_OK;
}

extern "C" pb_status pb_epoch_enqueue(pb_epoch* e, int32_t adapter, int64_t request_id) {
    if (!e) return pb::fail(PB_EINVAL, "pb_epoch_enqueue: null scheduler");
    if (adapter < -1 || adapter + 1 >= (int32_t)e->q.size()) return pb::fail(PB_EINVAL, "unknown adapter %d", adapter);
    e->q[adapter + 1].push_back(request_id);
    return PB_OK;
}

extern "C" pb_status pb_epoch_next(pb_epoch* e, double now_ms, int32_t max_batch, int32_t* adapter,
                                   int32_t* switch_needed, int64_t* ids, int32_t* n) {
    if (!e || !adapter || !switch_needed || !ids || !n) return pb::fail(PB_EINVAL, "pb_epoch_next: null argument");
    if (max_batch < 1) return pb::fail(PB_EINVAL, "max_batch must be >= 1");
    *n = 0;
    *switch_needed = 0;
    if (!any_nonempty(e)) {
        *adapter = -2;
        return PB_OK;
    }
    int32_t target = e->active;
    if (e->active == -2 || e->q[e->active + 1].empty()) {
        target = next_after(e, e->active);
        e->epoch_start = now_ms;
    } else if (now_ms - e->epoch_start >= e->epoch_ms) {
        const int32_t nq = (int32_t)e->q.size();
        for (int32_t i = 0; i < nq; ++i)
            if (i - 1 != e->active && !e->q[i].empty()) ++e->waited[i];
        int32_t starved = -2;
        for (int32_t i = 0; i < nq; ++i)   // most-waited starved queue, earliest in order on ties
            if (i - 1 != e->active && !e->q[i].empty() && e->waited[i] > e->K &&
                (starved == -2 || e->waited[i] > e->waited[starved + 1]))
                starved = i - 1;
        if (starved != -2) {
            target = starved;
        } else {
            const int32_t nx = next_after(e, e->active);
            target = nx != -2 ? nx : e->active;
        }
        e->epoch_start = now_ms;
    }
    *switch_needed = target != e->active ? 1 : 0;
    e->active = target;
    e->waited[target + 1] = 0;
    auto& dq = e->q[target + 1];
    while (*n < max_batch && !dq.empty()) {
        ids[(*n)++] = dq.front();
        dq.pop_front();
    }
    *adapter = target;
    return PB_OK;
}

extern "C" void pb_epoch_free(pb_epoch* e) { delete e; }
