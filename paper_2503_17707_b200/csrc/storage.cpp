// storage.cpp — f4 storage tier: the checkpoint comes from a FILE
// (NVMe / any POSIX file in the canonical host layout) instead of an image already resident in pinned DRAM.
// A reader thread per rank pread()s the rank's own copy groups, in load order, into a ring of pinned staging
// slots; the trial issuer DMAs a slot to HBM as soon as it is filled and hands it back to the reader when
// that copy's `landed` event has completed — so disk reads, PCIe DMA and merges overlap chunk by chunk, and
// every GPU reads only its own disjoint slice (aggregate storage bandwidth, like the PCIe links).
// O_DIRECT is used when the file system accepts it (no page-cache copy); reads are then rounded up to 4 KiB
// (tensor offsets are 4 KiB aligned by the plan; the staging slots are page aligned).
#include "storage.hpp"

#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>

#include "errors.hpp"
#include "runtime.hpp"

namespace pb {

namespace {
constexpr int64_t kDirectAlign = 4096;
}

FileSource::~FileSource() {
    stop_reader();
    if (fd >= 0) close(fd);
    if (fd_buffered >= 0) close(fd_buffered);
}

void FileSource::stop_reader() {
    stop.store(true);
    for (auto& t : readers)
        if (t.joinable()) t.join();
    readers.clear();
    stop.store(false);
}

void FileSource::start(const std::vector<CopyGroup>& groups, const char* host_base) {
    stop_reader();
    n_groups = (int64_t)groups.size();
    fidx.assign(groups.size(), -1);
    for (int64_t gi = 0, fi = 0; gi < n_groups; ++gi)
        if (groups[gi].from_file) fidx[gi] = fi++;
    for (size_t k = 0; k < slots.size(); ++k) {
        Slot& s = slots[k];
        s.state.store(kFree);
        s.parts.store(0);
        s.turn.store((int64_t)k);
        s.group = -1;
    }
    read_error.store(0);
    // R reader threads walk the groups in load order in lockstep; thread t reads slice t of every group (4 KiB
    // aligned for O_DIRECT) and the last one to finish a group publishes its slot.
    for (int t = 0; t < n_readers; ++t)
        readers.emplace_back([this, &groups, host_base, t]() {
            for (int64_t gi = 0; gi < n_groups && !stop.load(); ++gi) {
                const CopyGroup& g = groups[gi];
                if (!g.from_file) continue;
                const int64_t fi = fidx[gi];
                Slot& s = slots[fi % slots.size()];
                // free AND this group's turn (reclaim advances `turn` before it frees the slot)
                while (s.state.load(std::memory_order_acquire) != kFree || s.turn.load(std::memory_order_acquire) != fi)
                    if (stop.load()) return;
                    else std::this_thread::sleep_for(std::chrono::microseconds(2));
                const int64_t off = g.src - host_base;
                const bool use_direct = direct && off % kDirectAlign == 0;
                const int rfd = use_direct ? fd : fd_buffered;
                const int64_t total = use_direct ? (g.bytes + kDirectAlign - 1) / kDirectAlign * kDirectAlign : g.bytes;
                const int64_t unit = use_direct ? kDirectAlign : 1;
                const int64_t units = (total + unit - 1) / unit;
                const int64_t a = units * t / n_readers * unit, b = std::min(total, units * (t + 1) / n_readers * unit);
                for (int64_t done = a; done < b;) {
                    const ssize_t r = pread(rfd, s.buf + done, (size_t)(b - done), (off_t)(off + done));
                    if (r < 0 && errno == EINTR) continue;
                    if (r <= 0) {
                        if (done >= g.bytes) break;   // O_DIRECT round-up past the end of the file
                        read_error.store(r < 0 ? errno : EIO);
                        break;
                    }
                    done += r;
                }
                if (s.parts.fetch_add(1, std::memory_order_acq_rel) + 1 == n_readers) {
                    s.parts.store(0, std::memory_order_relaxed);
                    s.group = gi;
                    s.state.store(kReady, std::memory_order_release);
                }
            }
        });
}

// The staging slot holding group gi once the reader has filled it, else null.
const char* FileSource::ready(int64_t gi) {
    if (gi < 0 || gi >= (int64_t)fidx.size() || fidx[gi] < 0) return nullptr;
    Slot& s = slots[fidx[gi] % slots.size()];
    if (s.state.load(std::memory_order_acquire) != kReady) return nullptr;
    if (s.group != gi) return nullptr;
    return s.buf;
}

void FileSource::issued(int64_t gi, cudaEvent_t landed) {
    Slot& s = slots[fidx[gi] % slots.size()];
    s.landed = landed;
    s.state.store(kIssued, std::memory_order_release);
}

// Hand back every slot whose DMA has completed (called by the issuer while it polls).
void FileSource::reclaim() {
    for (auto& s : slots)
        if (s.state.load(std::memory_order_acquire) == kIssued && cudaEventQuery(s.landed) == cudaSuccess) {
            s.turn.store(s.turn.load(std::memory_order_relaxed) + (int64_t)slots.size(), std::memory_order_release);
            s.state.store(kFree, std::memory_order_release);
        }
}

}  // namespace pb

extern "C" pb_status pb_ctx_set_file_source(pb_ctx* c, const char* path, void* staging, int64_t staging_bytes) {
    using namespace pb;
    if (!c) return fail(PB_EINVAL, "pb_ctx_set_file_source: null ctx");
    if (c->phase == Phase::Loaded || c->phase == Phase::Merged || c->phase == Phase::Gathered)
        return fail(PB_EPROTOCOL, "pb_ctx_set_file_source: a trial is being armed");
    if (c->load_thread.joinable()) c->load_thread.join();
    c->file.reset();
    for (auto& g : c->copies) g.from_file = false;
    if (!path) return PB_OK;
    if (!staging || staging_bytes <= 0) return fail(PB_EINVAL, "pb_ctx_set_file_source: staging buffer needed");
    if (reinterpret_cast<uintptr_t>(staging) % 4096) return fail(PB_EINVAL, "staging must be 4 KiB aligned");
    int64_t slot = 0;
    for (auto& g : c->copies)
        if (!c->plan->chunks[c->plan->load[c->rank][g.first]].is_adapter) slot = std::max(slot, g.bytes);
    slot = (slot + 4095) / 4096 * 4096;
    int64_t n_slots = slot ? staging_bytes / slot : 0;
    if (const char* ns = getenv("PB_FILE_SLOTS")) n_slots = std::min<int64_t>(n_slots, std::max(2, atoi(ns)));
    if (slot && n_slots < 2)
        return fail(PB_ENOMEM, "staging: need >= 2 slots of %lld bytes (%lld given)", (long long)slot,
                    (long long)staging_bytes);
    auto fs = std::make_unique<FileSource>();
    fs->fd_buffered = open(path, O_RDONLY);
    if (fs->fd_buffered < 0)
        return fail(PB_EINVAL, "pb_ctx_set_file_source: cannot open %s: %s", path, strerror(errno));
    fs->fd = open(path, O_RDONLY | O_DIRECT);
    fs->direct = fs->fd >= 0;
    // one reader per host core up to 16 (measured on the B200 box, 16 cores, C2 from tmpfs: 8 readers 34.5 GB/s,
    // 16 readers 43 GB/s; a single pread() stream tops out near 5.7 GB/s); PB_FILE_READERS overrides
    fs->n_readers = (int)std::min<unsigned>(16, std::max(1u, std::thread::hardware_concurrency()));
    if (const char* r = getenv("PB_FILE_READERS")) fs->n_readers = std::max(1, atoi(r));
    fs->slots = std::vector<FileSource::Slot>((size_t)n_slots);
    for (int64_t i = 0; i < n_slots; ++i) fs->slots[i].buf = static_cast<char*>(staging) + i * slot;
    for (auto& g : c->copies)
        g.from_file = !c->plan->chunks[c->plan->load[c->rank][g.first]].is_adapter;
    c->file = std::move(fs);
    return PB_OK;
}
