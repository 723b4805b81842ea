// storage.hpp — f4: the checkpoint read from a file into pinned staging slots, overlapped with the DMA.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <thread>
#include <vector>

namespace pb {

struct CopyGroup;

struct FileSource {
    enum : int { kFree = 0, kReady = 2, kIssued = 3 };
    // Slot k serves the file-backed groups with file index fi = k, k + n, k + 2n, ... in that order: `turn` is the
    // file index it may be filled for next, advanced by n only when the DMA of the previous occupant has landed.
    // A reader that runs ahead therefore waits for its own turn instead of writing into a slot still being
    // filled (or not yet copied) for an earlier group.
    struct Slot {
        char* buf = nullptr;
        std::atomic<int> state{kFree};
        std::atomic<int> parts{0};        // reader threads done with this fill
        std::atomic<int64_t> turn{0};     // file index this slot is being (or may next be) filled for
        int64_t group = -1;
        cudaEvent_t landed = nullptr;
    };
    std::vector<int64_t> fidx;   // copy group -> file index (-1: not read from the file)
    int fd = -1;          // O_DIRECT when the file system accepts it
    int fd_buffered = -1; // for reads whose offset is not 4 KiB aligned
    bool direct = false;
    std::vector<Slot> slots;
    std::vector<std::thread> readers;   // each reads its 1/R slice of every group (host memcpy / NVMe queues)
    int n_readers = 16;
    std::atomic<bool> stop{false};
    std::atomic<int> read_error{0};
    int64_t n_groups = 0;

    ~FileSource();
    void start(const std::vector<CopyGroup>& groups, const char* host_base);
    void stop_reader();
    const char* ready(int64_t gi);
    void issued(int64_t gi, cudaEvent_t landed);
    void reclaim();
};

}  // namespace pb
