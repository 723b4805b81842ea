// runtime.hpp — per-rank context (pb_ctx) internals.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <thread>
#include <vector>

#include "kernels.hpp"
#include "plan.hpp"
#include "storage.hpp"

#include <atomic>
#include <memory>
#include <mutex>

namespace pb {

struct TrialRun;   // the trial issuer's state (runtime.cpp)

// Workspace layout (byte offsets inside the caller's workspace buffer), identical on every rank so a
// peer can address it: flags | tokens | h | x | qkv[n_qkv] | attn | mlp | y | logits | tok_out | nan | rope.
struct WsLayout {
    int64_t flags = 0, tokens = 0, h = 0, x = 0, qkv = 0, qkv_stride = 0, attn = 0, mlp = 0, y = 0, logits = 0,
            tok_out = 0, nan = 0, rope = 0, held = 0, dpos = 0, total = 0;
    int32_t n_qkv = 1;
    int32_t max_rows = 0, max_batch = 0, max_seq = 0;
    // readiness words (uint32) inside `flags`
    int32_t f_chunk = 0, f_act = 0, f_y = 0, f_logit = 0, n_words = 0;
    int32_t f_land = 0, f_tensor = 0;   // local words: copy group landed (by first chunk id), tensor ready
    int32_t f_tensor_recv = 0;          // local words: the received part of a tensor is in place
    int32_t f_gdone = 0;                // word f_gdone + r: rank r has received every chunk it gathers (T_full on r)
};
WsLayout ws_layout(const pb_plan* p, int32_t batch, int32_t seq);

struct MergeJob {
    int32_t chunk;       // base chunk whose rows it updates
    int32_t adapter;
    bool inplace;        // true: into the base weights; false: into adapter's out-of-place copy
    int32_t rows, cols, rank;
    float scale;
    std::vector<int32_t> need;   // adapter chunks that must have landed
    MergeMaps maps;              // bf16 path (TMA)
    // fp32 debug-parity path: plain pointers
    const float *W = nullptr, *Bp = nullptr, *Ap = nullptr;
    float* Wout = nullptr;
    int64_t ldw = 0;
};

// One cudaMemcpyAsync of the load list: a run of consecutive load-list chunks that are contiguous (up to
// alignment padding) in both the host image and the device buffer.
struct CopyGroup {
    const char* src;
    char* dst;
    int64_t bytes;
    int32_t first, count;   // range in the rank's load list
    bool from_file = false; // f4: staged from the checkpoint file (pb_ctx_set_file_source)
};

struct LayerMaps {
    CUtensorMap qkv, o, up, down;   // up = fc1 (OPT) or [gate; up] with 64-row boxes (Llama)
    const __nv_bfloat16* w[4];      // the same four weights as plain pointers (GEMV path)
    CUtensorMap w64[4];             // 64-row boxes for 64-column tiles (not for [gate; up])
    CUtensorMap w32[4];             // 32-row boxes for the persistent kernel's 160- / 224-column tiles (idem)
};

struct Peer {
    char* weights = nullptr;
    char* ws = nullptr;
    bool linked = false;
    std::vector<void*> ipc_bases;   // cudaIpcOpenMemHandle results to close
};

constexpr int32_t kMaxBatch = 64;   // sequences per trial (the paper's TTFT workload is 64 x 64)
enum class Phase { Idle, Begun, Loaded, Merged, Gathered, Prefilled };
constexpr int kEventPool = 64;

// Kernel classes timed by the optional per-launch profiler (pb_ctx_set_profiling).
enum KClass : int { K_MERGE = 0, K_GEMM, K_ATTN, K_NORM, K_ROPE, K_EMBED, K_LOGITS, K_ARGMAX, K_SIGNAL, K_NCLASS };
struct ProfRec {
    int cls;
    cudaEvent_t a, b;
    double flops, bytes;
};

}  // namespace pb

struct pb_ctx {
    const pb_plan* plan;
    int32_t rank, n;
    int device;
    char* weights;
    char* adapters;
    char* ws;
    pb_rank_bufs bufs;
    cudaStream_t h2d[2], merge, nv, comp;
    pb::WsLayout L;
    const void* host_base;
    const void* host_adapters;
    std::vector<pb::Peer> peers;

    // events
    cudaEvent_t t0 = nullptr, merge_done = nullptr, gather_done = nullptr, done = nullptr;
    cudaEvent_t load_end = nullptr;   // timing event after the last copy group (load_done)
    // per-group landed events carry timestamps (chunk_landed_ms) only with PB_LANDED_TIMING=1: measured on B200,
    // a timing-event record on the saturated copy lane costs ~20 us (C2 at 128 MB groups: 0.9895 -> 0.9934 of the
    // PCIe bound without them)
    bool landed_timing = false;
    cudaEvent_t ready_merge = nullptr, ready_recv = nullptr;   // timing: last stage chunk merged / received
    cudaEvent_t tok_ev = nullptr;                               // prompt tokens landed (copy lane)
    cudaEvent_t trial_fence[4] = {};                            // previous trial's streams drained (trial begin)
    int32_t last_own_stage_chunk = -1, last_recv_stage_chunk = -1;
    std::vector<cudaEvent_t> landed, gathered;
    std::vector<cudaEvent_t> merged_ev;          // per own chunk, after its merges (timing mode only)
    cudaEvent_t stage_begin = nullptr, stage_end = nullptr;   // first / last layer item of this rank's stage
    double ctx_create_ms = 0;                    // host time of pb_ctx_create (tables, TMA maps, events, staging)
    std::vector<char> tensor_own;        // this rank loads every piece of the tensor
    std::vector<int32_t> last_own_chunk; // per base tensor: last own chunk in load order (-1 if none)
    std::vector<int32_t> last_recv_chunk;
    int32_t n_held_src = 0;              // re-plan: chunks this rank holds and other ranks receive from it

    std::vector<pb::CopyGroup> copies;
    std::unique_ptr<pb::FileSource> file;   // f4: checkpoint file reader (null: pinned host image)
    std::vector<int32_t> landed_alias;   // chunk -> first chunk of its copy group (owner of the landed event)

    // merges: per chunk, indices into jobs
    std::vector<pb::MergeJob> jobs;
    std::vector<std::vector<int32_t>> jobs_of_chunk;

    // prefill tensor maps
    CUtensorMap map_x, map_attn, map_mlp;
    std::vector<pb::LayerMaps> lmaps;   // indexed by layer (only this rank's stage is encoded)
    // multi-adapter (PB_MERGE_ALL): out-of-place copies and per-adapter weight maps [adapter][layer]
    char* adapted = nullptr;
    char* backup = nullptr;              // f2: pristine copies of adapted tensors (bufs.backup), or null
    std::vector<char> in_load;           // chunk is in this rank's load list (its pristine bytes were saved here)
    std::vector<std::vector<pb::LayerMaps>> lmaps_ad;
    std::vector<int32_t> seq_adapter;   // per sequence of the current trial (-1: base / single in-place adapter)

    // pinned staging
    int32_t* h_tokens = nullptr;   // [max_rows]
    int32_t* h_out = nullptr;      // [max_batch + 1] tokens + nan flag

    // trial state
    uint32_t epoch = 0;
    uint32_t cold_epoch = 0;   // epoch of the last cold start (pb_trial_begin): the trial whose gather peers signal
    pb::Phase phase = pb::Phase::Idle;
    int32_t cur_batch = 0, cur_seq = 0;
    int32_t n_launches = 0;
    int64_t load_bytes = 0, recv_bytes = 0;
    std::vector<double> tl_landed, tl_gathered, tl_merged;
    bool use_wait_value = true;
    std::thread load_thread;                 // the trial issuer (see run_loop)
    std::shared_ptr<pb::TrialRun> run;       // the current trial's issuer state (cold start: from pb_gather_layers)
    std::mutex run_mu;                       // prompt hand-off between pb_prefill_enqueue and the issuer thread
    std::atomic<bool> posted{false};         // the trial's prompt is staged (cur_batch, cur_seq, h_tokens)
    bool loader_idle = true;                 // the issuer thread has issued everything posted so far and exited
    std::atomic<bool> abort_req{false};      // pb_ctx_abort: the issuer stops at its next poll
    bool aborted = false;                    // readiness words forced open; the ctx can only be freed
    pb_status issue_status = PB_OK;
    char issue_msg[512] = "";
    int32_t merge_adapter = -1;
    int32_t cold_adapter = -1;   // adapter merged by the cold start (every gathered copy of other stages holds it)
    std::vector<cudaEvent_t> budget_events;
    std::vector<cudaStream_t> owned_streams;   // created by the ctx when the caller passed NULL  // 4 streams x kEventPool progress marks
    bool profiling = false;
    // Warm replay as a CUDA graph (single-rank contexts): captured once per (batch, seq, profiling) and
    // relaunched, so the prefill's ~200 launches cost one host call instead of ~4 us of issue time each.
    bool capturing = false;
    // f3: replica mode (the whole model on this GPU, after T_full) and decode-step state
    bool replica = false;
    int32_t decode_t = -1;       // position of the token the current decode trial computes (-1: a prompt trial)
    int32_t n_decoded = 0;       // decode steps since the last prompt trial
    bool prompt_replica = false; // the last prompt trial ran in replica mode (its KV cache covers every layer)
    int32_t gemm_m_total = 0;    // rows that pick the GEMM split-K (whole prompt batch, or one decode step)
    // decode graphs (single rank / replica): captured once per batch size with every position read on the device
    const int* dyn_pos = nullptr;  // set while capturing a decode graph: device int holding the step's position
    int32_t* h_pos = nullptr;      // pinned: the host writes the position here before each graph launch
    struct DecodeGraph {
        int32_t B;
        cudaGraphExec_t exec;
        int32_t launches;
    };
    std::vector<DecodeGraph> decode_graphs;
    struct ReplayGraph {
        int32_t B, T, profiled, replica;
        cudaGraphExec_t exec;
        int32_t launches;
        size_t prof_n;
        std::vector<pb::ProfRec> prof;   // class / algorithmic work of each timed launch (events shared)
    };
    std::vector<ReplayGraph> replay_graphs;
    std::vector<pb::ProfRec> prof;
    size_t prof_n = 0;
};
