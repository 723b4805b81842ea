// runtime.cpp — pb_ctx: the per-rank cold-start engine.
//
//   pb_load_shard    (a2)  chunked cudaMemcpyAsync pinned host -> HBM over this GPU's own PCIe link,
//                          one ordered copy-engine lane; a `landed` event per chunk
//   pb_merge_lora    (a3)  per own chunk in load order: wait landed, tcgen05 merge of every adapted row
//                          range (after its adapter factors land), then publish the chunk to the peers
//                          (readiness word = epoch) and record per-tensor readiness
//   pb_gather_layers (a4)  receive list: wait the loader's readiness word (cuStreamWaitValue32 on local
//                          memory), copy peer HBM -> local HBM over NVLink (copy engine)
//   pb_prefill_*     (a5)  pipelined first-token prefill: each stage runs its layers as they become ready,
//                          hands the fp32 residual to the next stage (peer copy + readiness word),
//                          vocab-parallel logits, argmax on rank 0, token D2H
// Cross-rank dependencies are device-side (readiness words compared with the trial epoch), so the host
// threads / processes of different ranks never wait for each other inside a trial.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <deque>
#include <mutex>
#include <set>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX ranges (visible to Nsight Systems when one is attached)

#include "errors.hpp"
#include "runtime.hpp"

namespace {
// NVTX range for the calling host thread (the issuer's trial, a copy group, a layer's launches, a blocking wait).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    NvtxRange(const char* fmt, int a, int b) {
        char buf[96];
        snprintf(buf, sizeof buf, fmt, a, b);
        nvtxRangePushA(buf);
    }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace pb;

#define CU(call)                                                                                         \
    do {                                                                                                 \
        cudaError_t e_ = (call);                                                                         \
        if (e_ != cudaSuccess) return fail(PB_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
    } while (0)

namespace {

int64_t al(int64_t x, int64_t a = 256) { return (x + a - 1) / a * a; }

int32_t qkv_dim(const pb_plan* p) { return (p->model.n_heads + 2 * p->model.n_kv_heads) * p->head_dim(); }

// Head tensor: tied OPT -> embed, otherwise lm_head.
int32_t head_tensor(const pb_plan* p) {
    return p->model.arch == PB_ARCH_OPT && p->model.tied ? p->find_tensor("embed") : p->find_tensor("lm_head");
}

bool is_head_owner(const pb_plan* p, int32_t g) {
    const int32_t ht = head_tensor(p);
    for (auto& c : p->chunks)
        if (!c.is_adapter && c.tensor == ht && c.loader == g) return true;
    return false;
}

// Vocab rows [v0, v1) of the head this rank owns (contiguous by construction).
void head_slice(const pb_plan* p, int32_t g, int32_t* v0, int32_t* v1) {
    const int32_t ht = head_tensor(p);
    *v0 = INT32_MAX;
    *v1 = -1;
    for (auto& c : p->chunks)
        if (!c.is_adapter && c.tensor == ht && c.loader == g) {
            *v0 = std::min(*v0, c.r0);
            *v1 = std::max(*v1, c.r1);
        }
    if (*v1 < 0) *v0 = *v1 = 0;
}

void join_load(pb_ctx* c) {
    if (c->load_thread.joinable()) c->load_thread.join();
}

pb_status check_ctx(pb_ctx* c, const char* fn) {
    if (!c) return fail(PB_EINVAL, "%s: null ctx", fn);
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(PB_ECUDA, "%s: cudaSetDevice: %s", fn, cudaGetErrorString(e));
    if (c->aborted && strcmp(fn, "pb_timeline") != 0 && strcmp(fn, "pb_ctx_abort") != 0)
        return fail(PB_EPROTOCOL, "%s: the ctx was aborted (pb_ctx_abort); only pb_ctx_free remains", fn);
    return PB_OK;
}

struct IpcBlob {
    uint32_t magic;
    int32_t rank;
    int32_t device;
    int32_t pid;
    cudaIpcMemHandle_t wh, sh;
    int64_t w_off, s_off;
};
constexpr uint32_t kMagic = 0x50424950;  // "PBIP"

}  // namespace

// Process-wide pool of idle ctx-owned streams per device. CUDA maps streams onto CUDA_DEVICE_MAX_CONNECTIONS
// hardware queues round-robin in creation order, so a process that keeps creating contexts (tests, several
// logical ranks on one GPU) eventually puts two ranks' streams on one queue, where a device-side readiness wait
// can block the very work that satisfies it. Reusing handles keeps the set of queues fixed.
namespace {
std::mutex g_stream_mu;
std::vector<std::pair<int, cudaStream_t>> g_stream_pool;
cudaError_t stream_take(int dev, cudaStream_t* s) {
    {
        std::lock_guard<std::mutex> lk(g_stream_mu);
        for (size_t i = 0; i < g_stream_pool.size(); ++i)
            if (g_stream_pool[i].first == dev) {
                *s = g_stream_pool[i].second;
                g_stream_pool.erase(g_stream_pool.begin() + (long)i);
                return cudaSuccess;
            }
    }
    return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
}
void stream_give(int dev, cudaStream_t s) {
    if (cudaStreamQuery(s) != cudaSuccess) {   // still busy (a failed trial): never hand it to another ctx
        cudaStreamDestroy(s);
        return;
    }
    std::lock_guard<std::mutex> lk(g_stream_mu);
    g_stream_pool.emplace_back(dev, s);
}
}  // namespace

WsLayout pb::ws_layout(const pb_plan* p, int32_t batch, int32_t seq) {
    WsLayout L;
    const auto& m = p->model;
    const int64_t rows = (int64_t)batch * seq;
    const int64_t d = m.d_model, hd = p->head_dim(), qd = (int64_t)m.n_heads * hd, f = m.d_ffn;
    const int k = std::max(1, p->opts.prefill_chunks);
    L.max_rows = (int32_t)rows;
    L.max_batch = batch;
    L.max_seq = seq;
    L.f_chunk = 0;
    L.f_act = (int32_t)p->chunks.size();
    L.f_y = L.f_act + k * batch;   // one activation word per (microbatch, prompt chunk)
    L.f_logit = L.f_y + 1;
    L.f_land = L.f_logit + p->n_gpus;
    L.f_tensor = L.f_land + (int32_t)p->chunks.size();
    L.f_tensor_recv = L.f_tensor + (int32_t)p->tensors.size();
    L.f_gdone = L.f_tensor_recv + (int32_t)p->tensors.size();
    L.n_words = L.f_gdone + p->n_gpus;
    int64_t o = 0;
    L.flags = o;   o = al(o + 4 * (int64_t)L.n_words);
    L.tokens = o;  o = al(o + 4 * rows);
    L.h = o;       o = al(o + 4 * rows * d);
    const int64_t ea = p->es();   // activation element size: bf16 (product path) or fp32 (debug-parity path)
    L.x = o;       o = al(o + ea * rows * d);
    // one q|k|v slot per layer: prompt chunks and decode steps read the K/V of earlier positions (the KV cache),
    // and a replica (f3) runs every layer
    L.n_qkv = m.n_layers;
    (void)k;
    L.qkv_stride = al(ea * rows * qkv_dim(p));
    L.qkv = o;     o += L.qkv_stride * L.n_qkv;
    L.attn = o;    o = al(o + ea * rows * qd);
    L.mlp = o;     o = al(o + ea * rows * f);
    L.y = o;       o = al(o + ea * (int64_t)batch * d);
    L.logits = o;  o = al(o + 4 * (int64_t)batch * m.vocab);
    L.tok_out = o; o = al(o + 4 * (int64_t)batch);
    L.nan = o;     o = al(o + 4);
    L.rope = o;    o = al(o + (m.arch == PB_ARCH_LLAMA ? 8 * (int64_t)seq * (hd / 2) : 0));
    L.held = o;    o = al(o + (p->survivors.empty() ? 0 : 4 * (int64_t)p->chunks.size()));   // re-plan signal list
    L.dpos = o;    o = al(o + 4);   // f3 decode graphs: the step's position
    L.total = al(o, 4096);
    return L;
}

extern "C" pb_status pb_plan_workspace_bytes(const pb_plan* p, int32_t batch, int32_t seq, int64_t* out) {
    if (!p || !out) return fail(PB_EINVAL, "pb_plan_workspace_bytes: null argument");
    if (batch < 1 || batch > kMaxBatch || seq < 1) return fail(PB_EINVAL, "batch must be in [1, %d] and seq >= 1", kMaxBatch);
    if (p->model.arch == PB_ARCH_OPT && seq > p->model.max_pos) return fail(PB_EINVAL, "seq > max_pos");
    *out = ws_layout(p, batch, seq).total;
    return PB_OK;
}

// ------------------------------------------------------------------------------------------------
// context creation
// ------------------------------------------------------------------------------------------------

static pb_status build_merge_jobs(pb_ctx* c) {
    const pb_plan* p = c->plan;
    c->jobs_of_chunk.assign(p->chunks.size(), {});
    char err[512];
    const size_t NT = p->tensors.size();
    // adapter chunks of each atensor
    std::vector<std::vector<int32_t>> achunks(p->atensors.size());
    for (auto& ch : p->chunks)
        if (ch.is_adapter) achunks[ch.tensor].push_back(ch.id);
    for (auto& mr : p->merges) {
        const auto& bt = p->tensors[mr.base];
        const auto& A = p->atensors[mr.a_tensor];
        const auto& Bf = p->atensors[mr.b_tensor];
        const int rank = p->adapters[mr.adapter].rank;
        for (auto& ch : p->chunks) {
            if (ch.is_adapter || ch.tensor != mr.base || ch.loader != c->rank || p->is_resident(c->rank, ch.id)) continue;
            const int32_t ra = std::max(ch.r0, mr.row0), rb = std::min(ch.r1, mr.row0 + mr.rows);
            if (rb <= ra) continue;
            if (rank % 8 != 0 && !p->f32())
                return fail(PB_EUNSUPPORTED, "merge needs rank %% 8 == 0 (TMA 16-byte row pitch), got %d", rank);
            for (int inplace = 1; inplace >= 0; --inplace) {
                if (!inplace && !c->adapted) continue;
                MergeJob j;
                j.chunk = ch.id;
                j.adapter = mr.adapter;
                j.inplace = inplace != 0;
                j.rows = rb - ra;
                j.cols = mr.cols;
                j.rank = rank;
                j.scale = p->adapters[mr.adapter].alpha / (float)rank;
                // factor chunks this rank already holds (a re-plan's resident set) have nothing to wait for
                for (const auto* v : {&achunks[mr.a_tensor], &achunks[mr.b_tensor]})
                    for (int32_t a : *v)
                        if (!p->is_resident(c->rank, a)) j.need.push_back(a);
                char* W = c->weights + bt.dev_off + (int64_t)ra * bt.row_bytes();
                char* Wout = inplace ? W
                                     : c->adapted + p->adapted_off[mr.adapter * NT + mr.base] +
                                           (int64_t)ra * bt.row_bytes();
                const char* Bp = c->adapters + Bf.off + (int64_t)(ra - mr.row0) * Bf.row_bytes();
                const char* Ap = c->adapters + A.off;
                if (p->f32()) {
                    j.W = reinterpret_cast<const float*>(W);
                    j.Wout = reinterpret_cast<float*>(Wout);
                    j.Bp = reinterpret_cast<const float*>(Bp);
                    j.Ap = reinterpret_cast<const float*>(Ap);
                    j.ldw = bt.cols;
                } else if (!make_merge_maps(&j.maps, W, bt.cols, j.rows, j.cols, Bp, Ap, rank, err, sizeof err,
                                            Wout)) {
                    return fail(PB_EINVAL, "merge map: %s", err);
                }
                c->jobs_of_chunk[ch.id].push_back((int32_t)c->jobs.size());
                c->jobs.push_back(j);
            }
        }
    }
    return PB_OK;
}

// Coalesce the load list into DMA groups: a chunk joins the current group when it continues it in both
// address spaces with the same (< 4 KiB alignment) gap, and either the group stays within chunk_bytes or
// the chunk is small (biases / norms). Fewer, larger copies keep the copy engine at link speed.
// Within the last 2 x chunk_bytes of the load the groups are capped at 32 MB: what lands last is all that is
// left to compute after the link goes idle, so the final layers start as their own tensors arrive (measured
// per-group cost without timing events ~5 us).
static void build_copy_groups(pb_ctx* c) {
    const pb_plan* p = c->plan;
    const auto& ld = p->load[c->rank];
    const int64_t cap_main = p->opts.chunk_bytes, small = 256 << 10;
    const int64_t cap_tail = std::min<int64_t>(cap_main, 32 << 20);
    int64_t total = 0, before = 0;
    for (int32_t id : ld) total += p->chunks[id].bytes;
    c->copies.clear();
    for (int32_t i = 0; i < (int32_t)ld.size(); ++i) {
        const ChunkRec& ch = p->chunks[ld[i]];
        const int64_t cap = total - before <= 2 * cap_main ? cap_tail : cap_main;
        before += ch.bytes;
        const char* hbase = static_cast<const char*>(ch.is_adapter ? c->host_adapters : c->host_base);
        char* dbase = ch.is_adapter ? c->adapters : c->weights;
        const char* src = hbase + ch.host_off;
        char* dst = dbase + ch.dev_off;
        if (!c->copies.empty()) {
            CopyGroup& g = c->copies.back();
            const ChunkRec& prev = p->chunks[ld[g.first + g.count - 1]];
            const int64_t hgap = src - (g.src + g.bytes), dgap = dst - (g.dst + g.bytes);
            if (prev.is_adapter == ch.is_adapter && hgap == dgap && hgap >= 0 && hgap < kAlign &&
                (g.bytes + hgap + ch.bytes <= cap || ch.bytes < small)) {
                g.bytes += hgap + ch.bytes;
                g.count++;
                continue;
            }
        }
        c->copies.push_back(CopyGroup{src, dst, ch.bytes, i, 1, false});
    }
    c->landed_alias.assign(p->chunks.size(), -1);
    for (const CopyGroup& g : c->copies)
        for (int32_t i = g.first; i < g.first + g.count; ++i) c->landed_alias[ld[i]] = ld[g.first];
}

static cudaEvent_t landed_ev(pb_ctx* c, int32_t chunk) { return c->landed[c->landed_alias[chunk]]; }

static pb_status build_prefill_maps(pb_ctx* c) {
    const pb_plan* p = c->plan;
    if (p->f32()) return PB_OK;   // the fp32 path's SIMT kernels take plain pointers
    const auto& m = p->model;
    const int64_t d = m.d_model, qd = (int64_t)m.n_heads * p->head_dim(), f = m.d_ffn;
    const int64_t R = c->L.max_rows;
    char err[512];
    if (!make_map_bf16(&c->map_x, c->ws + c->L.x, R, d, d, 128, 64, 128, err, sizeof err) ||
        !make_map_bf16(&c->map_attn, c->ws + c->L.attn, R, qd, qd, 128, 64, 128, err, sizeof err) ||
        !make_map_bf16(&c->map_mlp, c->ws + c->L.mlp, R, f, f, 128, 64, 128, err, sizeof err))
        return fail(PB_EINVAL, "activation map: %s", err);
    const bool opt = m.arch == PB_ARCH_OPT;
    const size_t NT = p->tensors.size();
    const int A = c->adapted ? (int)p->adapters.size() : 0;
    c->lmaps.assign(m.n_layers, LayerMaps{});
    c->lmaps_ad.assign(A, std::vector<LayerMaps>(m.n_layers, LayerMaps{}));
    // every layer, not only this rank's stage: a replica (f3, after T_full) runs the whole model
    for (int l = 0; l < m.n_layers; ++l) {
        auto tid = [&](const char* s) { return p->find_tensor("L" + std::to_string(l) + "." + s); };
        const int32_t ids[4] = {tid("qkv"), tid("o"), tid(opt ? "fc1" : "gate_up"), tid(opt ? "fc2" : "down")};
        // adapter -1: base weights; a >= 0: adapter a's out-of-place copy where it has one, else the base
        for (int a = -1; a < A; ++a) {
            LayerMaps& lm = a < 0 ? c->lmaps[l] : c->lmaps_ad[a][l];
            CUtensorMap* maps[4] = {&lm.qkv, &lm.o, &lm.up, &lm.down};
            for (int i = 0; i < 4; ++i) {
                const TensorRec& t = p->tensors[ids[i]];
                const int64_t off = a >= 0 ? p->adapted_off[a * NT + ids[i]] : -1;
                const char* base = off >= 0 ? c->adapted + off : c->weights + t.dev_off;
                const uint32_t box_rows = (i == 2 && !opt) ? 64 : 128;   // [gate; up] is read as 64 + 64 rows
                if (!make_map_bf16(maps[i], base, t.rows, t.cols, t.cols, box_rows, 64, 128, err, sizeof err))
                    return fail(PB_EINVAL, "weight map layer %d: %s", l, err);
                lm.w[i] = reinterpret_cast<const __nv_bfloat16*>(base);
                if (!(i == 2 && !opt) &&
                    (!make_map_bf16(&lm.w64[i], base, t.rows, t.cols, t.cols, 64, 64, 128, err, sizeof err) ||
                     !make_map_bf16(&lm.w32[i], base, t.rows, t.cols, t.cols, 32, 64, 128, err, sizeof err)))
                    return fail(PB_EINVAL, "weight map layer %d: %s", l, err);
            }
        }
    }
    return PB_OK;
}

extern "C" pb_status pb_ctx_create(const pb_plan* plan, int32_t rank, const void* host_base, const void* host_adapters,
                                   const pb_rank_bufs* bufs, pb_ctx** out) {
    PB_TRY_BEGIN
    const auto t_create = std::chrono::steady_clock::now();
    if (!plan || !host_base || !bufs || !out) return fail(PB_EINVAL, "pb_ctx_create: null argument");
    *out = nullptr;
    if (rank < 0 || rank >= plan->n_gpus) return fail(PB_EINVAL, "rank %d out of [0, %d)", rank, plan->n_gpus);
    if (!bufs->weights || bufs->weights_cap < plan->dev_weight_bytes)
        return fail(PB_ENOMEM, "weights buffer: need %lld bytes", (long long)plan->dev_weight_bytes);
    if (!plan->adapters.empty() && (!bufs->adapters || bufs->adapters_cap < plan->host_adapter_bytes || !host_adapters))
        return fail(PB_ENOMEM, "adapters buffer: need %lld bytes (and a host image)", (long long)plan->host_adapter_bytes);
    if (bufs->max_batch < 1 || bufs->max_batch > kMaxBatch || bufs->max_seq < 1)
        return fail(PB_EINVAL, "max_batch must be in [1, %d], max_seq >= 1", kMaxBatch);
    if (plan->model.arch == PB_ARCH_OPT && bufs->max_seq > plan->model.max_pos)
        return fail(PB_EINVAL, "max_seq %d > max_pos %d", bufs->max_seq, plan->model.max_pos);
    const int hd = plan->head_dim();
    if (hd != 32 && hd != 64 && hd != 128) return fail(PB_EUNSUPPORTED, "head_dim %d (supported: 32, 64, 128)", hd);
    if (plan->model.d_model % 64 || plan->model.d_ffn % 8 || plan->model.d_model > 256 * 40)
        return fail(PB_EUNSUPPORTED, "d_model must be a multiple of 64 (<= 10240), d_ffn of 8");
    WsLayout L = ws_layout(plan, bufs->max_batch, bufs->max_seq);
    if (!bufs->workspace || bufs->workspace_cap < L.total)
        return fail(PB_ENOMEM, "workspace: need %lld bytes", (long long)L.total);
    char err[256];
    if (!driver_init(err, sizeof err)) return fail(PB_ECUDA, "%s", err);
    {
        static std::mutex warm_mu;
        static std::set<int> warmed;
        std::lock_guard<std::mutex> lk(warm_mu);
        int dev = 0;
        cudaGetDevice(&dev);
        if (!warmed.count(dev)) {
            cudaError_t e = warm_merge_kernels();
            if (e == cudaSuccess) e = warm_gemm_kernels();
            if (e == cudaSuccess) e = warm_simt_kernels();
            if (e == cudaSuccess) e = warm_attention_kernels();
            if (e == cudaSuccess) e = warm_f32_kernels();
            if (e != cudaSuccess) return fail(PB_ECUDA, "kernel load: %s", cudaGetErrorString(e));
            warmed.insert(dev);
        }
    }

    auto* c = new pb_ctx();
    c->plan = plan;
    c->rank = rank;
    c->n = plan->n_gpus;
    cudaGetDevice(&c->device);
    c->weights = static_cast<char*>(bufs->weights);
    c->adapters = static_cast<char*>(bufs->adapters);
    c->ws = static_cast<char*>(bufs->workspace);
    if (plan->adapters.size() > 0 && bufs->adapted && bufs->adapted_cap >= plan->dev_adapted_bytes &&
        plan->dev_adapted_bytes > 0)
        c->adapted = static_cast<char*>(bufs->adapted);
    if (plan->dev_backup_bytes > 0 && bufs->backup && bufs->backup_cap >= plan->dev_backup_bytes)
        c->backup = static_cast<char*>(bufs->backup);
    c->in_load.assign(plan->chunks.size(), 0);
    for (int32_t id : plan->load[rank]) c->in_load[id] = 1;
    c->bufs = *bufs;
    c->h2d[0] = (cudaStream_t)bufs->stream_h2d[0];
    c->h2d[1] = (cudaStream_t)bufs->stream_h2d[1];
    c->merge = (cudaStream_t)bufs->stream_merge;
    c->nv = (cudaStream_t)bufs->stream_nvlink;
    c->comp = (cudaStream_t)bufs->stream_compute;
    // NULL streams: the ctx creates its own (distinct, non-blocking). Each rank needs five DISTINCT streams:
    // device-side readiness waits on a stream shared with another rank's producer would deadlock.
    cudaStream_t* mine[5] = {&c->h2d[0], &c->h2d[1], &c->merge, &c->nv, &c->comp};
    for (auto* sp : mine)
        if (!*sp) {
            if (stream_take(c->device, sp) != cudaSuccess) {
                for (auto* q : mine)
                    if (*q && q != sp) { /* owned ones are released by pb_ctx_free below */ }
                return fail(PB_ECUDA, "cudaStreamCreateWithFlags failed");
            }
            c->owned_streams.push_back(*sp);
        }
    c->L = L;
    c->host_base = host_base;
    c->host_adapters = host_adapters;
    c->peers.assign(c->n, Peer{});
    c->peers[rank].weights = c->weights;
    c->peers[rank].ws = c->ws;
    c->peers[rank].linked = true;

    auto cleanup = [&](pb_status st) { pb_ctx_free(c); return st; };
    const size_t NC = plan->chunks.size(), NT = plan->tensors.size();
    c->landed.assign(NC, nullptr);
    c->gathered.assign(NC, nullptr);
    c->tl_landed.assign(NC, -1.0);
    c->tl_gathered.assign(NC, -1.0);
    c->tl_merged.assign(NC, -1.0);
    c->merged_ev.assign(NC, nullptr);
    // Events only where the timeline needs a timestamp (measured on B200: a timing-event record costs
    // ~20 us while the PCIe link is saturated by the load); dependencies are device-side readiness words.
    auto mk = [&](cudaEvent_t* e) { return cudaEventCreate(e); };
    if (mk(&c->t0) || mk(&c->merge_done) || mk(&c->gather_done) || mk(&c->done) || mk(&c->ready_merge) ||
        mk(&c->ready_recv) || mk(&c->stage_begin) || mk(&c->stage_end) ||
        cudaEventCreateWithFlags(&c->tok_ev, cudaEventDisableTiming))
        return cleanup(fail(PB_ECUDA, "cudaEventCreate failed"));
    for (auto& e : c->trial_fence)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) return cleanup(fail(PB_ECUDA, "cudaEventCreate failed"));
    if (const char* lt = getenv("PB_LANDED_TIMING")) c->landed_timing = atoi(lt) != 0;
    if (mk(&c->load_end)) return cleanup(fail(PB_ECUDA, "cudaEventCreate failed"));
    for (int32_t id : plan->load[rank]) {
        if (c->landed_timing ? mk(&c->landed[id]) : cudaEventCreateWithFlags(&c->landed[id], cudaEventDisableTiming))
            return cleanup(fail(PB_ECUDA, "cudaEventCreate failed"));
        if (c->landed_timing && !plan->chunks[id].is_adapter && mk(&c->merged_ev[id]))
            return cleanup(fail(PB_ECUDA, "cudaEventCreate failed"));
    }
    c->budget_events.assign(4 * kEventPool, nullptr);
    for (auto& e : c->budget_events)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) return cleanup(fail(PB_ECUDA, "cudaEventCreate failed"));
    for (int32_t id : plan->recv[rank])
        if (mk(&c->gathered[id])) return cleanup(fail(PB_ECUDA, "cudaEventCreate failed"));
    // per-tensor last own / received chunk
    c->last_own_chunk.assign(NT, -1);
    c->last_recv_chunk.assign(NT, -1);
    for (int32_t id : plan->load[rank])
        if (!plan->chunks[id].is_adapter) c->last_own_chunk[plan->chunks[id].tensor] = id;
    for (int32_t id : plan->recv[rank]) c->last_recv_chunk[plan->chunks[id].tensor] = id;
    {
        const auto st = plan->stages[rank];
        auto in_stage = [&](int32_t id) {
            const auto& ch = plan->chunks[id];
            const int32_t l = ch.is_adapter ? -1 : plan->tensors[ch.tensor].layer;
            return l >= st.first && l < st.second;
        };
        for (int32_t id : plan->load[rank])
            if (in_stage(id)) c->last_own_stage_chunk = id;
        for (int32_t id : plan->recv[rank])
            if (in_stage(id)) c->last_recv_stage_chunk = id;
    }

    if (!plan->survivors.empty()) {   // re-plan: chunks this rank holds that other ranks will copy from it
        std::vector<int32_t> held;
        for (const ChunkRec& ch : plan->chunks)
            if (!ch.is_adapter && ch.loader == rank && plan->is_resident(rank, ch.id)) held.push_back(ch.id);
        c->n_held_src = (int32_t)held.size();
        if (!held.empty() &&
            cudaMemcpy(c->ws + L.held, held.data(), 4 * held.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            return cleanup(fail(PB_ECUDA, "held-chunk list upload failed"));
    }
    build_copy_groups(c);
    pb_status st = build_merge_jobs(c);
    if (st != PB_OK) return cleanup(st);
    st = build_prefill_maps(c);
    if (st != PB_OK) return cleanup(st);
    if (cudaHostAlloc((void**)&c->h_pos, sizeof(int32_t), cudaHostAllocPortable) != cudaSuccess ||
        cudaHostAlloc((void**)&c->h_tokens, sizeof(int32_t) * L.max_rows, cudaHostAllocPortable) != cudaSuccess ||
        cudaHostAlloc((void**)&c->h_out, sizeof(int32_t) * (L.max_batch + 1), cudaHostAllocPortable) != cudaSuccess)
        return cleanup(fail(PB_ECUDA, "cudaHostAlloc failed"));
    // readiness words start at 0 (epochs are >= 1); the q|k|v slots start at 0 so a key row no step has written
    // yet is finite (decode graphs view keys up to max_seq and mask the later ones)
    if (cudaMemset(c->ws + L.flags, 0, 4 * (size_t)L.n_words) != cudaSuccess ||
        cudaMemset(c->ws + L.qkv, 0, (size_t)L.qkv_stride * L.n_qkv) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
        return cleanup(fail(PB_ECUDA, "flag init failed"));
    c->ctx_create_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_create).count();
    *out = c;
    return PB_OK;
    PB_TRY_END
}

// Wait (polling, at most `seconds`) for a stream to drain; false if it did not.
static bool drain_stream(cudaStream_t s, double seconds) {
    const auto t = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q != cudaErrorNotReady) { cudaGetLastError(); return true; }
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count() > seconds) return false;
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

extern "C" void pb_ctx_free(pb_ctx* c) {
    if (!c) return;
    c->abort_req.store(c->aborted);
    join_load(c);
    cudaSetDevice(c->device);
    if (c->aborted) {
        // after pb_ctx_abort the streams drain on their own (readiness words forced open); a stream that does not
        // drain in time is leaked rather than handed to the next context (it may still run this trial's work)
        std::vector<cudaStream_t> keep;
        for (auto st : c->owned_streams)
            if (drain_stream(st, 5.0)) keep.push_back(st);
        c->owned_streams.swap(keep);
    } else {
        cudaDeviceSynchronize();
    }
    auto d = [](cudaEvent_t e) { if (e) cudaEventDestroy(e); };
    d(c->t0); d(c->merge_done); d(c->gather_done); d(c->done); d(c->ready_merge); d(c->ready_recv); d(c->tok_ev);
    for (auto e : c->trial_fence) d(e);
    d(c->load_end); d(c->stage_begin); d(c->stage_end);
    for (auto e : c->merged_ev) d(e);
    for (auto e : c->budget_events) d(e);
    for (auto st : c->owned_streams) stream_give(c->device, st);
    for (auto e : c->landed) d(e);
    for (auto e : c->gathered) d(e);
    for (auto& r : c->prof) { d(r.a); d(r.b); }
    for (auto& g : c->replay_graphs) cudaGraphExecDestroy(g.exec);
    for (auto& g : c->decode_graphs) cudaGraphExecDestroy(g.exec);
    if (c->h_pos) cudaFreeHost(c->h_pos);
    for (auto& p : c->peers)
        for (void* b : p.ipc_bases) cudaIpcCloseMemHandle(b);
    if (c->h_tokens) cudaFreeHost(c->h_tokens);
    if (c->h_out) cudaFreeHost(c->h_out);
    delete c;
}

// ------------------------------------------------------------------------------------------------
// cross-rank wiring
// ------------------------------------------------------------------------------------------------

extern "C" pb_status pb_ctx_export(pb_ctx* c, void* blob, size_t cap, size_t* needed) {
    pb_status st = check_ctx(c, "pb_ctx_export");
    if (st) return st;
    if (!needed) return fail(PB_EINVAL, "pb_ctx_export: null needed");
    *needed = sizeof(IpcBlob);
    if (!blob || cap < sizeof(IpcBlob)) return fail(PB_ENOMEM, "pb_ctx_export: need %zu bytes", sizeof(IpcBlob));
    IpcBlob b{};
    b.magic = kMagic;
    b.rank = c->rank;
    b.device = c->device;
    b.pid = (int32_t)getpid();
    void* base = nullptr;
    size_t size = 0;
    CU(cudaIpcGetMemHandle(&b.wh, c->weights));
    {
        CUdeviceptr bp;
        size_t sz;
        // offset of our pointer inside its allocation
        using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static GetRange fn = nullptr;
        if (!fn) {
            cudaDriverEntryPointQueryResult q;
            cudaGetDriverEntryPoint("cuMemGetAddressRange", (void**)&fn, cudaEnableDefault, &q);
        }
        if (!fn) return fail(PB_ECUDA, "cuMemGetAddressRange unavailable");
        if (fn(&bp, &sz, (CUdeviceptr)c->weights) != CUDA_SUCCESS) return fail(PB_ECUDA, "cuMemGetAddressRange(weights)");
        b.w_off = (int64_t)((CUdeviceptr)c->weights - bp);
        if (fn(&bp, &sz, (CUdeviceptr)c->ws) != CUDA_SUCCESS) return fail(PB_ECUDA, "cuMemGetAddressRange(ws)");
        b.s_off = (int64_t)((CUdeviceptr)c->ws - bp);
    }
    (void)base;
    (void)size;
    CU(cudaIpcGetMemHandle(&b.sh, c->ws));
    memcpy(blob, &b, sizeof b);
    return PB_OK;
}

extern "C" pb_status pb_ctx_import_peer(pb_ctx* c, int32_t peer, const void* blob, size_t len) {
    pb_status st = check_ctx(c, "pb_ctx_import_peer");
    if (st) return st;
    if (!blob || len < sizeof(IpcBlob)) return fail(PB_EINVAL, "pb_ctx_import_peer: bad blob");
    if (peer < 0 || peer >= c->n || peer == c->rank) return fail(PB_EINVAL, "bad peer %d", peer);
    IpcBlob b;
    memcpy(&b, blob, sizeof b);
    if (b.magic != kMagic || b.rank != peer) return fail(PB_EINVAL, "blob is not rank %d's", peer);
    Peer& P = c->peers[peer];
    void* wb = nullptr;
    CU(cudaIpcOpenMemHandle(&wb, b.wh, cudaIpcMemLazyEnablePeerAccess));
    P.ipc_bases.push_back(wb);
    void* sb = nullptr;
    if (memcmp(&b.wh, &b.sh, sizeof b.wh) == 0) {
        sb = wb;   // same allocation
    } else {
        CU(cudaIpcOpenMemHandle(&sb, b.sh, cudaIpcMemLazyEnablePeerAccess));
        P.ipc_bases.push_back(sb);
    }
    P.weights = static_cast<char*>(wb) + b.w_off;
    P.ws = static_cast<char*>(sb) + b.s_off;
    P.linked = true;
    return PB_OK;
}

extern "C" pb_status pb_ctx_link_local(pb_ctx* c, int32_t peer, pb_ctx* pc) {
    pb_status st = check_ctx(c, "pb_ctx_link_local");
    if (st) return st;
    if (!pc || peer < 0 || peer >= c->n || peer == c->rank || pc->rank != peer || pc->plan->n_gpus != c->n)
        return fail(PB_EINVAL, "pb_ctx_link_local: bad peer");
    if (pc->device != c->device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(pc->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return fail(PB_ECUDA, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
        cudaGetLastError();
    }
    c->peers[peer].weights = pc->weights;
    c->peers[peer].ws = pc->ws;
    c->peers[peer].linked = true;
    return PB_OK;
}

// ------------------------------------------------------------------------------------------------
// trial
// ------------------------------------------------------------------------------------------------

static uint32_t* flag_ptr(char* ws, const WsLayout& L, int32_t word) {
    return reinterpret_cast<uint32_t*>(ws + L.flags) + word;
}

// Record an event observed outside the work (timeline, profiling): while the replay is being captured into a
// CUDA graph it must become an event-record node (cudaEventRecordExternal), not a capture-internal dependency.
static cudaError_t record_ev(pb_ctx* c, cudaEvent_t e, cudaStream_t s) {
    return c->capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
}

static int prof_begin(pb_ctx* c, int cls, cudaStream_t s) {
    if (!c->profiling) return -1;
    if (c->prof_n == c->prof.size()) {
        ProfRec r{};
        if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return -1;
        c->prof.push_back(r);
    }
    ProfRec& r = c->prof[c->prof_n];
    r.cls = cls;
    r.flops = r.bytes = 0;
    if (record_ev(c, r.a, s) != cudaSuccess) return -1;
    return (int)c->prof_n++;
}

static void prof_end(pb_ctx* c, int i, cudaStream_t s, double flops, double bytes) {
    if (i < 0) return;
    ProfRec& r = c->prof[i];
    r.flops = flops;
    r.bytes = bytes;
    record_ev(c, r.b, s);
}

// Publish readiness word `word` (= epoch) on the given ranks.
static cudaError_t signal_ranks(pb_ctx* c, int32_t word, const std::vector<int32_t>& ranks, cudaStream_t s) {
    SignalTargets t{};
    for (int32_t r : ranks) t.addr[t.n++] = flag_ptr(c->peers[r].ws, c->L, word);
    if (t.n == 0) return cudaSuccess;
    ++c->n_launches;
    const int pi = prof_begin(c, K_SIGNAL, s);
    cudaError_t e = launch_signal(t, c->epoch, s);
    prof_end(c, pi, s, 0, 4.0 * t.n);
    return e;
}

static cudaError_t wait_word(pb_ctx* c, int32_t word, cudaStream_t s) {
    return stream_wait_geq(s, flag_ptr(c->ws, c->L, word), c->epoch);
}

// Local readiness word: written by the producing stream after its prior work, so consumers can be
// enqueued in any host order (the load is enqueued from a worker thread that may block on a full queue).
static cudaError_t set_word(pb_ctx* c, int32_t word, cudaStream_t s) {
    return stream_write(s, flag_ptr(c->ws, c->L, word), c->epoch);
}


extern "C" pb_status pb_ctx_set_profiling(pb_ctx* c, int32_t enable) {
    pb_status st = check_ctx(c, "pb_ctx_set_profiling");
    if (st) return st;
    c->profiling = enable != 0;
    return PB_OK;
}

extern "C" pb_status pb_kernel_stats(pb_ctx* c, pb_kernel_stat* out, int32_t cap, int32_t* n) {
    pb_status st = check_ctx(c, "pb_kernel_stats");
    if (st) return st;
    if (!n) return fail(PB_EINVAL, "pb_kernel_stats: null n");
    static const char* names[K_NCLASS] = {"merge", "gemm", "attention", "norm", "rope", "embed", "logits", "argmax", "signal"};
    pb_kernel_stat agg[K_NCLASS];
    for (int k = 0; k < K_NCLASS; ++k) agg[k] = {names[k], 0, 0.0, 0.0, 0.0};
    for (size_t i = 0; i < c->prof_n; ++i) {
        const ProfRec& r = c->prof[i];
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, r.a, r.b));
        pb_kernel_stat& a = agg[r.cls];
        a.launches++;
        a.total_ms += ms;
        a.flops += r.flops;
        a.bytes += r.bytes;
    }
    *n = K_NCLASS;
    if (!out || cap < K_NCLASS) return fail(PB_ENOMEM, "pb_kernel_stats: need %d entries", (int)K_NCLASS);
    for (int k = 0; k < K_NCLASS; ++k) out[k] = agg[k];
    return PB_OK;
}

extern "C" pb_status pb_kernel_trace(pb_ctx* c, pb_kernel_event* out, int32_t cap, int32_t* n) {
    pb_status st = check_ctx(c, "pb_kernel_trace");
    if (st) return st;
    if (!n) return fail(PB_EINVAL, "pb_kernel_trace: null n");
    *n = (int32_t)c->prof_n;
    for (size_t i = 0; i < c->prof_n && out && (int32_t)i < cap; ++i) {
        const ProfRec& r = c->prof[i];
        out[i].cls = r.cls;
        CU(cudaEventElapsedTime(&out[i].start_ms, c->t0, r.a));
        CU(cudaEventElapsedTime(&out[i].end_ms, c->t0, r.b));
    }
    return PB_OK;
}

static pb_status start_load_issuer(pb_ctx* c);

extern "C" pb_status pb_trial_begin(pb_ctx* c, uint32_t epoch) {
    pb_status st = check_ctx(c, "pb_trial_begin");
    if (st) return st;
    if (c->aborted) return fail(PB_EPROTOCOL, "pb_trial_begin: the ctx was aborted (pb_ctx_free it)");
    if (epoch <= c->epoch) return fail(PB_EINVAL, "epoch %u must exceed the previous %u", epoch, c->epoch);
    join_load(c);
    c->run.reset();
    c->posted.store(false);
    for (int r = 0; r < c->n; ++r)
        if (!c->peers[r].linked) return fail(PB_EPROTOCOL, "peer %d not wired (import/link)", r);
    c->epoch = epoch;
    c->cold_epoch = epoch;
    c->n_launches = 0;
    c->prof_n = 0;
    c->load_bytes = c->recv_bytes = 0;
    std::fill(c->tl_landed.begin(), c->tl_landed.end(), -1.0);
    std::fill(c->tl_gathered.begin(), c->tl_gathered.end(), -1.0);
    // Every stream of the previous trial drains before this one starts: a trial armed and then left without a
    // prompt (a refused pb_prefill_enqueue) keeps loading / merging; its in-place merges must not run after this
    // trial's copies of the same bytes.
    cudaStream_t others[] = {c->h2d[1], c->merge, c->nv, c->comp};
    for (int i = 0; i < 4; ++i) {
        CU(cudaEventRecord(c->trial_fence[i], others[i]));
        CU(cudaStreamWaitEvent(c->h2d[0], c->trial_fence[i], 0));
    }
    CU(cudaEventRecord(c->t0, c->h2d[0]));
    for (auto s : others) CU(cudaStreamWaitEvent(s, c->t0, 0));
    // re-plan resume: chunks this rank already holds are ready for the peers that receive them from it
    for (int r = 0; r < c->n && c->n_held_src > 0; ++r)
        if (r != c->rank)
            CU(launch_set_words(flag_ptr(c->peers[r].ws, c->L, c->L.f_chunk),
                                reinterpret_cast<const int32_t*>(c->ws + c->L.held), c->n_held_src, epoch, c->merge));
    c->phase = Phase::Begun;
    return PB_OK;
}

extern "C" pb_status pb_load_shard(pb_ctx* c) {
    pb_status st = check_ctx(c, "pb_load_shard");
    if (st) return st;
    if (c->phase != Phase::Begun) return fail(PB_EPROTOCOL, "pb_load_shard: call pb_trial_begin first");
    for (int32_t id : c->plan->load[c->rank]) c->load_bytes += c->plan->chunks[id].bytes;
    c->phase = Phase::Loaded;   // armed: issued by the trial issuer (issue_trial) in data-arrival order
    return PB_OK;
}

extern "C" pb_status pb_merge_lora(pb_ctx* c, int32_t adapter_id) {
    pb_status st = check_ctx(c, "pb_merge_lora");
    if (st) return st;
    if (c->phase != Phase::Loaded) return fail(PB_EPROTOCOL, "pb_merge_lora: call pb_load_shard first");
    if (adapter_id < PB_MERGE_ALL || adapter_id >= (int32_t)c->plan->adapters.size())
        return fail(PB_EINVAL, "adapter_id %d out of range", adapter_id);
    if (adapter_id == PB_MERGE_ALL) {
        if (c->plan->adapters.empty()) return fail(PB_EINVAL, "PB_MERGE_ALL without adapters");
        if (!c->plan->survivors.empty()) return fail(PB_EUNSUPPORTED, "PB_MERGE_ALL on a re-plan");
        if (!c->adapted) return fail(PB_ENOMEM, "PB_MERGE_ALL needs bufs.adapted >= dev_adapted_bytes");
        if (c->n > 1 && c->plan->opts.policy != PB_LOAD_STAGE)
            return fail(PB_EUNSUPPORTED, "PB_MERGE_ALL with n_gpus > 1 needs the STAGE policy (stage owner = loader)");
    }
    c->merge_adapter = c->cold_adapter = adapter_id;
    c->phase = Phase::Merged;
    return PB_OK;
}

extern "C" pb_status pb_gather_layers(pb_ctx* c) {
    pb_status st = check_ctx(c, "pb_gather_layers");
    if (st) return st;
    if (c->phase != Phase::Merged) return fail(PB_EPROTOCOL, "pb_gather_layers: call pb_merge_lora first");
    for (int32_t id : c->plan->recv[c->rank]) c->recv_bytes += c->plan->chunks[id].bytes;
    c->phase = Phase::Gathered;
    // load, merge and gather are armed: start issuing them now (copy lane, merges as chunks land, receive copies
    // as peers publish); a prompt posted later (pb_prefill_enqueue) joins the same issuer, so the prefill still
    // overlaps the loads in flight, and pb_sync without a prompt waits for T_full
    return start_load_issuer(c);
}

// ------------------------------------------------------------------------------------------------
// prefill
// ------------------------------------------------------------------------------------------------

namespace {

const __nv_bfloat16* wt(pb_ctx* c, int l, const char* sfx) {
    const pb_plan* p = c->plan;
    const int32_t t = p->find_tensor(l >= 0 ? "L" + std::to_string(l) + "." + sfx : std::string(sfx));
    return t < 0 ? nullptr : reinterpret_cast<const __nv_bfloat16*>(c->weights + p->tensors[t].dev_off);
}


// Tensor t is complete in this rank's HBM: its own-loaded part merged (f_tensor) and its received part copied
// (f_tensor_recv); chunks a re-plan marks as already held need no wait.
cudaError_t wait_tensor_ready(pb_ctx* c, int32_t t, cudaStream_t s) {
    if (c->last_own_chunk[t] >= 0) {
        cudaError_t e = wait_word(c, c->L.f_tensor + t, s);
        if (e != cudaSuccess) return e;
    }
    if (c->last_recv_chunk[t] >= 0) return wait_word(c, c->L.f_tensor_recv + t, s);
    return cudaSuccess;
}

cudaError_t wait_tensor(pb_ctx* c, int l, const char* sfx) {
    const pb_plan* p = c->plan;
    return wait_tensor_ready(c, p->find_tensor("L" + std::to_string(l) + "." + sfx), c->comp);
}

// fp32 debug-parity path: tensor sfx of layer l (or a non-layer tensor when l < 0); adapter >= 0 selects that
// adapter's out-of-place copy where it has one.
const float* wt_f32(pb_ctx* c, int l, const char* sfx, int adapter = -1) {
    const pb_plan* p = c->plan;
    const int32_t t = p->find_tensor(l >= 0 ? "L" + std::to_string(l) + "." + sfx : std::string(sfx));
    if (t < 0) return nullptr;
    if (adapter >= 0 && c->adapted) {
        const int64_t off = p->adapted_off[(size_t)adapter * p->tensors.size() + t];
        if (off >= 0) return reinterpret_cast<const float*>(c->adapted + off);
    }
    return reinterpret_cast<const float*>(c->weights + p->tensors[t].dev_off);
}

// The fp32 twin of run_layer (PB_DTYPE_F32): same steps, same waits, SIMT fp32 kernels (f32.cu).
// Layer l on token rows [r0, r1) (prompt positions [ta, tb)). On the first prompt chunk each step waits
// only for the tensors it reads (layout is in compute order), so a layer starts while its tail loads.
// Rows [r0, r1) are absolute workspace rows; attention / RoPE see the B-sequence block that starts at
// row_base (token-major inside it); adapter >= 0 selects that adapter's out-of-place weight copies.
pb_status run_layer_f32(pb_ctx* c, int l, int r0, int r1, int ta, int tb, int B, bool first_chunk, int row_base,
                        int adapter);

pb_status run_layer(pb_ctx* c, int l, int r0, int r1, int ta, int tb, int B, bool first_chunk, int row_base,
                    int adapter, int parts = 15) {
    const pb_plan* p = c->plan;
    if (p->f32()) return run_layer_f32(c, l, r0, r1, ta, tb, B, first_chunk, row_base, adapter);
    const auto& m = p->model;
    const bool opt = m.arch == PB_ARCH_OPT;
    const int d = m.d_model, hd = p->head_dim(), H = m.n_heads, KVH = m.n_kv_heads, qd = H * hd, kvd = KVH * hd;
    const int f = m.d_ffn, qdim = qkv_dim(p);
    const WsLayout& L = c->L;
    float* h = reinterpret_cast<float*>(c->ws + L.h);
    __nv_bfloat16* x = reinterpret_cast<__nv_bfloat16*>(c->ws + L.x);
    const int li = l;
    __nv_bfloat16* qkv = reinterpret_cast<__nv_bfloat16*>(c->ws + L.qkv + L.qkv_stride * li);
    __nv_bfloat16* attn = reinterpret_cast<__nv_bfloat16*>(c->ws + L.attn);
    __nv_bfloat16* mlp = reinterpret_cast<__nv_bfloat16*>(c->ws + L.mlp);
    const LayerMaps& lm = adapter >= 0 ? c->lmaps_ad[adapter][l] : c->lmaps[l];
    cudaStream_t s = c->comp;
    const int rows = r1 - r0;
    auto G = [&](int M_begin, int N, int K, int epi, const __nv_bfloat16* bias, int relu, float scale, int scale_cols,
                 void* out, int ldo) {
        GemmArgs a{};
        a.M_begin = M_begin;
        a.M_end = r1;
        a.N = N;
        a.K = K;
        a.epi = epi;
        a.relu = relu;
        a.scale = scale;
        a.scale_cols = scale_cols;
        a.bias = bias;
        a.out = out;
        a.ldo = ldo;
        a.up_row0 = f;
        a.M_total = c->gemm_m_total;  // whole prompt batch (or one decode step): chunking never changes split-K
        a.pdl = c->profiling ? 0 : 1; // per-launch timing events between kernels would cancel the overlap anyway
        a.m_dyn = c->dyn_pos;         // decode graph: rows r0.. are relative to position * B
        a.m_dyn_mul = B;
        return a;
    };
    // Algorithmic work of a GEMM launch: 2MNK flops; bytes = X + W + output (fp32 residual read + write).
    // weight wi of the layer (0 qkv, 1 o, 2 fc1 | gate_up, 3 fc2 | down): its tensor maps and plain pointer
    auto gemm = [&](const CUtensorMap& mx, const CUtensorMap& mw, GemmArgs a, int n_w_rows, const __nv_bfloat16* X,
                    int ldx, int wi) -> cudaError_t {
        a.X = X;
        a.ldx = ldx;
        a.W = lm.w[wi];
        a.mapW64 = (wi == 2 && !opt) ? nullptr : &lm.w64[wi];
        a.mapW32 = (wi == 2 && !opt) ? nullptr : &lm.w32[wi];
        const int pi = prof_begin(c, K_GEMM, s);
        cudaError_t e = launch_gemm(mx, mw, a, s);
        const double M = rows, N = a.N, K = a.K;
        const double out_b = a.epi == EPI_RESID ? 8.0 * M * N : 2.0 * M * N;
        prof_end(c, pi, s, 2.0 * M * n_w_rows * K, 2.0 * M * K + 2.0 * n_w_rows * K + out_b);
        return e;
    };
    auto norm = [&](const char* g_name, const char* b_name) -> cudaError_t {
        const int pi = prof_begin(c, K_NORM, s);
        cudaError_t e = launch_norm(h + (size_t)r0 * d, d, x + (size_t)r0 * d, d, rows, d, wt(c, l, g_name),
                                    opt ? wt(c, l, b_name) : nullptr, m.norm_eps, s, !c->profiling, c->dyn_pos, B, B);
        prof_end(c, pi, s, 8.0 * rows * d, 6.0 * rows * d);
        return e;
    };
    auto need = [&](const char* sfx) -> cudaError_t { return first_chunk ? wait_tensor(c, l, sfx) : cudaSuccess; };
    // --- attention block. parts: 1 = norm 1, 2 = QKV, 8 = attention, 4 = O, norm 2, MLP (a multi-adapter batch runs 1
    // and 4 once over every sequence's rows, 2 per sequence with its adapter's weights, and the attention of all
    // sequences as one sequence-major launch)
    if (parts & 1) {
        CU(need(opt ? "ln1_b" : "ln1_g"));
        CU(norm("ln1_g", "ln1_b"));
        ++c->n_launches;
    }
    GemmArgs a{};
    if (parts & 2) {
    CU(need(opt ? "qkv_b" : "qkv"));
    a = G(r0, qdim, d, EPI_BF16, opt ? wt(c, l, "qkv_b") : nullptr, 0, opt ? 1.0f / sqrtf((float)hd) : 1.0f,
                   opt ? d : 0, qkv, qdim);
    if (!opt) {   // Llama: RoPE on the fp32 accumulator inside the QKV epilogue, one rounding (storage contract)
        a.rope = reinterpret_cast<const float2*>(c->ws + L.rope);
        a.rope_cols = qd + kvd;
        a.rope_hd = hd;
        a.rope_row0 = row_base;
        a.rope_B = B;
    }
    CU(gemm(c->map_x, lm.qkv, a, qdim, x, d, 0));
    if (parts & 8) {
        const int pi = prof_begin(c, K_ATTN, s);
        CU(launch_attention(qkv + (size_t)row_base * qdim, qdim, attn + (size_t)row_base * qd, qd, ta, tb, B, H, KVH,
                            hd, qd, qd + kvd, opt ? 1.0f : 1.0f / sqrtf((float)hd), s, !c->profiling, c->dyn_pos,
                            L.max_seq));
        // causal pairs: sum over queries t in [ta, tb) of (t + 1) keys
        const double pairs = (double)B * ((double)tb * (tb + 1) / 2 - (double)ta * (ta + 1) / 2);
        prof_end(c, pi, s, 4.0 * pairs * H * hd, 2.0 * rows * qd * 2 + 2.0 * B * tb * 2 * kvd);
    }
    c->n_launches += (parts & 8) ? 2 : 1;
    }
    if (!(parts & 4)) return PB_OK;
    CU(need(opt ? "o_b" : "o"));
    a = G(r0, d, qd, EPI_RESID, opt ? wt(c, l, "o_b") : nullptr, 0, 1.f, 0, h, d);
    CU(gemm(c->map_attn, lm.o, a, d, attn, qd, 1));
    // --- MLP block
    CU(need(opt ? "ln2_b" : "ln2_g"));
    CU(norm("ln2_g", "ln2_b"));
    if (opt) {
        CU(need("fc1_b"));
        a = G(r0, f, d, EPI_BF16, wt(c, l, "fc1_b"), 1, 1.f, 0, mlp, f);
        CU(gemm(c->map_x, lm.up, a, f, x, d, 2));
        CU(need("fc2_b"));
        a = G(r0, d, f, EPI_RESID, wt(c, l, "fc2_b"), 0, 1.f, 0, h, d);
        CU(gemm(c->map_mlp, lm.down, a, d, mlp, f, 3));
    } else {
        CU(need("gate_up"));
        a = G(r0, f, d, EPI_SILU_MUL, nullptr, 0, 1.f, 0, mlp, f);
        CU(gemm(c->map_x, lm.up, a, 2 * f, x, d, 2));
        CU(need("down"));
        a = G(r0, d, f, EPI_RESID, nullptr, 0, 1.f, 0, h, d);
        CU(gemm(c->map_mlp, lm.down, a, d, mlp, f, 3));
    }
    c->n_launches += 4;   // o, norm, fc1|gate_up, fc2|down
    return PB_OK;
}


pb_status run_layer_f32(pb_ctx* c, int l, int r0, int r1, int ta, int tb, int B, bool first_chunk, int row_base,
                        int adapter) {
    const pb_plan* p = c->plan;
    const auto& m = p->model;
    const bool opt = m.arch == PB_ARCH_OPT;
    const int d = m.d_model, hd = p->head_dim(), H = m.n_heads, KVH = m.n_kv_heads, qd = H * hd, kvd = KVH * hd;
    const int f = m.d_ffn, qdim = qkv_dim(p);
    const WsLayout& L = c->L;
    float* h = reinterpret_cast<float*>(c->ws + L.h);
    float* x = reinterpret_cast<float*>(c->ws + L.x);
    const int li = l;
    float* qkv = reinterpret_cast<float*>(c->ws + L.qkv + L.qkv_stride * li);
    float* attn = reinterpret_cast<float*>(c->ws + L.attn);
    float* mlp = reinterpret_cast<float*>(c->ws + L.mlp);
    cudaStream_t s = c->comp;
    const int rows = r1 - r0;
    auto W = [&](const char* sfx) { return wt_f32(c, l, sfx, adapter); };
    auto need = [&](const char* sfx) -> cudaError_t { return first_chunk ? wait_tensor(c, l, sfx) : cudaSuccess; };
    auto gemm = [&](const float* X, int ldx, const float* Wt, int N, int K, int epi, const float* bias, int relu,
                    float scale, int scale_cols, float* out, int ldo, int n_w_rows) -> cudaError_t {
        const int pi = prof_begin(c, K_GEMM, s);
        cudaError_t e = launch_gemm_f32(X, ldx, r0, r1, Wt, N, K, epi, bias, relu, scale, scale_cols, out, ldo, f, s);
        prof_end(c, pi, s, 2.0 * rows * n_w_rows * K, 4.0 * ((double)rows * K + (double)n_w_rows * K + 2.0 * rows * N));
        return e;
    };
    auto norm = [&](const char* g_name, const char* b_name) -> cudaError_t {
        const int pi = prof_begin(c, K_NORM, s);
        cudaError_t e = launch_norm_f32(h + (size_t)r0 * d, d, x + (size_t)r0 * d, d, rows, d, W(g_name),
                                        opt ? W(b_name) : nullptr, m.norm_eps, s);
        prof_end(c, pi, s, 8.0 * rows * d, 8.0 * rows * d);
        return e;
    };
    CU(need(opt ? "ln1_b" : "ln1_g"));
    CU(norm("ln1_g", "ln1_b"));
    CU(need(opt ? "qkv_b" : "qkv"));
    CU(gemm(x, d, W("qkv"), qdim, d, EPI_BF16, opt ? W("qkv_b") : nullptr, 0, opt ? 1.0f / sqrtf((float)hd) : 1.0f,
            opt ? d : 0, qkv, qdim, qdim));
    if (!opt) {
        const int pi = prof_begin(c, K_ROPE, s);
        CU(launch_rope_f32(qkv + (size_t)row_base * qdim, qdim, r0 - row_base, r1 - row_base, B, H, KVH, hd, qd,
                           reinterpret_cast<const float2*>(c->ws + L.rope), s));
        prof_end(c, pi, s, 6.0 * rows * (qd + kvd) / 2, 8.0 * rows * (qd + kvd));
    }
    {
        const int pi = prof_begin(c, K_ATTN, s);
        CU(launch_attention_f32(qkv + (size_t)row_base * qdim, qdim, attn + (size_t)row_base * qd, qd, ta, tb, B, H,
                                KVH, hd, qd, qd + kvd, opt ? 1.0f : 1.0f / sqrtf((float)hd), s));
        const double pairs = (double)B * ((double)tb * (tb + 1) / 2 - (double)ta * (ta + 1) / 2);
        prof_end(c, pi, s, 4.0 * pairs * H * hd, 4.0 * rows * qd * 2 + 4.0 * B * tb * 2 * kvd);
    }
    CU(need(opt ? "o_b" : "o"));
    CU(gemm(attn, qd, W("o"), d, qd, EPI_RESID, opt ? W("o_b") : nullptr, 0, 1.f, 0, h, d, d));
    CU(need(opt ? "ln2_b" : "ln2_g"));
    CU(norm("ln2_g", "ln2_b"));
    if (opt) {
        CU(need("fc1_b"));
        CU(gemm(x, d, W("fc1"), f, d, EPI_BF16, W("fc1_b"), 1, 1.f, 0, mlp, f, f));
        CU(need("fc2_b"));
        CU(gemm(mlp, f, W("fc2"), d, f, EPI_RESID, W("fc2_b"), 0, 1.f, 0, h, d, d));
    } else {
        CU(need("gate_up"));
        CU(gemm(x, d, W("gate_up"), f, d, EPI_SILU_MUL, nullptr, 0, 1.f, 0, mlp, f, 2 * f));
        CU(need("down"));
        CU(gemm(mlp, f, W("down"), d, f, EPI_RESID, nullptr, 0, 1.f, 0, h, d, d));
    }
    c->n_launches += opt ? 7 : 8;
    return PB_OK;
}

}  // namespace

// ================================================================================================
// Trial issuer: one thread per rank issues every operation of the trial in data-arrival order —
// copy group -> the merges / peer signals / tensor words of its chunks -> the receive copies (pro rata)
// -> the compute items whose weights have been issued. Every stream has an outstanding-op budget
// (mark events polled with cudaEventQuery), so no enqueue call ever blocks inside the driver on a full
// queue: measured on B200, an enqueue blocked behind a device-side wait never recovers, and a 70B model
// has thousands of copies. Every device-side wait is issued after the operation that satisfies it
// (topological order), so the issuer can only ever poll, never deadlock.
// ================================================================================================
namespace {

struct Budget {
    static constexpr int kMarkEvery = 16, kCap = 384;
    bool capture = false;          // stream capture: nothing executes, no queue to bound, no events to poll
    cudaStream_t s = nullptr;
    cudaEvent_t* pool = nullptr;   // kPool events, reused cyclically (at most kCap/kMarkEvery+1 in flight)
    size_t next = 0;
    std::deque<std::pair<cudaEvent_t, long>> marks;
    long issued = 0, done = 0, since = 0;
    void poll() {
        while (!marks.empty() && cudaEventQuery(marks.front().first) == cudaSuccess) {
            done = marks.front().second;
            marks.pop_front();
        }
    }
    cudaError_t mark() {   // a progress event covering every op issued so far
        since = 0;
        cudaEvent_t e = pool[next++ % kEventPool];
        marks.emplace_back(e, issued);
        return cudaEventRecord(e, s);
    }
    // True when n more ops fit. A request larger than the cap is admitted once the stream is empty; the
    // ops issued since the last mark get a mark of their own so that "empty" becomes observable.
    bool can(long n) {
        if (capture || issued - done + n <= kCap) return true;
        if (since > 0 && mark() != cudaSuccess) return false;
        poll();
        return issued - done + n <= kCap || issued == done;
    }
    cudaError_t add(long n) {
        if (capture) return cudaSuccess;
        issued += n;
        since += n;
        return since >= kMarkEvery ? mark() : cudaSuccess;
    }
};

enum ItemKind { I_PROLOGUE, I_EMBED, I_WAITACT, I_LAYER, I_PUSH, I_FINAL, I_HEAD, I_ARGMAX, I_DONE, I_LAYER_ALL };
struct Item {
    int kind, mb, j, l;
    std::vector<int32_t> prereq;   // tensors whose readiness-word writer must already be issued
};

struct Issuer {
    pb_ctx* c;
    int B, T, k;
    bool replay;
    bool mb_mode;   // PB_MERGE_ALL: every sequence is its own microbatch with its own adapter
    bool replica = false;   // f3: this GPU runs the whole model alone (after T_full)
    int dec_t = -1;         // f3: decode step producing the token after position dec_t - 1 (prompt: -1)
    int n_mb;
    std::vector<int> tb;
    std::vector<Item> items;
    // the own / received part of a tensor has its readiness write issued (prerequisites of compute items)
    std::vector<char> own_issued, recv_issued, adapter_waited;
    Budget h2d, merge, nv, comp;
};

int prof_ops(pb_ctx* c) { return c->profiling ? 2 : 0; }

// ---- loads and merges of one copy group
pb_status issue_group(Issuer& I, size_t gi) {
    pb_ctx* c = I.c;
    NvtxRange nv("pb.load+merge group %d (rank %d)", (int)gi, c->rank);
    if (getenv("PB_DEBUG_ISSUER") && atoi(getenv("PB_DEBUG_ISSUER")) >= 2)
        fprintf(stderr, "[pb r%d] group %zu\n", c->rank, gi);
    const pb_plan* p = c->plan;
    const CopyGroup& g = c->copies[gi];
    const auto& ld = p->load[c->rank];
    // The landed event doubles as the merge stream's dependency: the issuer issues every copy before the
    // waits on it, so a plain event works and the copy lane carries no memop (a stream write after each
    // copy stalls the copy engine between groups, measured ~10 us per group on B200).
    const char* src = g.src;
    if (g.from_file) {   // f4: the reader has staged this group (checked by the issuer loop)
        if (c->file->read_error.load()) return fail(PB_ECUDA, "checkpoint read failed: %s", strerror(c->file->read_error.load()));
        src = c->file->ready((int64_t)gi);
    }
    CU(cudaMemcpyAsync(g.dst, src, g.bytes, cudaMemcpyHostToDevice, c->h2d[0]));
    CU(cudaEventRecord(c->landed[ld[g.first]], c->h2d[0]));
    if (gi + 1 == c->copies.size()) CU(cudaEventRecord(c->load_end, c->h2d[0]));
    if (g.from_file) c->file->issued((int64_t)gi, c->landed[ld[g.first]]);
    CU(I.h2d.add(2));
    static thread_local std::vector<int32_t> others;
    others.clear();
    for (int r = 0; r < c->n; ++r)
        if (r != c->rank) others.push_back(r);
    long mops = 0;
    static thread_local std::vector<int32_t> group_jobs;
    group_jobs.clear();
    cudaEvent_t last_wait = nullptr;
    for (int32_t i = g.first; i < g.first + g.count; ++i) {
        const int32_t id = ld[i];
        const ChunkRec& ch = p->chunks[id];
        if (ch.is_adapter) continue;
        if (landed_ev(c, id) != last_wait) {   // the chunks of a group share its landed event
            last_wait = landed_ev(c, id);
            CU(cudaStreamWaitEvent(c->merge, last_wait, 0));
            ++mops;
        }
        const bool all = c->merge_adapter == PB_MERGE_ALL;
        if (c->backup && !all && p->backup_off[ch.tensor] >= 0) {   // f2: keep the pristine base of the chunk
            CU(launch_copy(c->backup + p->backup_off[ch.tensor] + (int64_t)ch.r0 * p->tensors[ch.tensor].row_bytes(),
                           c->weights + ch.dev_off, ch.bytes, c->merge));
            ++c->n_launches;
            ++mops;
        }
        if (all) {   // out of place: rows of the chunk no merge of adapter a writes are copied on the SMs
            const size_t NT = p->tensors.size();
            const TensorRec& t = p->tensors[ch.tensor];
            for (size_t a = 0; a < p->adapters.size(); ++a) {
                const int64_t off = p->adapted_off[a * NT + ch.tensor];
                if (off < 0) continue;
                std::vector<std::pair<int32_t, int32_t>> cover;
                for (auto& mr : p->merges)
                    if (mr.adapter == (int32_t)a && mr.base == ch.tensor) cover.push_back({mr.row0, mr.row0 + mr.rows});
                std::sort(cover.begin(), cover.end());
                int32_t r = ch.r0;
                auto copy_rows = [&](int32_t r_a, int32_t r_b) -> cudaError_t {
                    if (r_b <= r_a) return cudaSuccess;
                    ++mops;
                    return launch_copy(c->adapted + off + (int64_t)r_a * t.row_bytes(),
                                       c->weights + t.dev_off + (int64_t)r_a * t.row_bytes(),
                                       (int64_t)(r_b - r_a) * t.row_bytes(), c->merge);
                };
                for (auto& cv : cover) {
                    CU(copy_rows(r, std::min(cv.first, ch.r1)));
                    r = std::max(r, std::min(cv.second, ch.r1));
                }
                CU(copy_rows(r, ch.r1));
            }
        }
        for (int32_t j : c->jobs_of_chunk[id]) {
            const MergeJob& job = c->jobs[j];
            if (all ? job.inplace : (!job.inplace || job.adapter != c->merge_adapter)) continue;
            for (int32_t a : job.need)
                if (!I.adapter_waited[a] && c->landed_alias[a] >= 0) {   // < 0: not loaded by this trial (held)
                    CU(cudaStreamWaitEvent(c->merge, landed_ev(c, a), 0));
                    I.adapter_waited[a] = 1;
                    ++mops;
                }
            group_jobs.push_back(j);
        }
    }
    // The adapted chunks of the group (they landed together) merge in as few launches as possible: up to
    // kMaxMergeJobs jobs of one padded rank per persistent launch.
    for (size_t k = 0; k < group_jobs.size();) {
        if (p->f32()) {
            const MergeJob& job = c->jobs[group_jobs[k++]];
            const int pi = prof_begin(c, K_MERGE, c->merge);
            CU(launch_merge_f32(job.W, job.Wout, job.ldw, job.rows, job.cols, job.Bp, job.Ap, job.rank, job.scale,
                                c->merge));
            prof_end(c, pi, c->merge, 2.0 * job.rows * job.cols * job.rank,
                     p->es() * (2.0 * job.rows * job.cols + (double)job.rank * (job.rows + job.cols)));
            ++c->n_launches;
            mops += 1 + prof_ops(c);
            continue;
        }
        MergeJobDesc batch[kMaxMergeJobs];
        int nb = 0;
        double flops = 0, bytes = 0;
        const int rk = merge_rk(c->jobs[group_jobs[k]].rank);
        while (k < group_jobs.size() && nb < kMaxMergeJobs && merge_rk(c->jobs[group_jobs[k]].rank) == rk) {
            const MergeJob& job = c->jobs[group_jobs[k++]];
            batch[nb++] = MergeJobDesc{&job.maps, job.rows, job.cols, job.rank, job.scale};
            flops += 2.0 * job.rows * job.cols * job.rank;
            bytes += p->es() * (2.0 * job.rows * job.cols + (double)job.rank * (job.rows + job.cols));
        }
        const int pi = prof_begin(c, K_MERGE, c->merge);
        CU(launch_merge_batch(batch, nb, c->merge));
        prof_end(c, pi, c->merge, flops, bytes);
        ++c->n_launches;
        mops += 1 + prof_ops(c);
    }
    for (int32_t i = g.first; i < g.first + g.count; ++i) {
        const int32_t id = ld[i];
        const ChunkRec& ch = p->chunks[id];
        if (ch.is_adapter) continue;
        if (c->merged_ev[id]) {   // timing mode (PB_LANDED_TIMING=1): per-chunk merged timestamp
            CU(cudaEventRecord(c->merged_ev[id], c->merge));
            ++mops;
        }
        if (!others.empty()) {
            CU(signal_ranks(c, c->L.f_chunk + id, others, c->merge));
            mops += 1 + prof_ops(c);
        }
        if (c->last_own_chunk[ch.tensor] == id) {
            CU(set_word(c, c->L.f_tensor + ch.tensor, c->merge));
            I.own_issued[ch.tensor] = 1;
            ++mops;
        }
        if (id == c->last_own_stage_chunk) {
            CU(cudaEventRecord(c->ready_merge, c->merge));
            ++mops;
        }
    }
    CU(I.merge.add(mops));
    return PB_OK;
}

// A compute item's prerequisite t >= 0: every part of tensor t this rank does not already hold (own loads and
// received chunks) has its readiness write issued; -(t+1): only the own-loaded part (vocab slices).
bool prereq_issued(const Issuer& I, int32_t t) {
    const pb_ctx* c = I.c;
    if (t < 0) {
        t = -t - 1;
        return I.own_issued[t] || c->last_own_chunk[t] < 0;
    }
    return (I.own_issued[t] || c->last_own_chunk[t] < 0) && (I.recv_issued[t] || c->last_recv_chunk[t] < 0);
}

long group_merge_ops(Issuer& I, size_t gi) {
    pb_ctx* c = I.c;
    const CopyGroup& g = c->copies[gi];
    long n = 0;
    for (int32_t i = g.first; i < g.first + g.count; ++i) {
        const int32_t id = c->plan->load[c->rank][i];
        n += 7 + (long)c->plan->adapters.size() + (long)c->jobs_of_chunk[id].size() * (5 + prof_ops(c));
    }
    return n;
}

pb_status issue_recv(Issuer& I, size_t ri) {
    pb_ctx* c = I.c;
    NvtxRange nv("pb.gather recv %d (rank %d)", (int)ri, c->rank);
    if (getenv("PB_DEBUG_ISSUER") && atoi(getenv("PB_DEBUG_ISSUER")) >= 2)
        fprintf(stderr, "[pb r%d] recv %zu\n", c->rank, ri);
    const int32_t id = c->plan->recv[c->rank][ri];
    const ChunkRec& ch = c->plan->chunks[id];
    CU(wait_word(c, c->L.f_chunk + id, c->nv));
    CU(cudaMemcpyAsync(c->weights + ch.dev_off, c->peers[ch.loader].weights + ch.dev_off, ch.bytes,
                       cudaMemcpyDeviceToDevice, c->nv));
    CU(cudaEventRecord(c->gathered[id], c->nv));
    long n = 3;
    if (c->last_recv_chunk[ch.tensor] == id) {
        CU(set_word(c, c->L.f_tensor_recv + ch.tensor, c->nv));
        I.recv_issued[ch.tensor] = 1;
        ++n;
    }
    if (id == c->last_recv_stage_chunk) {
        CU(cudaEventRecord(c->ready_recv, c->nv));
        ++n;
    }
    CU(I.nv.add(n));
    return PB_OK;
}

// Multi-adapter microbatches (PB_MERGE_ALL: each sequence on its adapter's out-of-place copies) at the last stage:
// when no adapter of the batch touches layer l's O / MLP weights (every microbatch's maps point at the same base
// tensors), norm 1, O, norm 2 and the MLP of all sequences run as ONE launch each over all rows (weights read once
// instead of once per sequence; the M_total that picks the kernel and the split stays one sequence's rows, so the
// sums are the same as per sequence); QKV + attention stay per sequence. PB_NO_MB_BATCH=1 disables it.
static bool shared_weight_batch(const Issuer& I, int l) {
    const pb_ctx* c = I.c;
    static const bool off = getenv("PB_NO_MB_BATCH") != nullptr;
    if (off || !I.mb_mode || I.k != 1 || I.n_mb < 2 || I.dec_t >= 0 || c->plan->f32() || c->dyn_pos) return false;
    for (int mb = 0; mb < I.n_mb; ++mb) {
        const int a = c->seq_adapter[mb];
        if (a < 0) return false;
        for (int wi = 1; wi < 4; ++wi)
            if (c->lmaps_ad[a][l].w[wi] != c->lmaps[l].w[wi]) return false;
    }
    return true;
}

void build_items(Issuer& I) {
    pb_ctx* c = I.c;
    const pb_plan* p = c->plan;
    const bool opt = p->model.arch == PB_ARCH_OPT;
    const int g = c->rank, N = c->n;
    const bool rep = I.replica;
    const auto stage = rep ? std::make_pair(0, p->model.n_layers) : p->stages[g];
    const bool first = g == 0 || rep, last = g == N - 1 || rep;
    auto add = [&](int kind, int mb, int j, int l, std::vector<int32_t> pre) {
        if (I.replay) pre.clear();
        I.items.push_back(Item{kind, mb, j, l, std::move(pre)});
    };
    add(I_PROLOGUE, 0, 0, 0, {});
    auto layer_pre = [&](int l) {
        std::vector<int32_t> pre;
        for (size_t t = 0; t < p->tensors.size(); ++t)
            if (p->tensors[t].layer == l) pre.push_back((int32_t)t);
        return pre;
    };
    auto head_item = [&](int mb, int j) {   // embedding (stage 0) or the previous stage's activation
        if (first) {
            std::vector<int32_t> pre;
            if (mb == 0 && j == 0) {
                const int32_t et = p->find_tensor("embed");
                if (p->opts.vocab_sliced) {
                    if (c->last_own_chunk[et] >= 0) pre.push_back(-et - 1);   // own slice only
                } else {
                    pre.push_back(et);
                }
                if (opt) pre.push_back(p->find_tensor("pos"));
            }
            add(I_EMBED, mb, j, 0, pre);
        } else {
            add(I_WAITACT, mb, j, 0, {});
        }
    };
    if (last && (I.n_mb > 1 || I.k > 1)) {
        // Last stage (no downstream consumer): layer-major, so every microbatch / prompt chunk advances as each
        // layer lands instead of all but the first waiting for the whole stage.
        for (int l = stage.first; l < stage.second; ++l) {
            if (shared_weight_batch(I, l)) {   // the sequences' shared projections as one GEMM each
                if (l == stage.first)
                    for (int mb = 0; mb < I.n_mb; ++mb) head_item(mb, 0);
                add(I_LAYER_ALL, 0, 0, l, layer_pre(l));
                continue;
            }
            for (int mb = 0; mb < I.n_mb; ++mb)
                for (int j = 0; j < I.k; ++j) {
                    if (l == stage.first) head_item(mb, j);
                    add(I_LAYER, mb, j, l, mb == 0 && j == 0 ? layer_pre(l) : std::vector<int32_t>{});
                }
        }
    } else {
        // Intermediate stage: chunk-major, so chunk 0 reaches the next stage as early as possible.
        for (int mb = 0; mb < I.n_mb; ++mb)
            for (int j = 0; j < I.k; ++j) {
                head_item(mb, j);
                for (int l = stage.first; l < stage.second; ++l)
                    add(I_LAYER, mb, j, l, mb == 0 && j == 0 ? layer_pre(l) : std::vector<int32_t>{});
                if (!last) add(I_PUSH, mb, j, 0, {});
            }
    }
    if (last) {
        std::vector<int32_t> pre{p->find_tensor("final_g")};
        if (opt) pre.push_back(p->find_tensor("final_b"));
        add(I_FINAL, 0, 0, 0, pre);
    }
    if (rep || is_head_owner(p, g))
        add(I_HEAD, 0, 0, 0, {p->opts.vocab_sliced ? -head_tensor(p) - 1 : head_tensor(p)});
    if (first) add(I_ARGMAX, 0, 0, 0, {});
    add(I_DONE, 0, 0, 0, {});
}

long item_ops(Issuer& I, const Item& it) {
    const int po = prof_ops(I.c);
    switch (it.kind) {
        case I_LAYER: return 16 + 8 * po;
        case I_LAYER_ALL: return (16 + 8 * po) * (I.n_mb + 1);
        case I_EMBED: return 8 + po;
        default: return 8 + po;
    }
}

static bool issuer_trace() {
    static const bool on = getenv("PB_DEBUG_ISSUER") && atoi(getenv("PB_DEBUG_ISSUER")) >= 2;
    return on;
}

pb_status issue_item(Issuer& I, const Item& it, bool late_tokens) {
    pb_ctx* c = I.c;
    NvtxRange nv("pb.prefill item kind %d layer %d", it.kind, it.l);
    if (issuer_trace()) fprintf(stderr, "[pb r%d] item kind=%d mb=%d j=%d l=%d\n", c->rank, it.kind, it.mb, it.j, it.l);
    const pb_plan* p = c->plan;
    const auto& m = p->model;
    const bool opt = m.arch == PB_ARCH_OPT;
    const int g = c->rank, N = c->n, d = m.d_model, hd = p->head_dim(), B = I.B, T = I.T, V = m.vocab;
    const bool rep = I.replica;
    const WsLayout& L = c->L;
    cudaStream_t s = c->comp;
    float* h = reinterpret_cast<float*>(c->ws + L.h);
    __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(c->ws + L.y);
    float* logits = reinterpret_cast<float*>(c->ws + L.logits);
    const int j = it.j;
    // microbatch mode: sequence it.mb occupies rows [mb*T, (mb+1)*T) (one sequence, Bk = 1);
    // otherwise all B sequences share the token-major rows t*B + b.
    const int Bk = I.mb_mode ? 1 : B;
    const int row_base = I.mb_mode ? it.mb * T : 0;
    const int r0 = row_base + I.tb[j] * Bk, r1 = row_base + I.tb[j + 1] * Bk;
    const int act_word = L.f_act + it.mb * I.k + j;
    std::vector<int32_t> owners;   // ranks computing a slice of the logits (a replica: itself, the whole vocabulary)
    if (rep) owners.push_back(g);
    else
        for (int r = 0; r < N; ++r)
            if (is_head_owner(p, r)) owners.push_back(r);
    switch (it.kind) {
        case I_PROLOGUE:
            if (!opt && I.dec_t < 0) {   // positions up to the workspace's max_seq: decode steps reuse the table
                CU(launch_rope_table(reinterpret_cast<float2*>(c->ws + L.rope), L.max_seq, hd, m.rope_theta, s));
                ++c->n_launches;
            }
            if (g == 0 || rep) {
                // the token upload went out on the copy lane ahead of the weights (issue_trial): an H2D copy on
                // this stream would queue behind the whole load in the copy engine (measured: drains per stream)
                if (c->dyn_pos) {   // decode graph: position from the host's pinned word, then feed the tokens
                    CU(cudaMemcpyAsync(c->ws + L.dpos, c->h_pos, sizeof(int32_t), cudaMemcpyHostToDevice, s));
                    CU(launch_feed_tokens(reinterpret_cast<int32_t*>(c->ws + L.tokens),
                                          reinterpret_cast<const int32_t*>(c->ws + L.tok_out), c->dyn_pos, B, s));
                    ++c->n_launches;
                } else if (I.dec_t >= 0)   // decode: the previous step's tokens become position dec_t's inputs
                    CU(cudaMemcpyAsync(c->ws + L.tokens + sizeof(int32_t) * (size_t)I.dec_t * B, c->ws + L.tok_out,
                                       sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, s));
                else if (I.replay)
                    CU(cudaMemcpyAsync(c->ws + L.tokens, c->h_tokens, sizeof(int32_t) * B * T, cudaMemcpyHostToDevice, s));
                else if (late_tokens)   // posted after the load started: SM copy from the mapped pinned staging
                    CU(launch_copy(c->ws + L.tokens, c->h_tokens, sizeof(int32_t) * B * T, s));
                else
                    CU(cudaStreamWaitEvent(s, c->tok_ev, 0));
                CU(cudaMemsetAsync(c->ws + L.nan, 0, 4, s));
            }
            break;
        case I_EMBED: {
            const int32_t et = p->find_tensor("embed");
            if (j == 0 && !I.replay) {
                if (p->opts.vocab_sliced) {
                    // embedding rows live on every rank (vocab slices): wait for each remote piece at its owner
                    for (auto& ch : p->chunks)
                        if (!ch.is_adapter && ch.tensor == et && ch.loader != g) CU(wait_word(c, L.f_chunk + ch.id, s));
                    if (c->last_own_chunk[et] >= 0) CU(wait_word(c, L.f_tensor + et, s));
                } else {
                    CU(wait_tensor_ready(c, et, s));
                }
                if (opt) CU(wait_tensor_ready(c, p->find_tensor("pos"), s));
            }
            EmbedSrc E{};
            if (p->opts.vocab_sliced && !rep) {
                std::vector<int32_t> sl(N + 1, 0);
                for (auto& ch : p->chunks)
                    if (!ch.is_adapter && ch.tensor == et) sl[ch.loader + 1] = std::max(sl[ch.loader + 1], ch.r1);
                for (int r = 0; r < N; ++r) {
                    E.base[r] = c->peers[r].weights + p->tensors[et].dev_off;
                    E.slice_begin[r] = r == 0 ? 0 : sl[r];
                }
                E.slice_begin[N] = INT32_MAX;
                E.n = N;
            } else {
                E.base[0] = wt(c, -1, "embed");
                E.slice_begin[0] = 0;
                E.slice_begin[1] = INT32_MAX;
                E.n = 1;
            }
            const int pi = prof_begin(c, K_EMBED, s);
            if (p->f32())
                CU(launch_embed_f32(E, opt ? wt_f32(c, -1, "pos") : nullptr,
                                    reinterpret_cast<const int32_t*>(c->ws + L.tokens) + row_base,
                                    h + (size_t)row_base * d, d, r0 - row_base, r1 - row_base, Bk, s));
            else
                CU(launch_embed(E, opt ? wt(c, -1, "pos") : nullptr,
                                reinterpret_cast<const int32_t*>(c->ws + L.tokens) + row_base, h + (size_t)row_base * d,
                                d, r0 - row_base, r1 - row_base, Bk, s, !c->profiling, c->dyn_pos));
            prof_end(c, pi, s, (opt ? 1.0 : 0.0) * (r1 - r0) * d, (r1 - r0) * d * (opt ? 8.0 : 6.0));
            ++c->n_launches;
            break;
        }
        case I_WAITACT:
            CU(wait_word(c, act_word, s));
            break;
        case I_LAYER: {
            const int adapter = I.mb_mode ? c->seq_adapter[it.mb] : -1;
            const auto stage = rep ? std::make_pair(0, m.n_layers) : p->stages[g];
            if (it.l == stage.first && it.mb == 0 && j == 0) CU(record_ev(c, c->stage_begin, s));
            pb_status st = run_layer(c, it.l, r0, r1, I.tb[j], I.tb[j + 1], Bk, it.mb == 0 && j == 0 && !I.replay,
                                     row_base, adapter);
            if (st) return st;
            if (it.l == stage.second - 1 && it.mb == I.n_mb - 1 && j == I.k - 1) CU(record_ev(c, c->stage_end, s));
            break;
        }
        case I_LAYER_ALL: {   // shared_weight_batch(): sequence mb occupies rows [mb*T, (mb+1)*T)
            const auto stage = rep ? std::make_pair(0, m.n_layers) : p->stages[g];
            const bool first_chunk = !I.replay;
            if (it.l == stage.first) CU(record_ev(c, c->stage_begin, s));
            pb_status st = run_layer(c, it.l, 0, I.n_mb * T, 0, T, 1, first_chunk, 0, -1, 1);
            for (int mb = 0; mb < I.n_mb && st == PB_OK; ++mb)
                st = run_layer(c, it.l, mb * T, (mb + 1) * T, 0, T, 1, first_chunk, mb * T, c->seq_adapter[mb], 2);
            if (st) return st;
            {   // the attention of every sequence in one launch (sequence-major rows b*T + t)
                const int H = m.n_heads, KVH = m.n_kv_heads, qd = H * hd, kvd = KVH * hd, qdim = qkv_dim(p);
                const __nv_bfloat16* qkv = reinterpret_cast<const __nv_bfloat16*>(c->ws + L.qkv + L.qkv_stride * it.l);
                __nv_bfloat16* attn = reinterpret_cast<__nv_bfloat16*>(c->ws + L.attn);
                const int pi = prof_begin(c, K_ATTN, s);
                CU(launch_attention(qkv, qdim, attn, qd, 0, T, I.n_mb, H, KVH, hd, qd, qd + kvd,
                                    opt ? 1.0f : 1.0f / sqrtf((float)hd), s, !c->profiling, nullptr, 0, T));
                const double pairs = (double)I.n_mb * ((double)T * (T + 1) / 2);
                prof_end(c, pi, s, 4.0 * pairs * H * hd, 2.0 * I.n_mb * T * qd * 2 + 2.0 * I.n_mb * T * 2 * kvd);
                ++c->n_launches;
            }
            st = run_layer(c, it.l, 0, I.n_mb * T, 0, T, 1, first_chunk, 0, -1, 4);
            if (st) return st;
            if (it.l == stage.second - 1) CU(record_ev(c, c->stage_end, s));
            break;
        }
        case I_PUSH:
            CU(cudaMemcpyAsync(c->peers[g + 1].ws + L.h + (size_t)r0 * d * 4, h + (size_t)r0 * d,
                               (size_t)(r1 - r0) * d * 4, cudaMemcpyDeviceToDevice, s));
            CU(signal_ranks(c, act_word, {g + 1}, s));
            break;
        case I_FINAL: {
            if (!I.replay) {
                CU(wait_tensor_ready(c, p->find_tensor("final_g"), s));
                if (opt) CU(wait_tensor_ready(c, p->find_tensor("final_b"), s));
            }
            // last position of every sequence: token-major rows (T-1)*B + b, or microbatch rows b*T + T-1
            const float* last = I.mb_mode ? h + (size_t)(T - 1) * d : h + (size_t)(T - 1) * B * d;
            const int ldh = I.mb_mode ? T * d : d;
            const int pi = prof_begin(c, K_NORM, s);
            if (p->f32())
                CU(launch_norm_f32(last, ldh, reinterpret_cast<float*>(c->ws + L.y), d, B, d, wt_f32(c, -1, "final_g"),
                                   opt ? wt_f32(c, -1, "final_b") : nullptr, m.norm_eps, s));
            else
                CU(launch_norm(last, ldh, y, d, B, d, wt(c, -1, "final_g"), opt ? wt(c, -1, "final_b") : nullptr,
                               m.norm_eps, s, !c->profiling, c->dyn_pos, B, 0));
            prof_end(c, pi, s, 8.0 * B * d, 6.0 * B * d);
            ++c->n_launches;
            std::vector<int32_t> remote;
            for (int32_t r : owners)
                if (r != g) {
                    CU(cudaMemcpyAsync(c->peers[r].ws + L.y, c->ws + L.y, (size_t)B * d * p->es(),
                                       cudaMemcpyDeviceToDevice, s));
                    remote.push_back(r);
                }
            CU(signal_ranks(c, L.f_y, remote, s));
            break;
        }
        case I_HEAD: {
            if (!rep && g != N - 1) CU(wait_word(c, L.f_y, s));
            const int32_t ht = head_tensor(p);
            if (!I.replay) {   // vocab slices: this rank's own rows; whole head: every part of it
                if (p->opts.vocab_sliced) CU(wait_word(c, L.f_tensor + ht, s));
                else CU(wait_tensor_ready(c, ht, s));
            }
            int32_t v0 = 0, v1 = V;
            if (!rep) head_slice(p, g, &v0, &v1);
            const __nv_bfloat16* E = reinterpret_cast<const __nv_bfloat16*>(c->weights + p->tensors[ht].dev_off);
            const int pi = prof_begin(c, K_LOGITS, s);
            if (p->f32())
                CU(launch_logits_f32(reinterpret_cast<const float*>(c->ws + L.y), B, d,
                                     reinterpret_cast<const float*>(E), v0, v1, logits, V, s));
            else
                CU(launch_logits(y, B, d, E, v0, v1, logits, V, s, !c->profiling));
            prof_end(c, pi, s, 2.0 * B * (v1 - v0) * d, 2.0 * (double)(v1 - v0) * d + 4.0 * B * (v1 - v0));
            ++c->n_launches;
            if (g != 0 && !rep) {
                CU(cudaMemcpy2DAsync(c->peers[0].ws + L.logits + (size_t)v0 * 4, (size_t)V * 4, logits + v0,
                                     (size_t)V * 4, (size_t)(v1 - v0) * 4, B, cudaMemcpyDeviceToDevice, s));
                CU(signal_ranks(c, L.f_logit + g, {0}, s));
            }
            break;
        }
        case I_ARGMAX: {
            for (int32_t r : owners)
                if (r != g) CU(wait_word(c, L.f_logit + r, s));
            const int pi = prof_begin(c, K_ARGMAX, s);
            CU(launch_argmax(logits, B, V, V, reinterpret_cast<int32_t*>(c->ws + L.tok_out),
                             reinterpret_cast<int32_t*>(c->ws + L.nan), s, !c->profiling));
            prof_end(c, pi, s, 0, 4.0 * B * V);
            ++c->n_launches;
            CU(cudaMemcpyAsync(c->h_out, c->ws + L.tok_out, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpyAsync(c->h_out + B, c->ws + L.nan, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            break;
        }
        case I_DONE:
            CU(record_ev(c, c->done, s));
            break;
    }
    return PB_OK;
}

}  // namespace

// One trial's issuer state. A cold start creates it in pb_gather_layers (load -> merge -> gather are armed, so the
// copy lane, the merges and the receive copies start at once); pb_prefill_enqueue later posts the prompt and the
// same issuer adds the compute items to the loads still in flight. Replays and decode steps create it with the
// prompt already posted and nothing to load.
struct pb::TrialRun {
    Issuer I;
    size_t G = 0, R = 0, gi = 0, ri = 0, ii = 0;
    bool merge_done_rec = false, gather_done_rec = false;
    bool items_built = false;
    bool late_tokens = false;   // the prompt came after the first copy group was issued (see I_PROLOGUE)
};

namespace {

std::shared_ptr<TrialRun> init_run(pb_ctx* c, bool replay) {
    const pb_plan* p = c->plan;
    auto run = std::make_shared<TrialRun>();
    Issuer& I = run->I;
    I.c = c;
    I.replay = replay;
    I.mb_mode = c->merge_adapter == PB_MERGE_ALL;
    I.replica = c->replica;
    I.own_issued.assign(p->tensors.size(), replay ? 1 : 0);
    I.recv_issued.assign(p->tensors.size(), replay ? 1 : 0);
    I.adapter_waited.assign(p->chunks.size(), 0);
    cudaStream_t ss[4] = {c->h2d[0], c->merge, c->nv, c->comp};
    Budget* bs[4] = {&I.h2d, &I.merge, &I.nv, &I.comp};
    for (int i = 0; i < 4; ++i) {
        bs[i]->s = ss[i];
        bs[i]->pool = c->budget_events.data() + i * kEventPool;
        bs[i]->capture = c->capturing;
    }
    run->G = replay ? 0 : c->copies.size();
    run->R = replay ? 0 : p->recv[c->rank].size();
    run->merge_done_rec = run->gather_done_rec = replay;
    if (!replay && c->file) c->file->start(c->copies, static_cast<const char*>(c->host_base));
    return run;
}

// The prompt of the trial: batch B x T tokens staged in c->h_tokens (rank 0 / replica).
pb_status post_prompt(pb_ctx* c, TrialRun& run, int B, int T) {
    const pb_plan* p = c->plan;
    Issuer& I = run.I;
    I.B = B;
    I.T = T;
    I.n_mb = I.mb_mode ? B : 1;
    I.dec_t = c->decode_t;
    if (I.dec_t >= 0) {   // f3 decode step: one "prompt chunk" holding position dec_t of every sequence
        I.k = 1;
        I.tb = {I.dec_t, I.dec_t + 1};
        c->gemm_m_total = B;
    } else {
        I.k = std::max(1, std::min(p->opts.prefill_chunks, T));
        I.tb.assign(I.k + 1, 0);
        for (int j = 0, t = 0; j <= I.k; ++j) {   // prompt chunk boundaries, remainder to lower chunks
            I.tb[j] = t;
            if (j < I.k) t += T / I.k + (j < T % I.k ? 1 : 0);
        }
        // rows one GEMM launch covers at most: the whole batch, or one sequence in microbatch mode (PB_MERGE_ALL)
        c->gemm_m_total = I.mb_mode ? T : B * T;
    }
    build_items(I);
    if (!I.replay && c->rank == 0) {
        if (run.gi == 0) {   // nothing on the copy lane yet: the tokens go first and land in microseconds
            CU(cudaMemcpyAsync(c->ws + c->L.tokens, c->h_tokens, sizeof(int32_t) * B * T, cudaMemcpyHostToDevice,
                               c->h2d[0]));
            CU(cudaEventRecord(c->tok_ev, c->h2d[0]));
            CU(I.h2d.add(2));
        } else {
            // the load is already streaming: an H2D copy would queue behind it in the copy engine (measured: the
            // engine drains one stream's queue before another's), so the prologue pulls the tokens from the
            // pinned (device-mapped) staging buffer with an SM copy instead
            run.late_tokens = true;
        }
    }
    run.items_built = true;
    return PB_OK;
}

// Issue the trial in data-arrival order until everything known so far is issued. Returns once the loads and
// receives are issued and either the prompt's compute items are issued too or no prompt has been posted (the
// caller then marks the loader idle under run_mu; a later post restarts the loop).
pb_status run_loop(pb_ctx* c, TrialRun& run) {
    const pb_plan* p = c->plan;
    Issuer& I = run.I;
    static const bool dbg = getenv("PB_DEBUG_ISSUER") != nullptr;
    auto last_report = std::chrono::steady_clock::now();
    const size_t G = run.G, R = run.R;
    size_t& gi = run.gi;
    size_t& ri = run.ri;
    size_t& ii = run.ii;
    for (;;) {
        if (c->abort_req.load(std::memory_order_relaxed)) return fail(PB_ECUDA, "trial aborted (pb_ctx_abort)");
        if (!run.items_built && c->posted.load(std::memory_order_acquire)) {
            pb_status st = post_prompt(c, run, c->cur_batch, c->cur_seq);
            if (st) return st;
        }
        const size_t NI = run.items_built ? I.items.size() : 0;
        if (gi >= G && ri >= R && (ii >= NI && (run.items_built || !c->posted.load(std::memory_order_acquire))))
            break;
        bool progressed = false;
        if (c->file && !I.replay) c->file->reclaim();
        auto staged = [&](size_t k) {   // f4: a file-backed group can go once the reader has filled its slot
            return !c->copies[k].from_file || c->file->ready((int64_t)k) || c->file->read_error.load();
        };
        while (gi < G && staged(gi) && I.h2d.can(2) && I.merge.can(group_merge_ops(I, gi))) {
            pb_status st = issue_group(I, gi++);
            if (st) return st;
            progressed = true;
        }
        if (!run.merge_done_rec && gi == G) {   // t_full: recorded once the last merge work is on its stream
            CU(cudaEventRecord(c->merge_done, c->merge));
            run.merge_done_rec = true;
        }
        const size_t target = gi >= G ? R : (gi * R) / std::max<size_t>(G, 1);
        while (ri < target && I.nv.can(5)) {
            pb_status st = issue_recv(I, ri++);
            if (st) return st;
            progressed = true;
        }
        if (!run.gather_done_rec && ri == R && gi == G) {
            CU(cudaEventRecord(c->gather_done, c->nv));
            if (c->n > 1) {   // tell every peer this rank has copied all it gathers (an in-place switch waits on it)
                std::vector<int32_t> others;
                for (int r = 0; r < c->n; ++r)
                    if (r != c->rank) others.push_back(r);
                CU(signal_ranks(c, c->L.f_gdone + c->rank, others, c->nv));
            }
            run.gather_done_rec = true;
        }
        while (ii < NI) {
            const Item& it = I.items[ii];
            bool ok = true;
            for (int32_t t : it.prereq) ok = ok && prereq_issued(I, t);
            if (!ok || !I.comp.can(item_ops(I, it))) break;
            pb_status st = issue_item(I, it, run.late_tokens);
            if (st) return st;
            CU(I.comp.add(item_ops(I, it)));
            ++ii;
            progressed = true;
        }
        if (!progressed) {
            std::this_thread::sleep_for(std::chrono::microseconds(20));
            if (dbg && std::chrono::steady_clock::now() - last_report > std::chrono::seconds(2)) {
                last_report = std::chrono::steady_clock::now();
                const Item* it = ii < NI ? &I.items[ii] : nullptr;
                int missing = -1;
                if (it)
                    for (int32_t t : it->prereq)
                        if (!prereq_issued(I, t)) { missing = t; break; }
                fprintf(stderr,
                        "[pb issuer r%d] stalled: groups %zu/%zu recv %zu/%zu items %zu/%zu (kind %d j %d l %d, missing "
                        "tensor %d) outstanding h2d %ld merge %ld nv %ld comp %ld\n",
                        c->rank, gi, G, ri, R, ii, NI, it ? it->kind : -1, it ? it->j : -1, it ? it->l : -1,
                        missing, I.h2d.issued - I.h2d.done, I.merge.issued - I.merge.done, I.nv.issued - I.nv.done,
                        I.comp.issued - I.comp.done);
            }
        }
    }
    (void)p;
    return PB_OK;
}

// Synchronous trial (replays, decode steps, graph capture): prompt posted up front, nothing to load.
pb_status issue_trial(pb_ctx* c, int B, int T, bool replay) {
    auto run = init_run(c, replay);
    pb_status st = post_prompt(c, *run, B, T);
    if (st) return st;
    c->posted.store(true);
    st = run_loop(c, *run);
    if (st) return st;
    if (!run->merge_done_rec) CU(cudaEventRecord(c->merge_done, c->merge));
    if (!run->gather_done_rec) CU(cudaEventRecord(c->gather_done, c->nv));
    return PB_OK;
}

// The issuer thread of a cold start: loops until everything posted is issued; if the prompt has not been posted
// by then it marks itself idle (under run_mu, so a concurrent post either sees the running thread or restarts it).
void issuer_thread(pb_ctx* c, std::shared_ptr<TrialRun> run) {
    cudaSetDevice(c->device);
    NvtxRange nv("pb.issuer trial (rank %d, epoch %d)", c->rank, (int)c->epoch);
    for (;;) {
        pb_status st = run_loop(c, *run);
        if (st != PB_OK) {
            std::lock_guard<std::mutex> lk(c->run_mu);
            c->issue_status = st;
            snprintf(c->issue_msg, sizeof c->issue_msg, "%s", pb_last_error());
            c->loader_idle = true;
            return;
        }
        std::lock_guard<std::mutex> lk(c->run_mu);
        if (run->items_built || !c->posted.load()) {   // done, or nothing more to do until a prompt is posted
            c->loader_idle = true;
            return;
        }
    }
}

void spawn_issuer(pb_ctx* c) {
    c->loader_idle = false;
    c->load_thread = std::thread(issuer_thread, c, c->run);
}

}  // namespace

static pb_status start_load_issuer(pb_ctx* c) {
    std::lock_guard<std::mutex> lk(c->run_mu);
    c->issue_status = PB_OK;
    c->issue_msg[0] = '\0';
    c->run = init_run(c, false);
    c->posted.store(false);
    spawn_issuer(c);
    return PB_OK;
}

namespace {

pb_status start_issuer(pb_ctx* c, const int32_t* tokens, const int32_t* adapter_of_seq, int32_t B, int32_t T,
                       bool replay) {
    if (B < 1 || T < 1 || B > c->L.max_batch || T > c->L.max_seq || (int64_t)B * T > c->L.max_rows)
        return fail(PB_EINVAL, "batch %d x seq %d exceeds the workspace (%d x %d)", B, T, c->L.max_batch, c->L.max_seq);
    if ((c->rank == 0 || c->replica) && !tokens) return fail(PB_EINVAL, "rank 0 (every rank of a replica) needs tokens");
    if (tokens) {
        const int32_t V = c->plan->model.vocab;
        for (int64_t i = 0; i < (int64_t)B * T; ++i)
            if (tokens[i] < 0 || tokens[i] >= V)
                return fail(PB_EINVAL, "token %d at [%lld] outside the vocabulary [0, %d)", tokens[i], (long long)i, V);
    }
    const bool mb = c->merge_adapter == PB_MERGE_ALL;
    std::vector<int32_t> seq_adapter(B, -1);
    if (!replay) {
        if (mb) {
            const int A = (int)c->plan->adapters.size();
            for (int b = 0; b < B; ++b) {
                const int a = adapter_of_seq ? adapter_of_seq[b] : b % A;
                if (a < 0 || a >= A) return fail(PB_EINVAL, "adapter_of_seq[%d] = %d out of range", b, a);
                seq_adapter[b] = a;
            }
        } else if (adapter_of_seq) {
            for (int b = 0; b < B; ++b)
                if (adapter_of_seq[b] != c->merge_adapter)
                    return fail(PB_EINVAL, "sequence %d asks for adapter %d but the in-place merge holds %d (use "
                                           "PB_MERGE_ALL for mixed batches)", b, adapter_of_seq[b], c->merge_adapter);
        }
    }
    std::unique_lock<std::mutex> lk(c->run_mu);
    if (replay || !c->run) {   // replay / decode: a fresh run with nothing to load
        lk.unlock();
        join_load(c);
        lk.lock();
        c->issue_status = PB_OK;
        c->issue_msg[0] = '\0';
        c->run = init_run(c, replay);
        c->posted.store(false);
    }
    // The issuer reads the staged prompt only after `posted` is set (release below), so staging it here is safe
    // while a cold start's loads are being issued.
    if (!replay) c->seq_adapter = seq_adapter;
    if (c->rank == 0 || c->replica)
        for (int b = 0; b < B; ++b)   // token-major rows t*B + b; microbatch mode: sequence-major b*T + t
            for (int t = 0; t < T; ++t) c->h_tokens[mb ? b * T + t : t * B + b] = tokens[(size_t)b * T + t];
    c->cur_batch = B;
    c->cur_seq = T;
    c->n_decoded = 0;
    c->prompt_replica = c->replica;
    c->phase = Phase::Prefilled;
    c->posted.store(true, std::memory_order_release);
    if (c->load_thread.joinable() && !c->loader_idle) return PB_OK;   // the running issuer picks the prompt up
    lk.unlock();
    join_load(c);
    if (c->issue_status != PB_OK) return fail(c->issue_status, "issuer: %s", c->issue_msg);
    spawn_issuer(c);
    return PB_OK;
}

}  // namespace

extern "C" pb_status pb_prefill_enqueue(pb_ctx* c, const int32_t* tokens, int32_t B, int32_t T) {
    pb_status st = check_ctx(c, "pb_prefill_enqueue");
    if (st) return st;
    if (c->phase != Phase::Gathered) return fail(PB_EPROTOCOL, "pb_prefill_enqueue: call pb_gather_layers first");
    return start_issuer(c, tokens, nullptr, B, T, false);
}

extern "C" pb_status pb_prefill_enqueue_ex(pb_ctx* c, const int32_t* tokens, const int32_t* adapter_of_seq, int32_t B,
                                           int32_t T) {
    pb_status st = check_ctx(c, "pb_prefill_enqueue_ex");
    if (st) return st;
    if (c->phase != Phase::Gathered) return fail(PB_EPROTOCOL, "pb_prefill_enqueue_ex: call pb_gather_layers first");
    return start_issuer(c, tokens, adapter_of_seq, B, T, false);
}

extern "C" pb_status pb_prefill_replay(pb_ctx* c, uint32_t epoch, const int32_t* tokens, int32_t B, int32_t T) {
    pb_status st = check_ctx(c, "pb_prefill_replay");
    if (st) return st;
    if (c->phase != Phase::Prefilled && c->phase != Phase::Gathered)
        return fail(PB_EPROTOCOL, "pb_prefill_replay: needs a completed cold start");
    if (epoch <= c->epoch) return fail(PB_EINVAL, "epoch %u must exceed the previous %u", epoch, c->epoch);
    join_load(c);
    if (c->phase == Phase::Gathered) {   // a cold start without a prompt: serve once it has reached T_full
        if (c->issue_status != PB_OK) return fail(c->issue_status, "issuer: %s", c->issue_msg);
        if (cudaEventQuery(c->gather_done) != cudaSuccess || cudaEventQuery(c->merge_done) != cudaSuccess) {
            cudaGetLastError();
            return fail(PB_EPROTOCOL, "pb_prefill_replay: the armed cold start has not reached T_full (pb_sync first)");
        }
    }
    CU(cudaStreamSynchronize(c->comp));
    c->epoch = epoch;
    c->n_launches = 0;
    c->prof_n = 0;
    if ((c->n == 1 || c->replica) && c->merge_adapter != PB_MERGE_ALL) {
        // Single rank: the replay has no cross-rank waits, so it is captured once as a CUDA graph and relaunched
        // (the token upload / result download are graph nodes on the pinned staging buffers).
        if (B < 1 || T < 1 || B > c->L.max_batch || T > c->L.max_seq || (int64_t)B * T > c->L.max_rows)
            return fail(PB_EINVAL, "batch %d x seq %d exceeds the workspace", B, T);
        if (!tokens) return fail(PB_EINVAL, "rank 0 (every rank of a replica) needs tokens");
        for (int64_t i = 0; i < (int64_t)B * T; ++i)
            if (tokens[i] < 0 || tokens[i] >= c->plan->model.vocab)
                return fail(PB_EINVAL, "token %d at [%lld] outside the vocabulary [0, %d)", tokens[i], (long long)i,
                            c->plan->model.vocab);
        for (int b = 0; b < B; ++b)
            for (int t = 0; t < T; ++t) c->h_tokens[t * B + b] = tokens[(size_t)b * T + t];
        c->cur_batch = B;
        c->cur_seq = T;
        c->n_decoded = 0;
        c->prompt_replica = c->replica;
        const int pi = c->profiling ? 1 : 0, rp = c->replica ? 1 : 0;
        pb_ctx::ReplayGraph* rg = nullptr;
        for (auto& g : c->replay_graphs)
            if (g.B == B && g.T == T && g.profiled == pi && g.replica == rp) rg = &g;
        if (!rg) {
            CU(cudaStreamBeginCapture(c->comp, cudaStreamCaptureModeThreadLocal));
            c->capturing = true;
            pb_status ist = issue_trial(c, B, T, true);
            c->capturing = false;
            cudaGraph_t g = nullptr;
            cudaError_t ce = cudaStreamEndCapture(c->comp, &g);
            if (ist != PB_OK) {
                if (g) cudaGraphDestroy(g);
                return ist;
            }
            CU(ce);
            cudaGraphExec_t ge = nullptr;
            cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            CU(ie);
            c->replay_graphs.push_back({B, T, pi, rp, ge, c->n_launches, c->prof_n,
                                        std::vector<ProfRec>(c->prof.begin(), c->prof.begin() + c->prof_n)});
            rg = &c->replay_graphs.back();
        }
        c->n_launches = rg->launches;
        c->prof_n = rg->prof_n;
        for (size_t i = 0; i < rg->prof_n; ++i) c->prof[i] = rg->prof[i];
        c->issue_status = PB_OK;
        c->phase = Phase::Prefilled;
        CU(cudaEventRecord(c->t0, c->comp));
        CU(cudaGraphLaunch(rg->exec, c->comp));
        return PB_OK;
    }
    CU(cudaEventRecord(c->t0, c->comp));
    return start_issuer(c, tokens, nullptr, B, T, true);
}

// ------------------------------------------------------------------------------------------------
// f3 — pipelined decode and the switch to single-GPU replicas
// ------------------------------------------------------------------------------------------------
extern "C" pb_status pb_decode_step(pb_ctx* c, uint32_t epoch) {
    pb_status st = check_ctx(c, "pb_decode_step");
    if (st) return st;
    if (c->phase != Phase::Prefilled) return fail(PB_EPROTOCOL, "pb_decode_step: needs a prefilled batch");
    if (c->merge_adapter == PB_MERGE_ALL)
        return fail(PB_EUNSUPPORTED, "pb_decode_step: PB_MERGE_ALL microbatches (decode one adapter per batch)");
    if (epoch <= c->epoch) return fail(PB_EINVAL, "epoch %u must exceed the previous %u", epoch, c->epoch);
    if (c->prompt_replica != c->replica)
        return fail(PB_EPROTOCOL, "pb_decode_step: the batch was prefilled in the other mode (pipeline / replica); "
                                  "prefill it again in this mode first (P:L295: batches after the switch)");
    const int32_t t = c->cur_seq + c->n_decoded;
    if (t >= c->L.max_seq) return fail(PB_EINVAL, "decode position %d reaches the workspace's max_seq %d", t, c->L.max_seq);
    join_load(c);
    if (c->issue_status != PB_OK) return fail(c->issue_status, "%s", c->issue_msg);
    CU(cudaStreamSynchronize(c->comp));
    c->epoch = epoch;
    c->n_launches = 0;
    c->prof_n = 0;
    c->n_decoded++;
    const int B = c->cur_batch;
    const int hd = c->plan->head_dim();
    if ((c->n == 1 || c->replica) && !c->plan->f32() && (hd == 64 || hd == 128)) {
        // Single GPU (or a replica): the step is a CUDA graph captured once per batch size; the position is a
        // device word filled from a pinned host word by the graph's first node, so every step relaunches it.
        pb_ctx::DecodeGraph* dg = nullptr;
        for (auto& g : c->decode_graphs)
            if (g.B == B) dg = &g;
        if (!dg) {
            const int saved = c->n_launches;
            CU(cudaStreamBeginCapture(c->comp, cudaStreamCaptureModeThreadLocal));
            c->capturing = true;
            c->decode_t = 0;
            c->dyn_pos = reinterpret_cast<const int*>(c->ws + c->L.dpos);
            pb_status ist = issue_trial(c, B, 1, true);
            c->capturing = false;
            c->decode_t = -1;
            c->dyn_pos = nullptr;
            cudaGraph_t g = nullptr;
            cudaError_t ce = cudaStreamEndCapture(c->comp, &g);
            if (ist != PB_OK) {
                if (g) cudaGraphDestroy(g);
                return ist;
            }
            CU(ce);
            cudaGraphExec_t ge = nullptr;
            cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            CU(ie);
            c->decode_graphs.push_back({B, ge, c->n_launches - saved});
            dg = &c->decode_graphs.back();
        }
        c->n_launches = dg->launches;
        *c->h_pos = t;
        c->issue_status = PB_OK;
        CU(cudaEventRecord(c->t0, c->comp));
        CU(cudaGraphLaunch(dg->exec, c->comp));
        return PB_OK;
    }
    CU(cudaEventRecord(c->t0, c->comp));
    c->issue_status = PB_OK;
    c->issue_msg[0] = '\0';
    c->load_thread = std::thread([c, B, t]() {
        cudaSetDevice(c->device);
        c->decode_t = t;
        pb_status ist = issue_trial(c, B, t + 1, true);
        c->decode_t = -1;
        if (ist != PB_OK) {
            c->issue_status = ist;
            snprintf(c->issue_msg, sizeof c->issue_msg, "%s", pb_last_error());
        }
    });
    return PB_OK;
}

extern "C" pb_status pb_ctx_set_replica(pb_ctx* c, int32_t on) {
    pb_status st = check_ctx(c, "pb_ctx_set_replica");
    if (st) return st;
    if (on) {
        if (c->phase != Phase::Prefilled) return fail(PB_EPROTOCOL, "pb_ctx_set_replica: needs a completed cold start");
        join_load(c);
        // T_full: every merge and every receive copy of the cold start has completed on this GPU
        if (cudaStreamQuery(c->merge) != cudaSuccess || cudaStreamQuery(c->nv) != cudaSuccess ||
            cudaEventQuery(c->gather_done) != cudaSuccess || cudaEventQuery(c->merge_done) != cudaSuccess)
            return fail(PB_EPROTOCOL, "pb_ctx_set_replica: T_full not reached (pb_sync first)");
        if (c->merge_adapter == PB_MERGE_ALL) return fail(PB_EUNSUPPORTED, "replica of a PB_MERGE_ALL context");
        // a replica runs every layer from this GPU's weights: the other stages' gathered copies hold the cold
        // start's adapter, so the stage (pb_switch_adapter) must hold it too
        if (c->merge_adapter != c->cold_adapter)
            return fail(PB_EUNSUPPORTED, "pb_ctx_set_replica: the stage was switched to adapter %d but the gathered "
                                         "layers hold the cold start's adapter %d", c->merge_adapter, c->cold_adapter);
    }
    c->replica = on != 0;
    return PB_OK;
}

// ------------------------------------------------------------------------------------------------
// f2 — epoch-based adapter switching
// ------------------------------------------------------------------------------------------------
extern "C" pb_status pb_switch_adapter(pb_ctx* c, int32_t adapter_id) {
    pb_status st = check_ctx(c, "pb_switch_adapter");
    if (st) return st;
    const pb_plan* p = c->plan;
    if (c->phase != Phase::Prefilled) return fail(PB_EPROTOCOL, "pb_switch_adapter: needs a completed cold start");
    if (c->merge_adapter == PB_MERGE_ALL)
        return fail(PB_EUNSUPPORTED, "pb_switch_adapter: PB_MERGE_ALL already holds every adapter (per-sequence)");
    if (adapter_id < -1 || adapter_id >= (int32_t)p->adapters.size())
        return fail(PB_EINVAL, "adapter_id %d out of range", adapter_id);
    if (!c->backup) return fail(PB_ENOMEM, "pb_switch_adapter needs bufs.backup >= dev_backup_bytes");
    if (!p->survivors.empty()) return fail(PB_EUNSUPPORTED, "pb_switch_adapter on a re-plan");
    if (c->replica)
        return fail(PB_EUNSUPPORTED, "pb_switch_adapter in replica mode (only the stage would switch; the gathered "
                                     "layers keep the cold start's adapter)");
    join_load(c);   // the trial issuer has issued everything: the switch queues behind it on the compute stream
    if (c->issue_status != PB_OK) return fail(c->issue_status, "%s", c->issue_msg);
    cudaStream_t s = c->comp;
    // the stage is rewritten in place: every peer must have finished copying it first (device-side wait on the
    // peers' gather-complete words, so the switch cannot tear a copy still in flight)
    // (peers signal it in their cold start's epoch; replays and decode steps gather nothing and do not signal)
    for (int r = 0; r < c->n; ++r)
        if (r != c->rank) CU(stream_wait_geq(s, flag_ptr(c->ws, c->L, c->L.f_gdone + r), c->cold_epoch));
    const auto stage = p->stages[c->rank];
    const char* hb = static_cast<const char*>(c->host_base);
    const char* ha = static_cast<const char*>(c->host_adapters);
    auto in_stage = [&](int32_t t) { return p->tensors[t].layer >= stage.first && p->tensors[t].layer < stage.second; };
    // 1. restore the pristine base of every adapted tensor of the stage: from the copy saved by this rank's
    //    cold-start merge where it loaded the chunk, else from the host image
    for (const ChunkRec& ch : p->chunks) {
        if (ch.is_adapter || !in_stage(ch.tensor) || p->backup_off[ch.tensor] < 0) continue;
        if (c->in_load[ch.id]) {
            CU(launch_copy(c->weights + ch.dev_off,
                           c->backup + p->backup_off[ch.tensor] + (int64_t)ch.r0 * p->tensors[ch.tensor].row_bytes(),
                           ch.bytes, s));
            ++c->n_launches;
        } else {
            CU(cudaMemcpyAsync(c->weights + ch.dev_off, hb + ch.host_off, ch.bytes, cudaMemcpyHostToDevice, s));
        }
    }
    // 2. merge the new adapter in place (factors this rank did not load come from the host image)
    if (adapter_id >= 0) {
        for (const ChunkRec& ch : p->chunks)
            if (ch.is_adapter && p->atensors[ch.tensor].adapter == adapter_id && in_stage(p->atensors[ch.tensor].base) &&
                !c->in_load[ch.id])
                CU(cudaMemcpyAsync(c->adapters + ch.dev_off, ha + ch.host_off, ch.bytes, cudaMemcpyHostToDevice, s));
        char err[512];
        for (const MergeRec& mr : p->merges) {
            if (mr.adapter != adapter_id || !in_stage(mr.base)) continue;
            const TensorRec& bt = p->tensors[mr.base];
            const ATensorRec& A = p->atensors[mr.a_tensor];
            const ATensorRec& Bf = p->atensors[mr.b_tensor];
            const int rank = p->adapters[adapter_id].rank;
            const float scale = p->adapters[adapter_id].alpha / (float)rank;
            char* W = c->weights + bt.dev_off + (int64_t)mr.row0 * bt.row_bytes();
            if (p->f32()) {
                CU(launch_merge_f32(reinterpret_cast<const float*>(W), reinterpret_cast<float*>(W), bt.cols, mr.rows,
                                    mr.cols, reinterpret_cast<const float*>(c->adapters + Bf.off),
                                    reinterpret_cast<const float*>(c->adapters + A.off), rank, scale, s));
            } else {
                MergeMaps maps;
                if (!make_merge_maps(&maps, W, bt.cols, mr.rows, mr.cols, c->adapters + Bf.off, c->adapters + A.off,
                                     rank, err, sizeof err))
                    return fail(PB_EINVAL, "merge map: %s", err);
                CU(launch_merge(maps, mr.rows, mr.cols, rank, scale, s));
            }
            ++c->n_launches;
        }
    }
    c->merge_adapter = adapter_id;
    return PB_OK;
}

extern "C" pb_status pb_prefill_wait(pb_ctx* c, float* logits_out, int32_t* tokens_out) {
    NvtxRange nv("pb_prefill_wait");
    pb_status st = check_ctx(c, "pb_prefill_wait");
    if (st) return st;
    if (c->phase != Phase::Prefilled) return fail(PB_EPROTOCOL, "pb_prefill_wait: nothing enqueued");
    join_load(c);
    if (c->issue_status != PB_OK) return fail(c->issue_status, "issuer: %s", c->issue_msg);
    // Optional watchdog (PB_WAIT_TIMEOUT_S): poll instead of blocking; on timeout report which streams are
    // stuck and which readiness words are still below the epoch, and return PB_ECUDA instead of hanging.
    static const char* wt_env = getenv("PB_WAIT_TIMEOUT_S");
    if (wt_env) {
        const double limit = atof(wt_env);
        const auto t_start = std::chrono::steady_clock::now();
        for (;;) {
            cudaError_t q = cudaEventQuery(c->done);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) CU(q);
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count() > limit) {
                cudaStream_t ss[] = {c->h2d[0], c->merge, c->nv, c->comp};
                const char* nm[] = {"h2d", "merge", "nvlink", "compute"};
                char msg[1024];
                int o = snprintf(msg, sizeof msg, "rank %d: prefill not done after %.0f s; streams:", c->rank, limit);
                for (int i = 0; i < 4; ++i)
                    o += snprintf(msg + o, sizeof msg - o, " %s=%s", nm[i],
                                  cudaStreamQuery(ss[i]) == cudaSuccess ? "idle" : "busy");
                std::vector<uint32_t> w(c->L.n_words);
                cudaStream_t probe;
                if (cudaStreamCreateWithFlags(&probe, cudaStreamNonBlocking) == cudaSuccess) {
                    cudaMemcpyAsync(w.data(), c->ws + c->L.flags, 4 * w.size(), cudaMemcpyDeviceToHost, probe);
                    cudaStreamSynchronize(probe);
                    cudaStreamDestroy(probe);
                    auto dump = [&](const char* name, int32_t lo, int32_t hi) {
                        int shown = 0, low = 0;
                        for (int32_t i = lo; i < hi; ++i)
                            if (w[i] < c->epoch) {
                                ++low;
                                if (shown < 6) o += snprintf(msg + o, sizeof msg - o, "%s%d", shown++ ? "," : " ", i - lo);
                            }
                        o += snprintf(msg + o, sizeof msg - o, " (%s: %d below epoch)", name, low);
                    };
                    o += snprintf(msg + o, sizeof msg - o, "; words below epoch %u:", c->epoch);
                    dump("chunk", c->L.f_chunk, c->L.f_act);
                    dump("act", c->L.f_act, c->L.f_y);
                    dump("y", c->L.f_y, c->L.f_logit);
                    dump("logit", c->L.f_logit, c->L.f_land);
                    dump("tensor", c->L.f_tensor, c->L.n_words);
                }
                return fail(PB_ECUDA, "%s", msg);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(200));
        }
    }
    CU(cudaEventSynchronize(c->done));
    CU(cudaGetLastError());
    if (c->rank == 0 || c->replica) {
        const int B = c->cur_batch;
        if (tokens_out) memcpy(tokens_out, c->h_out, sizeof(int32_t) * B);
        if (logits_out)
            CU(cudaMemcpy(logits_out, c->ws + c->L.logits, sizeof(float) * B * c->plan->model.vocab,
                          cudaMemcpyDeviceToHost));
        if (c->h_out[B]) return fail(PB_ENUMERIC, "non-finite logits");
    }
    return PB_OK;
}

extern "C" pb_status pb_prefill_first_token(pb_ctx* c, const int32_t* tokens, int32_t B, int32_t T, float* logits_out,
                                            int32_t* tokens_out) {
    pb_status st = pb_prefill_enqueue(c, tokens, B, T);
    if (st) return st;
    return pb_prefill_wait(c, logits_out, tokens_out);
}

extern "C" pb_status pb_sync(pb_ctx* c) {
    pb_status st = check_ctx(c, "pb_sync");
    if (st) return st;
    join_load(c);
    if (c->issue_status != PB_OK) return fail(c->issue_status, "issuer: %s", c->issue_msg);
    cudaStream_t ss[] = {c->h2d[0], c->h2d[1], c->merge, c->nv, c->comp};
    for (auto s : ss) CU(cudaStreamSynchronize(s));
    CU(cudaGetLastError());
    return PB_OK;
}

extern "C" pb_status pb_ctx_abort(pb_ctx* c) {
    pb_status st = check_ctx(c, "pb_ctx_abort");
    if (st) return st;
    c->abort_req.store(true);
    join_load(c);   // the issuer returns at its next poll (it never blocks in an enqueue: outstanding-op budgets)
    // force every readiness word of this rank open. CU_STREAM_WAIT_VALUE_GEQ compares cyclically,
    // (int32_t)(word - epoch) >= 0, so the words get epoch + 2^30 (0xFFFFFFFF would read as "before" the epoch)
    // on the ctx's spare lane (stream_h2d[1]): it never waits on a readiness word and owns its hardware queue (a
    // freshly created stream could share a queue with a blocked one and sit behind the very wait it must release)
    const std::vector<uint32_t> open_words((size_t)c->L.n_words, c->epoch + 0x40000000u);
    cudaError_t e = cudaMemcpyAsync(c->ws + c->L.flags, open_words.data(), 4 * open_words.size(),
                                    cudaMemcpyHostToDevice, c->h2d[1]);
    if (e == cudaSuccess) e = drain_stream(c->h2d[1], 10.0) ? cudaSuccess : cudaErrorNotReady;
    c->aborted = true;
    c->phase = Phase::Idle;
    CU(e);
    return PB_OK;
}

extern "C" pb_status pb_timeline(pb_ctx* c, pb_timeline_t* out) {
    pb_status st = check_ctx(c, "pb_timeline");
    if (st) return st;
    if (!out) return fail(PB_EINVAL, "pb_timeline: null out");
    if (c->phase == Phase::Idle) return fail(PB_EPROTOCOL, "pb_timeline: no trial");
    const pb_plan* p = c->plan;
    auto ms = [&](cudaEvent_t e) -> double {
        float v = 0;
        if (!e || cudaEventElapsedTime(&v, c->t0, e) != cudaSuccess) { cudaGetLastError(); return -1; }
        return v;
    };
    double load_done = c->copies.empty() ? 0 : ms(c->load_end);
    for (int32_t id : p->load[c->rank]) {
        c->tl_landed[id] = c->landed_timing ? ms(landed_ev(c, id)) : -1;
        load_done = std::max(load_done, c->tl_landed[id]);
    }
    for (int32_t id : p->recv[c->rank]) c->tl_gathered[id] = ms(c->gathered[id]);
    for (int32_t id : p->load[c->rank]) c->tl_merged[id] = c->merged_ev[id] ? ms(c->merged_ev[id]) : -1;
    double ready = 0;
    if (c->last_own_stage_chunk >= 0) ready = std::max(ready, ms(c->ready_merge));
    if (c->last_recv_stage_chunk >= 0) ready = std::max(ready, ms(c->ready_recv));
    out->t_ready_ms = ready;
    out->t_full_ms = std::max(ms(c->merge_done), ms(c->gather_done));
    out->ttft_ms = c->phase == Phase::Prefilled ? ms(c->done) : -1;
    out->load_done_ms = load_done;
    out->load_bytes = c->load_bytes;
    out->recv_bytes = c->recv_bytes;
    out->n_chunks = (int32_t)p->chunks.size();
    out->chunk_landed_ms = c->tl_landed.data();
    out->chunk_gathered_ms = c->tl_gathered.data();
    out->n_launches = c->n_launches;
    out->chunk_merged_ms = c->tl_merged.data();
    const bool staged = c->phase == Phase::Prefilled && p->stages[c->rank].second > p->stages[c->rank].first;
    out->stage_begin_ms = staged ? ms(c->stage_begin) : -1;
    out->stage_end_ms = staged ? ms(c->stage_end) : -1;
    out->ctx_create_ms = c->ctx_create_ms;
    return PB_OK;
}
