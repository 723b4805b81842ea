// plan.cpp — pb_plan_create / pb_plan_dump: the PipeBoost load planner (host, pure).
//
// Follows the paper's statement of layer-partitioned loading:
//   P:L234-236  split the checkpoint into N parts, GPU g loads part g ("GPU 0 reads A-0 while GPU 1 reads A-1")
//   P:L244-245  adapters partitioned the same way; GPU g loads part g of every adapter
//   P:L353-357  Load Balance / Layer Contiguity -> contiguous balanced stages, remainder to lower g
//   P:L360-361  rotation order "GPU 3 loads 3, 0, 1 and 2" -> receive list (g+i) mod N after own part
// and the readings recorded in DESIGN.md §3 (fused qkv/gate_up tensors, 4 KiB alignment,
// 128-row chunk granularity, INTERLEAVE policy, vocab slicing).
#include <algorithm>
#include <array>
#include <cinttypes>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <set>
#include <unordered_map>

#include "errors.hpp"
#include "plan.hpp"

using namespace pb;

namespace {

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Shape { const char* sfx; int64_t rows, cols; };

std::vector<Shape> layer_shapes(const pb_model_desc& m) {
    const int64_t d = m.d_model, f = m.d_ffn, hd = m.d_model / m.n_heads;
    // Compute order (norm, qkv, o, norm, mlp): a layer's kernels can start as its tensors land.
    if (m.arch == PB_ARCH_OPT)
        return {{"ln1_g", 1, d}, {"ln1_b", 1, d}, {"qkv", 3 * d, d}, {"qkv_b", 1, 3 * d}, {"o", d, d},
                {"o_b", 1, d}, {"ln2_g", 1, d}, {"ln2_b", 1, d}, {"fc1", f, d}, {"fc1_b", 1, f},
                {"fc2", d, f}, {"fc2_b", 1, d}};
    const int64_t qkv = (int64_t)(m.n_heads + 2 * m.n_kv_heads) * hd;
    return {{"ln1_g", 1, d}, {"qkv", qkv, d}, {"o", d, (int64_t)m.n_heads * hd}, {"ln2_g", 1, d},
            {"gate_up", 2 * f, d}, {"down", d, f}};
}

// Target geometry: base suffix, first base row, out features, in features.
struct Geo { const char* base; int64_t row0, out, in; };

const int kOptTargets[] = {PB_T_Q, PB_T_K, PB_T_V, PB_T_O, PB_T_FC1, PB_T_FC2};
const int kLlamaTargets[] = {PB_T_Q, PB_T_K, PB_T_V, PB_T_O, PB_T_GATE, PB_T_UP, PB_T_DOWN};

const char* target_name(int bit) {
    switch (bit) {
        case PB_T_Q: return "q"; case PB_T_K: return "k"; case PB_T_V: return "v"; case PB_T_O: return "o";
        case PB_T_FC1: return "fc1"; case PB_T_FC2: return "fc2"; case PB_T_GATE: return "gate";
        case PB_T_UP: return "up"; case PB_T_DOWN: return "down";
    }
    return "?";
}

bool target_geo(const pb_model_desc& m, int bit, Geo* g) {
    const int64_t d = m.d_model, f = m.d_ffn, hd = m.d_model / m.n_heads;
    if (m.arch == PB_ARCH_OPT) {
        switch (bit) {
            case PB_T_Q: *g = {"qkv", 0, d, d}; return true;
            case PB_T_K: *g = {"qkv", d, d, d}; return true;
            case PB_T_V: *g = {"qkv", 2 * d, d, d}; return true;
            case PB_T_O: *g = {"o", 0, d, d}; return true;
            case PB_T_FC1: *g = {"fc1", 0, f, d}; return true;
            case PB_T_FC2: *g = {"fc2", 0, d, f}; return true;
        }
        return false;
    }
    const int64_t qd = (int64_t)m.n_heads * hd, kvd = (int64_t)m.n_kv_heads * hd;
    switch (bit) {
        case PB_T_Q: *g = {"qkv", 0, qd, d}; return true;
        case PB_T_K: *g = {"qkv", qd, kvd, d}; return true;
        case PB_T_V: *g = {"qkv", qd + kvd, kvd, d}; return true;
        case PB_T_O: *g = {"o", 0, d, qd}; return true;
        case PB_T_GATE: *g = {"gate_up", 0, f, d}; return true;
        case PB_T_UP: *g = {"gate_up", f, f, d}; return true;
        case PB_T_DOWN: *g = {"down", 0, d, f}; return true;
    }
    return false;
}

int32_t rows_per_chunk(int64_t row_bytes, int64_t chunk_bytes) {
    int64_t rpc = chunk_bytes / row_bytes;
    if (rpc < 1) rpc = 1;
    if (rpc >= 128) rpc -= rpc % 128;
    if (rpc > INT32_MAX) rpc = INT32_MAX;
    return (int32_t)rpc;
}

// Balanced contiguous split of n items into p parts, remainder to the lower parts.
std::vector<std::pair<int32_t, int32_t>> balanced(int32_t n, int32_t p) {
    std::vector<std::pair<int32_t, int32_t>> out;
    int32_t base = n / p, rem = n % p, s = 0;
    for (int32_t g = 0; g < p; ++g) {
        int32_t size = base + (g < rem ? 1 : 0);
        out.push_back({s, s + size});
        s += size;
    }
    return out;
}

}  // namespace

int32_t pb_plan::stage_of_layer(int32_t l) const {
    for (int32_t g = 0; g < (int32_t)stages.size(); ++g)
        if (stages[g].first <= l && l < stages[g].second) return g;
    return -1;
}

int32_t pb_plan::find_tensor(const std::string& name) const {
    auto it = name_index.find(name);
    return it == name_index.end() ? -1 : it->second;
}

static int32_t layer_loader(const pb_plan* p, int32_t l) {
    return p->opts.policy == PB_LOAD_STAGE ? p->stage_of_layer(l) : l % p->n_gpus;
}

// Chunk ids in the canonical load order (G8): the non-layer tensors before the first layer, then every adapter
// chunk in atensor order (= host layout order: adapter, layer, target, A then B), then the layers' base tensors and
// the remaining non-layer tensors, each tensor's chunks in row order. base_chunks / ad_chunks: per (a)tensor.
static std::vector<int32_t> canonical_order(const pb_plan* p, const std::vector<std::vector<int32_t>>& base_chunks,
                                            const std::vector<std::vector<int32_t>>& ad_chunks) {
    std::vector<int32_t> order;
    bool adapters_done = false;
    for (size_t ti = 0; ti < p->tensors.size(); ++ti) {
        if (p->tensors[ti].layer >= 0 && !adapters_done) {
            for (size_t ai = 0; ai < p->atensors.size(); ++ai)
                order.insert(order.end(), ad_chunks[ai].begin(), ad_chunks[ai].end());
            adapters_done = true;
        }
        order.insert(order.end(), base_chunks[ti].begin(), base_chunks[ti].end());
    }
    return order;
}

extern "C" pb_status pb_plan_create(const pb_model_desc* model, const pb_adapter_desc* adapters,
                                    int32_t n_adapters, int32_t n_gpus, const pb_plan_opts* opts,
                                    pb_plan** out) {
    PB_TRY_BEGIN
    if (!model || !opts || !out) return pb::fail(PB_EINVAL, "pb_plan_create: null argument");
    *out = nullptr;
    const pb_model_desc& m = *model;
    if (m.arch != PB_ARCH_OPT && m.arch != PB_ARCH_LLAMA) return pb::fail(PB_EINVAL, "bad arch");
    if (m.n_layers < 1 || m.d_model < 1 || m.n_heads < 1 || m.n_kv_heads < 1 || m.d_ffn < 1 || m.vocab < 1)
        return pb::fail(PB_EINVAL, "model dimensions must be >= 1");
    if (m.d_model % m.n_heads || m.n_heads % m.n_kv_heads)
        return pb::fail(PB_EINVAL, "d_model %% n_heads and n_heads %% n_kv_heads must be 0");
    if (m.arch == PB_ARCH_OPT && (m.n_kv_heads != m.n_heads || m.max_pos < 1))
        return pb::fail(PB_EINVAL, "OPT needs n_kv_heads == n_heads and max_pos >= 1");
    if (m.arch == PB_ARCH_LLAMA && m.tied) return pb::fail(PB_EUNSUPPORTED, "tied Llama head");
    if (m.dtype != PB_DTYPE_BF16 && m.dtype != PB_DTYPE_F32) return pb::fail(PB_EINVAL, "dtype %d", m.dtype);
    if (n_gpus < 1 || n_gpus > kMaxGpus) return pb::fail(PB_EINVAL, "n_gpus must be in [1, 8]");
    if (n_gpus > m.n_layers) return pb::fail(PB_EPARTITION, "n_gpus %d > n_layers %d", n_gpus, m.n_layers);
    if (n_adapters < 0 || (n_adapters > 0 && !adapters)) return pb::fail(PB_EINVAL, "bad adapters");
    if (opts->policy != PB_LOAD_STAGE && opts->policy != PB_LOAD_INTERLEAVE) return pb::fail(PB_EINVAL, "bad policy");
    if (opts->chunk_bytes < 2 || opts->prefill_chunks < 1 || opts->host_alias_layers < 0)
        return pb::fail(PB_EINVAL, "bad opts");
    const int valid_mask = m.arch == PB_ARCH_OPT ? 63 : (PB_T_Q | PB_T_K | PB_T_V | PB_T_O | PB_T_GATE | PB_T_UP | PB_T_DOWN);
    for (int a = 0; a < n_adapters; ++a) {
        if (adapters[a].rank < 1) return pb::fail(PB_EINVAL, "adapter %d: rank < 1", a);
        if (adapters[a].rank > 64) return pb::fail(PB_EUNSUPPORTED, "adapter %d: rank > 64", a);
        if (!(adapters[a].alpha == adapters[a].alpha)) return pb::fail(PB_EINVAL, "adapter %d: alpha NaN", a);
        if (adapters[a].targets & ~valid_mask) return pb::fail(PB_EINVAL, "adapter %d: target not in this arch", a);
    }

    auto* p = new pb_plan();
    p->model = m;
    p->adapters.assign(adapters, adapters + n_adapters);
    p->n_gpus = n_gpus;
    p->opts = *opts;
    const int32_t L = m.n_layers, N = n_gpus, K = opts->host_alias_layers;

    // Step 1: stages.
    p->stages = balanced(L, N);

    // Step 2: base tensor table.
    struct Pending { std::string name; int64_t rows, cols; int32_t layer; };
    std::vector<Pending> names;
    names.push_back({"embed", m.vocab, m.d_model, -1});
    if (m.arch == PB_ARCH_OPT) names.push_back({"pos", (int64_t)m.max_pos + 2, m.d_model, -1});
    auto ls = layer_shapes(m);
    for (int32_t l = 0; l < L; ++l)
        for (auto& s : ls) names.push_back({"L" + std::to_string(l) + "." + s.sfx, s.rows, s.cols, l});
    names.push_back({"final_g", 1, m.d_model, -1});
    if (m.arch == PB_ARCH_OPT) {
        names.push_back({"final_b", 1, m.d_model, -1});
        if (!m.tied) names.push_back({"lm_head", m.vocab, m.d_model, -1});
    } else {
        names.push_back({"lm_head", m.vocab, m.d_model, -1});
    }
    int64_t dev = 0, host = 0;
    std::unordered_map<std::string, int32_t> idx;
    for (auto& n : names) {
        if (n.rows > INT32_MAX || n.cols > INT32_MAX) { delete p; return pb::fail(PB_EINVAL, "tensor too large"); }
        TensorRec t{n.name, (int32_t)n.rows, (int32_t)n.cols, n.layer, 0, 0, m.dtype == PB_DTYPE_F32 ? 4 : 2};
        dev = round_up(dev, kAlign);
        t.dev_off = dev;
        dev += t.bytes();
        if (K > 0 && n.layer >= K) {
            std::string src = "L" + std::to_string(n.layer % K) + "." + n.name.substr(n.name.find('.') + 1);
            t.host_off = p->tensors[idx.at(src)].host_off;
        } else {
            host = round_up(host, kAlign);
            t.host_off = host;
            host += t.bytes();
        }
        idx[t.name] = (int32_t)p->tensors.size();
        p->name_index[t.name] = (int32_t)p->tensors.size();
        p->tensors.push_back(t);
    }
    p->dev_weight_bytes = round_up(dev, kAlign);
    p->host_base_bytes = round_up(host, kAlign);

    // Adapter factor table: adapter, layer, target (canonical order), A then B.
    const int* tord = m.arch == PB_ARCH_OPT ? kOptTargets : kLlamaTargets;
    const int ntord = m.arch == PB_ARCH_OPT ? 6 : 7;
    int64_t aoff = 0;
    for (int32_t a = 0; a < n_adapters; ++a) {
        for (int32_t l = 0; l < L; ++l) {
            for (int ti = 0; ti < ntord; ++ti) {
                const int bit = tord[ti];
                if (!(adapters[a].targets & bit)) continue;
                Geo g{};
                target_geo(m, bit, &g);
                const int32_t base = idx.at("L" + std::to_string(l) + "." + g.base);
                MergeRec mr{a, l, bit, base, (int32_t)g.row0, (int32_t)g.out, (int32_t)g.in, 0, 0};
                for (int f = 0; f < 2; ++f) {
                    ATensorRec at;
                    at.name = "A" + std::to_string(a) + ".L" + std::to_string(l) + "." + target_name(bit) + (f ? ".B" : ".A");
                    at.rows = f ? (int32_t)g.out : adapters[a].rank;
                    at.cols = f ? adapters[a].rank : (int32_t)g.in;
                    at.layer = l; at.adapter = a; at.target_bit = bit; at.is_B = f;
                    at.base = base; at.row0 = (int32_t)g.row0;
                    at.es = m.dtype == PB_DTYPE_F32 ? 4 : 2;
                    aoff = round_up(aoff, kAlign);
                    at.off = aoff;
                    aoff += at.bytes();
                    (f ? mr.b_tensor : mr.a_tensor) = (int32_t)p->atensors.size();
                    p->atensors.push_back(at);
                }
                p->merges.push_back(mr);
            }
        }
    }
    p->host_adapter_bytes = round_up(aoff, kAlign);
    // Out-of-place copies for multi-adapter serving (not part of the canonical dump).
    {
        const size_t NT = p->tensors.size();
        p->adapted_off.assign(p->adapters.size() * NT, -1);
        int64_t off = 0;
        for (size_t a = 0; a < p->adapters.size(); ++a)
            for (auto& mr : p->merges)
                if (mr.adapter == (int32_t)a && p->adapted_off[a * NT + mr.base] < 0) {
                    off = round_up(off, kAlign);
                    p->adapted_off[a * NT + mr.base] = off;
                    off += p->tensors[mr.base].bytes();
                }
        p->dev_adapted_bytes = round_up(off, kAlign);
        // f2: pristine copy of every tensor some adapter modifies (one region, union over adapters), saved by
        // the cold-start merges so an adapter switch re-merges from the base (no bf16 drift across switches).
        p->backup_off.assign(NT, -1);
        off = 0;
        for (auto& mr : p->merges)
            if (p->backup_off[mr.base] < 0) {
                off = round_up(off, kAlign);
                p->backup_off[mr.base] = off;
                off += p->tensors[mr.base].bytes();
            }
        p->dev_backup_bytes = round_up(off, kAlign);
    }

    // Step 3: pieces -> chunks (global ids: base tensors in table order, then adapter factors).
    std::vector<std::vector<int32_t>> base_chunks(p->tensors.size()), ad_chunks(p->atensors.size());
    const bool sliced = opts->vocab_sliced != 0;
    for (size_t ti = 0; ti < p->tensors.size(); ++ti) {
        const TensorRec& t = p->tensors[ti];
        std::vector<std::array<int32_t, 3>> pcs;
        if (t.layer >= 0) pcs.push_back({0, t.rows, layer_loader(p, t.layer)});
        else if ((t.name == "embed" || t.name == "lm_head") && sliced) {
            auto sl = balanced(t.rows, N);
            for (int32_t g = 0; g < N; ++g) pcs.push_back({sl[g].first, sl[g].second, g});
        } else if (t.name == "embed" || t.name == "pos") pcs.push_back({0, t.rows, 0});
        else pcs.push_back({0, t.rows, N - 1});
        const int32_t rpc = rows_per_chunk(t.row_bytes(), opts->chunk_bytes);
        for (auto& pc : pcs) {
            for (int32_t r = pc[0]; r < pc[1];) {
                int32_t r1 = (int32_t)std::min<int64_t>(pc[1], (int64_t)r + rpc);
                ChunkRec c{(int32_t)p->chunks.size(), 0, (int32_t)ti, r, r1,
                           t.host_off + (int64_t)r * t.row_bytes(), t.dev_off + (int64_t)r * t.row_bytes(),
                           (int64_t)(r1 - r) * t.row_bytes(), pc[2]};
                base_chunks[ti].push_back(c.id);
                p->chunks.push_back(c);
                r = r1;
            }
        }
    }
    for (size_t ai = 0; ai < p->atensors.size(); ++ai) {
        const ATensorRec& at = p->atensors[ai];
        const int32_t rpc = rows_per_chunk(at.row_bytes(), opts->chunk_bytes);
        const int32_t g = layer_loader(p, at.layer);
        for (int32_t r = 0; r < at.rows;) {
            int32_t r1 = (int32_t)std::min<int64_t>(at.rows, (int64_t)r + rpc);
            ChunkRec c{(int32_t)p->chunks.size(), 1, (int32_t)ai, r, r1, at.off + (int64_t)r * at.row_bytes(),
                       at.off + (int64_t)r * at.row_bytes(), (int64_t)(r1 - r) * at.row_bytes(), g};
            ad_chunks[ai].push_back(c.id);
            p->chunks.push_back(c);
            r = r1;
        }
    }

    // Per-GPU load lists: canonical table order with every adapter factor right before the first layer tensor, in
    // host layout order (G8: a GPU's parts of one adapter are contiguous in host and device memory, so they cross
    // PCIe as one DMA instead of one small DMA per layer, and every adapted tensor can merge the moment it lands).
    p->load.assign(N, {});
    for (int32_t c : canonical_order(p, base_chunks, ad_chunks)) p->load[p->chunks[c].loader].push_back(c);

    // Step 4: receive lists. (1) base chunks of my stage's layers loaded elsewhere, in id order;
    // (2) for i = 1..N-1, loader (g+i) mod N's base chunks in its load order.
    p->recv.assign(N, {});
    for (int32_t g = 0; g < N; ++g) {
        std::vector<char> seen(p->chunks.size(), 0);
        auto& rv = p->recv[g];
        for (auto& c : p->chunks) {
            if (c.is_adapter || c.loader == g) continue;
            const int32_t l = p->tensors[c.tensor].layer;
            if (l >= p->stages[g].first && l < p->stages[g].second) { rv.push_back(c.id); seen[c.id] = 1; }
        }
        for (int32_t i = 1; i < N; ++i) {
            const int32_t q = (g + i) % N;
            for (int32_t c : p->load[q])
                if (!p->chunks[c].is_adapter && !seen[c]) { rv.push_back(c); seen[c] = 1; }
        }
    }
    // Step 5: adapter ownership own(g) = g mod A.
    for (int32_t g = 0; g < N; ++g) p->own.push_back(n_adapters ? g % n_adapters : -1);
    *out = p;
    return PB_OK;
    PB_TRY_END
}

// ------------------------------------------------------------------------------------------------
// f1 — recovery for model loading (§4.4.2). Steps R1-R6 as in oracle/plan.py
// replan(): survivors, balanced contiguous blocks, overlap-maximising block assignment (lexicographic
// first maximum over all m! assignments), sources, load lists (missing chunks only), receive lists.
// ------------------------------------------------------------------------------------------------
extern "C" pb_status pb_plan_replan(const pb_plan* plan, const int32_t* alive, const uint8_t* resident,
                                    pb_plan** out) {
    PB_TRY_BEGIN
    using namespace pb;
    if (!plan || !alive || !resident || !out) return pb::fail(PB_EINVAL, "pb_plan_replan: null argument");
    *out = nullptr;
    if (!plan->survivors.empty()) return pb::fail(PB_EUNSUPPORTED, "pb_plan_replan: re-planning a re-plan");
    const int32_t N = plan->n_gpus, L = plan->model.n_layers;
    const int32_t NC = (int32_t)plan->chunks.size();
    std::vector<int32_t> surv;
    for (int32_t g = 0; g < N; ++g)
        if (alive[g]) surv.push_back(g);
    const int32_t m = (int32_t)surv.size();
    if (m == 0) return pb::fail(PB_EINVAL, "pb_plan_replan: no surviving GPU");
    if (m > L) return pb::fail(PB_EPARTITION, "%d survivors > %d layers", m, L);
    const auto blocks = balanced(L, m);                                                // R2
    auto layer_of = [&](const ChunkRec& c) {
        return c.is_adapter ? plan->atensors[c.tensor].layer : plan->tensors[c.tensor].layer;
    };
    // R3: overlap[i][b] = bytes of block b's layer chunks survivor i holds
    std::vector<std::vector<int64_t>> ov(m, std::vector<int64_t>(m, 0));
    for (int32_t i = 0; i < m; ++i)
        for (const ChunkRec& c : plan->chunks) {
            if (c.is_adapter || !resident[(size_t)surv[i] * NC + c.id]) continue;
            const int32_t l = layer_of(c);
            if (l < 0) continue;
            for (int32_t b = 0; b < m; ++b)
                if (l >= blocks[b].first && l < blocks[b].second) ov[i][b] += c.bytes;
        }
    std::vector<int32_t> perm(m), best_perm;
    for (int32_t i = 0; i < m; ++i) perm[i] = i;
    int64_t best = -1;
    do {
        int64_t tot = 0;
        for (int32_t i = 0; i < m; ++i) tot += ov[i][perm[i]];
        if (tot > best) {
            best = tot;
            best_perm = perm;
        }
    } while (std::next_permutation(perm.begin(), perm.end()));
    std::vector<int32_t> gpu_of_rank(m);
    for (int32_t i = 0; i < m; ++i) gpu_of_rank[best_perm[i]] = surv[i];
    auto held = [&](int32_t r, int32_t c) { return resident[(size_t)gpu_of_rank[r] * NC + c] != 0; };
    auto block_rank = [&](int32_t l) {
        for (int32_t r = 0; r < m; ++r)
            if (l >= blocks[r].first && l < blocks[r].second) return r;
        return -1;
    };
    auto home_rank = [&](const ChunkRec& c) {
        const int32_t l = layer_of(c);
        if (l >= 0) return block_rank(l);
        const std::string& nm = plan->tensors[c.tensor].name;
        return (nm == "embed" || nm == "pos") ? 0 : m - 1;
    };

    auto* p = new pb_plan(*plan);
    p->n_gpus = m;
    p->opts.vocab_sliced = 0;
    p->stages = blocks;
    p->survivors = gpu_of_rank;
    p->resident.assign(m, std::vector<char>(NC, 0));
    for (int32_t r = 0; r < m; ++r)
        for (int32_t c = 0; c < NC; ++c) p->resident[r][c] = held(r, c) ? 1 : 0;
    // R4: sources
    std::vector<int32_t> src(NC, -1);
    for (const ChunkRec& c : plan->chunks) {
        if (c.is_adapter) continue;
        for (int32_t r = 0; r < m && src[c.id] < 0; ++r)
            if (held(r, c.id)) src[c.id] = r;
        if (src[c.id] < 0) src[c.id] = home_rank(c);
    }
    std::vector<std::vector<char>> need_ad(m, std::vector<char>(NC, 0));
    for (const ChunkRec& c : plan->chunks) {
        if (c.is_adapter || held(src[c.id], c.id)) continue;
        const int32_t r = src[c.id];
        for (size_t ai = 0; ai < plan->atensors.size(); ++ai) {
            if (plan->atensors[ai].base != c.tensor) continue;
            for (const ChunkRec& ac : plan->chunks)
                if (ac.is_adapter && ac.tensor == (int32_t)ai && !held(r, ac.id)) need_ad[r][ac.id] = 1;
        }
    }
    for (const ChunkRec& c : plan->chunks) {
        if (!c.is_adapter) continue;
        int32_t s = -1;
        for (int32_t r = 0; r < m && s < 0; ++r)
            if (need_ad[r][c.id]) s = r;
        for (int32_t r = 0; r < m && s < 0; ++r)
            if (held(r, c.id)) s = r;
        src[c.id] = s >= 0 ? s : home_rank(c);
    }
    for (ChunkRec& c : p->chunks) c.loader = src[c.id];
    // canonical order (pb_plan_create's load order): per layer, adapter parts then base tensors
    std::vector<std::vector<int32_t>> base_chunks(p->tensors.size()), ad_chunks(p->atensors.size());
    for (const ChunkRec& c : p->chunks) (c.is_adapter ? ad_chunks : base_chunks)[c.tensor].push_back(c.id);
    const std::vector<int32_t> order = canonical_order(p, base_chunks, ad_chunks);
    // R5: load lists
    p->load.assign(m, {});
    for (int32_t cid : order) {
        const ChunkRec& c = p->chunks[cid];
        if (!c.is_adapter) {
            if (!held(src[cid], cid)) p->load[src[cid]].push_back(cid);
        } else {
            for (int32_t r = 0; r < m; ++r)
                if (need_ad[r][cid]) p->load[r].push_back(cid);
        }
    }
    // R6: receive lists
    p->recv.assign(m, {});
    for (int32_t r = 0; r < m; ++r) {
        std::vector<char> have(NC, 0), seen(NC, 0);
        for (int32_t c = 0; c < NC; ++c) have[c] = held(r, c);
        for (int32_t c : p->load[r]) have[c] = 1;
        auto& rv = p->recv[r];
        for (int32_t cid : order) {
            const ChunkRec& c = p->chunks[cid];
            if (c.is_adapter || have[cid]) continue;
            const int32_t l = p->tensors[c.tensor].layer;
            if ((l >= blocks[r].first && l < blocks[r].second) || (l < 0 && home_rank(c) == r)) {
                rv.push_back(cid);
                seen[cid] = 1;
            }
        }
        for (int32_t k = 1; k < m; ++k) {
            const int32_t q = (r + k) % m;
            for (int32_t cid : order) {
                const ChunkRec& c = p->chunks[cid];
                if (!c.is_adapter && src[cid] == q && !have[cid] && !seen[cid]) {
                    rv.push_back(cid);
                    seen[cid] = 1;
                }
            }
        }
    }
    const int32_t A = (int32_t)p->adapters.size();
    p->own.clear();
    for (int32_t r = 0; r < m; ++r) p->own.push_back(A ? r % A : -1);
    *out = p;
    return PB_OK;
    PB_TRY_END
}

extern "C" pb_status pb_plan_gpu_of_rank(const pb_plan* p, int32_t rank, int32_t* gpu) {
    if (!p || !gpu) return pb::fail(PB_EINVAL, "pb_plan_gpu_of_rank: null argument");
    if (rank < 0 || rank >= p->n_gpus) return pb::fail(PB_EINVAL, "rank %d out of range", rank);
    *gpu = p->survivors.empty() ? rank : p->survivors[rank];
    return PB_OK;
}

namespace {
struct Out {
    std::string s;
    void f(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        int n = vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        if (n >= (int)sizeof buf) {
            std::string big(n + 1, '\0');
            va_start(ap, fmt);
            vsnprintf(&big[0], n + 1, fmt, ap);
            va_end(ap);
            big.resize(n);
            s += big;
        } else {
            s.append(buf, n);
        }
    }
};
}  // namespace

static std::string dump_string(const pb_plan* p) {
    Out o;
    const pb_model_desc& m = p->model;
    o.f("pipeboost-plan 1\n");
    o.f("model arch=%s layers=%d d_model=%d heads=%d kv_heads=%d d_ffn=%d vocab=%d max_pos=%d tied=%d dtype=%s\n",
        m.arch == PB_ARCH_OPT ? "opt" : "llama", m.n_layers, m.d_model, m.n_heads, m.n_kv_heads, m.d_ffn, m.vocab,
        m.max_pos, m.tied, m.dtype == PB_DTYPE_F32 ? "f32" : "bf16");
    o.f("gpus %d policy=%s vocab_sliced=%d chunk_bytes=%" PRId64 " prefill_chunks=%d host_alias_layers=%d\n", p->n_gpus,
        p->opts.policy == PB_LOAD_STAGE ? "stage" : "interleave", p->opts.vocab_sliced, p->opts.chunk_bytes,
        p->opts.prefill_chunks, p->opts.host_alias_layers);
    const int* tord = m.arch == PB_ARCH_OPT ? kOptTargets : kLlamaTargets;
    const int ntord = m.arch == PB_ARCH_OPT ? 6 : 7;
    for (size_t a = 0; a < p->adapters.size(); ++a) {
        std::string tg;
        for (int i = 0; i < ntord; ++i)
            if (p->adapters[a].targets & tord[i]) { if (!tg.empty()) tg += ","; tg += target_name(tord[i]); }
        o.f("adapter %zu rank=%d alpha=%.6f targets=%s\n", a, p->adapters[a].rank, (double)p->adapters[a].alpha, tg.c_str());
    }
    for (size_t g = 0; g < p->stages.size(); ++g)
        o.f("stage %zu layers=[%d,%d)\n", g, p->stages[g].first, p->stages[g].second);
    for (size_t i = 0; i < p->tensors.size(); ++i) {
        auto& t = p->tensors[i];
        o.f("tensor %zu %s rows=%d cols=%d layer=%d host_off=%" PRId64 " dev_off=%" PRId64 " bytes=%" PRId64 "\n", i,
            t.name.c_str(), t.rows, t.cols, t.layer, t.host_off, t.dev_off, t.bytes());
    }
    for (size_t i = 0; i < p->atensors.size(); ++i) {
        auto& t = p->atensors[i];
        o.f("atensor %zu %s rows=%d cols=%d layer=%d base=%d row0=%d off=%" PRId64 " bytes=%" PRId64 "\n", i,
            t.name.c_str(), t.rows, t.cols, t.layer, t.base, t.row0, t.off, t.bytes());
    }
    for (auto& c : p->chunks)
        o.f("chunk %d %s tensor=%d rows=[%d,%d) host_off=%" PRId64 " dev_off=%" PRId64 " bytes=%" PRId64 " loader=%d\n",
            c.id, c.is_adapter ? "adapter" : "base", c.tensor, c.r0, c.r1, c.host_off, c.dev_off, c.bytes, c.loader);
    for (int g = 0; g < p->n_gpus; ++g) {
        o.f("load %d:", g);
        for (int32_t c : p->load[g]) o.f(" %d", c);
        o.f("\n");
    }
    for (int g = 0; g < p->n_gpus; ++g) {
        o.f("recv %d:", g);
        for (int32_t c : p->recv[g]) o.f(" %d", c);
        o.f("\n");
    }
    for (int g = 0; g < p->n_gpus; ++g) o.f("own %d adapter=%d\n", g, p->own[g]);
    if (!p->survivors.empty())
        for (int g = 0; g < p->n_gpus; ++g) {
            o.f("replan rank %d gpu=%d resident:", g, p->survivors[g]);
            for (size_t c = 0; c < p->chunks.size(); ++c)
                if (p->resident[g][c]) o.f(" %zu", c);
            o.f("\n");
        }
    o.f("sizes host_base=%" PRId64 " host_adapter=%" PRId64 " dev_weights=%" PRId64 " dev_adapters=%" PRId64 "\n",
        p->host_base_bytes, p->host_adapter_bytes, p->dev_weight_bytes, p->host_adapter_bytes);
    o.f("end\n");
    return o.s;
}

extern "C" pb_status pb_plan_dump(const pb_plan* plan, char* buf, size_t cap, size_t* needed) {
    PB_TRY_BEGIN
    if (!plan || !needed) return pb::fail(PB_EINVAL, "pb_plan_dump: null argument");
    std::string s = dump_string(plan);
    *needed = s.size() + 1;
    if (buf && cap > 0) {
        size_t n = std::min(cap - 1, s.size());
        memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    if (!buf || cap < s.size() + 1) return pb::fail(PB_ENOMEM, "pb_plan_dump: need %zu bytes", s.size() + 1);
    return PB_OK;
    PB_TRY_END
}

extern "C" pb_status pb_plan_sizes(const pb_plan* p, pb_plan_sizes_t* out) {
    if (!p || !out) return pb::fail(PB_EINVAL, "pb_plan_sizes: null argument");
    out->host_base_bytes = p->host_base_bytes;
    out->host_adapter_bytes = p->host_adapter_bytes;
    out->dev_weight_bytes = p->dev_weight_bytes;
    out->dev_adapter_bytes = p->host_adapter_bytes;
    out->dev_adapted_bytes = p->dev_adapted_bytes;
    out->dev_backup_bytes = p->dev_backup_bytes;
    out->n_tensors = (int32_t)p->tensors.size();
    out->n_atensors = (int32_t)p->atensors.size();
    out->n_chunks = (int32_t)p->chunks.size();
    out->n_gpus = p->n_gpus;
    return PB_OK;
}

extern "C" pb_status pb_plan_tensor(const pb_plan* p, int32_t i, pb_tensor_info* out) {
    if (!p || !out) return pb::fail(PB_EINVAL, "pb_plan_tensor: null argument");
    if (i < 0 || i >= (int32_t)p->tensors.size()) return pb::fail(PB_EINVAL, "tensor index %d out of range", i);
    auto& t = p->tensors[i];
    *out = {t.name.c_str(), t.rows, t.cols, t.layer, t.host_off, t.dev_off, t.bytes()};
    return PB_OK;
}

extern "C" pb_status pb_plan_atensor(const pb_plan* p, int32_t i, pb_atensor_info* out) {
    if (!p || !out) return pb::fail(PB_EINVAL, "pb_plan_atensor: null argument");
    if (i < 0 || i >= (int32_t)p->atensors.size()) return pb::fail(PB_EINVAL, "atensor index %d out of range", i);
    auto& t = p->atensors[i];
    *out = {t.name.c_str(), t.rows, t.cols, t.layer, t.adapter, t.target_bit, t.is_B, t.base, t.row0, t.off, t.bytes()};
    return PB_OK;
}

extern "C" void pb_plan_free(pb_plan* p) { delete p; }
