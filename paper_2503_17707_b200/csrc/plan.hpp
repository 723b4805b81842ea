// plan.hpp — internal representation of a pb_plan (host only).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/pipeboost.h"

namespace pb {

constexpr int64_t kAlign = 4096;
constexpr int kMaxGpus = 8;

struct TensorRec {
    std::string name;
    int32_t rows, cols, layer;
    int64_t host_off, dev_off;
    int32_t es = 2;   // element size: 2 (bf16) or 4 (fp32)
    int64_t bytes() const { return (int64_t)rows * cols * es; }
    int64_t row_bytes() const { return (int64_t)cols * es; }
};

struct ATensorRec {
    std::string name;
    int32_t rows, cols, layer, adapter;
    int32_t target_bit;   // PB_T_*
    int32_t is_B;         // 0: A [r x in], 1: B [out x r]
    int32_t base;         // base tensor id
    int32_t row0;         // first base row it modifies
    int64_t off;
    int32_t es = 2;
    int64_t bytes() const { return (int64_t)rows * cols * es; }
    int64_t row_bytes() const { return (int64_t)cols * es; }
};

struct ChunkRec {
    int32_t id;
    int32_t is_adapter;
    int32_t tensor;        // base tensor id or atensor id
    int32_t r0, r1;
    int64_t host_off, dev_off, bytes;
    int32_t loader;
};

// One LoRA target region of one layer for one adapter: the merge unit.
struct MergeRec {
    int32_t adapter, layer, target_bit;
    int32_t base;          // base tensor id
    int32_t row0, rows, cols;   // rows = out_features, cols = in_features
    int32_t a_tensor, b_tensor; // atensor ids of A and B
};

}  // namespace pb

struct pb_plan {
    pb_model_desc model;
    std::vector<pb_adapter_desc> adapters;
    int32_t n_gpus;
    pb_plan_opts opts;
    std::vector<std::pair<int32_t, int32_t>> stages;
    std::vector<pb::TensorRec> tensors;
    std::vector<pb::ATensorRec> atensors;
    std::vector<pb::ChunkRec> chunks;
    std::vector<std::vector<int32_t>> load, recv;
    std::vector<int32_t> own;
    std::vector<pb::MergeRec> merges;
    int64_t host_base_bytes = 0, host_adapter_bytes = 0, dev_weight_bytes = 0;
    // Multi-adapter (out-of-place) merges: a full copy of every base tensor an adapter modifies, per adapter,
    // in a separate device region. adapted_off[a * n_tensors + t] = offset, or -1 when adapter a does not touch t.
    std::vector<int64_t> adapted_off;
    int64_t dev_adapted_bytes = 0;
    // f2 adapter switching: backup_off[t] = offset of tensor t's pristine copy (-1: no adapter touches t)
    std::vector<int64_t> backup_off;
    int64_t dev_backup_bytes = 0;
    // f1 re-plans (pb_plan_replan): original GPU of every new rank, and per rank the chunks it already holds
    // (never loaded or received again). Empty for a plan made by pb_plan_create.
    std::vector<int32_t> survivors;
    std::vector<std::vector<char>> resident;   // [rank][chunk]
    bool is_resident(int32_t rank, int32_t chunk) const {
        return !resident.empty() && resident[rank][chunk];
    }

    // derived helpers
    int32_t head_dim() const { return model.d_model / model.n_heads; }
    bool f32() const { return model.dtype == PB_DTYPE_F32; }
    int32_t es() const { return f32() ? 4 : 2; }
    int32_t stage_of_layer(int32_t l) const;
    int32_t find_tensor(const std::string& name) const;   // -1 if absent (O(1): the prefill looks tensors up per layer)
    std::unordered_map<std::string, int32_t> name_index;
};
