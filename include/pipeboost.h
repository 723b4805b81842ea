/*
 * pipeboost.h — C ABI of the B200-native PipeBoost layer-sharded cold start.
 *
 * Method (PAPER.md = "P:L<line>"; SURVEY.md §8 is the scope contract):
 *   plan    — which GPU loads which layers, in which order
 *   load    — each GPU DMAs its own disjoint slice over PCIe    P:L235-236 ("GPU 0 reads A-0 while GPU 1 reads A-1")
 *   merge   — W' = W + (alpha/r) * B * A on the loader          P:L111-114, P:L267-270 (merged LoRA, §4.3.2)
 *   gather  — merged slices all-gathered over NVLink            P:L239, P:L247 (progressive loading of the rest)
 *   prefill — pipeline-parallel first token as layers arrive    P:L259-264 (§4.3.1)
 *
 * Conventions for every entry point:
 *   - Returns pb_status: 0 (PB_OK) or a negative error; never throws, never aborts.
 *     pb_last_error() returns a thread-local, human-readable message for the
 *     last failing call on the calling thread.
 *   - Preconditions (null pointers, ranges, call order) are checked synchronously.
 *     Asynchronous CUDA failures surface at the next blocking call
 *     (pb_sync, pb_prefill_wait, pb_prefill_first_token).
 *   - Pointers: "host" = CPU memory, "device" = memory of the rank's CUDA device.
 *     The caller owns every buffer and every stream; the library BORROWS them
 *     for the lifetime of the object it hands them to. The library owns only
 *     pb_plan, pb_ctx, and the CUDA events / tensor maps / IPC mappings inside a ctx.
 *   - One process (or one logical rank) per GPU. A pb_ctx belongs to one rank;
 *     calls on distinct contexts may run concurrently from different host threads
 *     (the paper coordinates GPUs with threads); calls on the same ctx
 *     must not.
 *   - Data type: weights and LoRA factors are bf16 (north star; the paper never
 *     states its dtype). Residual stream and logits are fp32.
 *     pb_model_desc.dtype = PB_DTYPE_F32 selects the fp32 debug-parity path (same
 *     calls, same layouts with 4-byte elements).
 */
#ifndef PIPEBOOST_H
#define PIPEBOOST_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PB_API __attribute__((visibility("default")))
#else
#define PB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PB_OK = 0,
    PB_EINVAL = -1,        /* bad argument: null pointer, out-of-range value, buffer too small for the plan */
    PB_EPARTITION = -2,    /* n_gpus > n_layers: no balanced contiguous partition */
    PB_EPROTOCOL = -3,     /* call order violated (per rank: trial_begin -> load -> merge -> gather -> prefill) */
    PB_ECUDA = -4,         /* a CUDA runtime/driver call failed (message has the CUDA error string) */
    PB_ENOMEM = -6,        /* caller-provided capacity smaller than required (see pb_plan_sizes) */
    PB_ENUMERIC = -7,      /* non-finite logits */
    PB_EUNSUPPORTED = -8   /* valid request this build does not implement (message says which) */
} pb_status;

typedef enum { PB_ARCH_OPT = 0, PB_ARCH_LLAMA = 1 } pb_arch;

/* Storage type of the weights and LoRA factors (SURVEY.md §8(c) "Tolerances"):
 *   PB_DTYPE_BF16 — the product path (tcgen05 merge / GEMM / attention), gated at 1e-2 relative;
 *   PB_DTYPE_F32  — fp32 debug-parity path: weights, factors and every activation fp32, merge and
 *                   projections on CUDA-core FFMA; gated at 1e-4 relative. Not timed. */
typedef enum { PB_DTYPE_BF16 = 0, PB_DTYPE_F32 = 1 } pb_dtype;

/* Decoder description (HF conventions). */
typedef struct {
    int32_t arch;          /* pb_arch */
    int32_t n_layers;
    int32_t d_model;
    int32_t n_heads;
    int32_t n_kv_heads;    /* == n_heads for OPT; GQA for Llama */
    int32_t d_ffn;
    int32_t vocab;
    int32_t max_pos;       /* OPT learned positions: table has max_pos + 2 rows; ignored for Llama */
    int32_t tied;          /* OPT: LM head tied to the token embedding */
    float norm_eps;        /* 1e-5 */
    float rope_theta;      /* 1e4 (Llama) */
    int32_t dtype;         /* pb_dtype of weights and adapters (0 = bf16) */
} pb_model_desc;

/* LoRA targets (bit mask). OPT: Q,K,V,O,FC1,FC2. Llama: Q,K,V,O,GATE,UP,DOWN. */
enum {
    PB_T_Q = 1, PB_T_K = 2, PB_T_V = 4, PB_T_O = 8, PB_T_FC1 = 16, PB_T_FC2 = 32,
    PB_T_GATE = 64, PB_T_UP = 128, PB_T_DOWN = 256
};

/* One adapter: B is [out x rank], A is [rank x in]; delta W = (alpha/rank) * B * A
 * (Hu et al. naming; the paper's P:L113 swaps the names). */
typedef struct {
    int32_t rank;          /* 1..64 */
    float alpha;
    uint32_t targets;      /* PB_T_* mask */
} pb_adapter_desc;

typedef enum {
    PB_LOAD_STAGE = 0,       /* GPU g loads its own stage's layers (paper, fig:ftpp_loading(c)) */
    PB_LOAD_INTERLEAVE = 1   /* layer l loaded by GPU l mod N; stage owners receive the rest over NVLink */
} pb_load_policy;

typedef struct {
    int32_t policy;            /* pb_load_policy */
    int32_t vocab_sliced;      /* 1: embedding / LM head split into N balanced row slices, one per GPU (G5) */
    int64_t chunk_bytes;       /* DMA chunk size (rows per chunk = chunk_bytes / row_bytes, rounded down to x128) */
    int32_t prefill_chunks;    /* k >= 1 prompt chunks pipelined through the stages */
    int32_t host_alias_layers; /* 0: host image holds every layer; K>0: layer l reads host image of layer l mod K */
} pb_plan_opts;

typedef struct pb_plan pb_plan;   /* opaque, immutable after creation, safe to share between threads */
typedef struct pb_ctx pb_ctx;     /* opaque, one per rank */

/* ------------------------------------------------------------------------ */
/* a1 — plan (host only, pure, deterministic)                                 */
/* ------------------------------------------------------------------------ */

/* Build the plan for `n_gpus` GPUs. Layer stages are contiguous and balanced,
 * the first (L mod N) stages one layer longer (remainder rule S:L130).
 * Errors: PB_EINVAL (null, n_gpus < 1, bad model/adapter field), PB_EPARTITION (n_gpus > n_layers),
 * PB_EUNSUPPORTED (rank > 64). *out receives a plan to release with pb_plan_free. */
PB_API pb_status pb_plan_create(const pb_model_desc* model, const pb_adapter_desc* adapters, int32_t n_adapters,
                         int32_t n_gpus, const pb_plan_opts* opts, pb_plan** out);

/* Canonical text dump of the plan (stages, tensor table, chunks, per-GPU load and
 * receive lists, adapter ownership, sizes). Writes at most cap bytes including the
 * terminating NUL; *needed = full length + 1. PB_ENOMEM if cap is too small
 * (buf then holds a truncated, NUL-terminated prefix). */
PB_API pb_status pb_plan_dump(const pb_plan* plan, char* buf, size_t cap, size_t* needed);

typedef struct {
    int64_t host_base_bytes;     /* pinned host image of the base model (canonical layout) */
    int64_t host_adapter_bytes;  /* pinned host image of all adapters */
    int64_t dev_weight_bytes;    /* per-GPU device buffer: the whole model, same offsets on every GPU */
    int64_t dev_adapter_bytes;   /* per-GPU device buffer for adapter factors (same layout as host) */
    int32_t n_tensors, n_atensors, n_chunks, n_gpus;
    int64_t dev_adapted_bytes;   /* per-GPU device buffer for out-of-place per-adapter copies of the adapted
                                    tensors (multi-adapter merge, pb_merge_lora(ctx, PB_MERGE_ALL)) */
    int64_t dev_backup_bytes;    /* per-GPU device buffer for the pristine base of every adapted tensor
                                    (saved by the cold-start merges; needed by pb_switch_adapter) */
} pb_plan_sizes_t;
PB_API pb_status pb_plan_sizes(const pb_plan* plan, pb_plan_sizes_t* out);

/* Device workspace bytes a rank needs to prefill `batch` sequences of `seq` tokens. */
PB_API pb_status pb_plan_workspace_bytes(const pb_plan* plan, int32_t batch, int32_t seq, int64_t* out);

/* Base tensor i (0 <= i < n_tensors) of the canonical table. name is owned by the plan. */
typedef struct {
    const char* name;
    int32_t rows, cols, layer;   /* layer = -1 for embed / pos / final norm / lm_head */
    int64_t host_off, dev_off, bytes;
} pb_tensor_info;
PB_API pb_status pb_plan_tensor(const pb_plan* plan, int32_t i, pb_tensor_info* out);

/* Adapter factor i (0 <= i < n_atensors): A ([rank x in]) or B ([out x rank]) of one target. */
typedef struct {
    const char* name;
    int32_t rows, cols, layer, adapter, target_bit, is_B, base_tensor, base_row0;
    int64_t off, bytes;          /* same offset in the host and device adapter buffers */
} pb_atensor_info;
PB_API pb_status pb_plan_atensor(const pb_plan* plan, int32_t i, pb_atensor_info* out);

PB_API void pb_plan_free(pb_plan* plan);

/* f1 — recovery for model loading (§4.4.2 "Recovery for model loading").
 * After GPUs crash during the cold start, build the plan that finishes it on the survivors without moving
 * any byte a survivor already holds:
 *   alive    host [plan n_gpus]: 1 = the GPU survived, 0 = crashed;
 *   resident host [plan n_gpus x n_chunks] bytes: 1 = that chunk is resident on that GPU (landed, and merged
 *            when its tensor is adapted); rows of crashed GPUs are ignored.
 * The new plan has m = (number of survivors) ranks. Its stages are m contiguous balanced blocks of layers
 * ("Load Balance", "Layer Contiguity") assigned to survivors so that the bytes each already
 * holds in its block are maximal (first maximum over all m! assignments in lexicographic order, so a tie
 * keeps the lower GPU id on the lower block); new rank r runs block r (pb_plan_gpu_of_rank maps it back to
 * the original GPU). Same tensor table, chunk table and offsets as `plan`; embedding / head whole
 * (vocab_sliced = 0). Every chunk no survivor holds is loaded once, by the rank whose block needs it; the
 * receive lists bring each rank its block's missing chunks first, then the rest of the model in rotation
 * order — e.g. GPUs 1, 2 of 4 crash: GPU 0 keeps "0, 1, 2, 3", GPU 3 becomes "2, 3, 0, 1".
 * pb_ctx_create on the new plan treats held chunks as already resident (marks them ready at trial start).
 * Errors: PB_EINVAL (null / no survivor), PB_EPARTITION (more survivors than layers),
 * PB_EUNSUPPORTED (re-planning a re-plan). *out receives a plan to release with pb_plan_free. */
PB_API pb_status pb_plan_replan(const pb_plan* plan, const int32_t* alive, const uint8_t* resident, pb_plan** out);
/* Original GPU index of rank `rank` of a re-plan (identity for a plan from pb_plan_create). */
PB_API pb_status pb_plan_gpu_of_rank(const pb_plan* plan, int32_t rank, int32_t* gpu);

/* ------------------------------------------------------------------------ */
/* Per-rank context                                                           */
/* ------------------------------------------------------------------------ */

typedef struct {
    void* weights;        int64_t weights_cap;    /* device, >= dev_weight_bytes */
    void* adapters;       int64_t adapters_cap;   /* device, >= dev_adapter_bytes (may be NULL if no adapters) */
    void* adapted;        int64_t adapted_cap;    /* device, >= dev_adapted_bytes for PB_MERGE_ALL, else may be NULL */
    void* workspace;      int64_t workspace_cap;  /* device, >= pb_plan_workspace_bytes(max_batch, max_seq) */
    int32_t max_batch, max_seq;   /* sequences per trial 1..64 (batch 64 x 64 tokens); max_seq <= max_pos (OPT) */
    /* cudaStream_t handles, five DISTINCT streams per rank; NULL = the ctx creates and owns its own
     * non-blocking streams (recommended: torch's stream pool recycles handles across ranks). */
    void* stream_h2d[2];  /* cudaStream_t: copy-engine H2D lane(s) (one ordered lane is used) */
    void* stream_merge;   /* cudaStream_t: merge kernels + per-layer readiness */
    void* stream_nvlink;  /* cudaStream_t: peer (NVLink) receive copies */
    void* stream_compute; /* cudaStream_t: prefill kernels */
    void* backup;         int64_t backup_cap;     /* device, >= dev_backup_bytes to enable pb_switch_adapter, else NULL */
} pb_rank_bufs;

/* Create rank `rank`'s context on the current CUDA device. host_base / host_adapters
 * are PINNED host images in the canonical layout (cudaHostAlloc / torch pin_memory);
 * host_adapters may be NULL when the plan has no adapters. Precomputes TMA tensor maps
 * and events; enqueues nothing. Errors: PB_EINVAL, PB_ENOMEM (capacity), PB_ECUDA. */
PB_API pb_status pb_ctx_create(const pb_plan* plan, int32_t rank, const void* host_base, const void* host_adapters,
                        const pb_rank_bufs* bufs, pb_ctx** out);

/* Cross-rank wiring (N > 1). Each rank exports an opaque blob of CUDA IPC handles
 * (weights, workspace, flag words); every other rank imports it. Blobs are
 * exchanged by the caller (e.g. torch.distributed all_gather_object).
 * pb_ctx_export: *needed = blob size; PB_ENOMEM if cap too small. */
PB_API pb_status pb_ctx_export(pb_ctx* ctx, void* blob, size_t cap, size_t* needed);
PB_API pb_status pb_ctx_import_peer(pb_ctx* ctx, int32_t peer, const void* blob, size_t len);
/* Same-process wiring (several ranks driven by one process, e.g. logical ranks on
 * one GPU in tests, or one process driving N devices): peer pointers taken directly. */
PB_API pb_status pb_ctx_link_local(pb_ctx* ctx, int32_t peer, pb_ctx* peer_ctx);

/* Start cold-start trial `epoch` (>= 1, strictly increasing, identical on all ranks).
 * Records t0 on stream_h2d[0]. Cross-rank readiness words are compared against the
 * epoch, so device flags never need resetting. */
PB_API pb_status pb_trial_begin(pb_ctx* ctx, uint32_t epoch);

/* f4 — storage tier ("a model checkpoint already residing in DRAM" is the
 * paper's starting point; its Table 1, charges 20.9-30.8% of TTFT to reading the checkpoint). With a
 * file source, the base weights of the cold start come from `path` — the checkpoint in the canonical host
 * layout (byte host_off of the plan at file offset host_off) — instead of the pinned host image: a reader
 * thread pread()s this rank's own copy groups, in load order, into the caller's PINNED, 4 KiB-aligned
 * staging buffer (>= 2 slots of the largest group; O_DIRECT when the file system allows), and each slot is
 * DMA'd as soon as it is full and refilled once its copy has landed — file reads, PCIe and merges overlap
 * chunk by chunk, every rank reading only its disjoint slice. LoRA factors still come from host_adapters.
 * path = NULL returns to the pinned image. Call between trials. Errors: PB_EINVAL (open / staging),
 * PB_ENOMEM (staging too small), PB_EPROTOCOL (a trial is being armed); read errors surface from the trial. */
PB_API pb_status pb_ctx_set_file_source(pb_ctx* ctx, const char* path, void* staging, int64_t staging_bytes);

/* a2 — arm this rank's load list ("GPU 0 reads A-0 while GPU 1 reads A-1"): chunked
 * cudaMemcpyAsync pinned host -> HBM over this GPU's own PCIe link, on ONE ordered copy lane
 * (stream_h2d[0]; measured on B200 the H2D engine drains one stream's queue before another's, so a second lane
 * would only delay layers), consecutive contiguous chunks coalesced into copy groups <= chunk_bytes, a
 * non-timing `landed` event per group. Load, merge and gather are armed in that order (PB_EPROTOCOL otherwise);
 * the copies start when the trial is fully armed, i.e. in pb_gather_layers, because each chunk's merge and peer
 * signal are issued right behind its copy group by the same per-rank issuer thread. Async. */
PB_API pb_status pb_load_shard(pb_ctx* ctx);

/* a3 — arm the LoRA merge of every adapted row range this rank loaded (tcgen05 kernel,
 * W <- RNE_bf16(W + s * B * A), fp32 accumulate), each issued right after its chunks land, followed by the
 * chunk's peer signal and readiness word. Must be called (even without adapters) after pb_load_shard.
 * adapter_id >= 0: merge that adapter IN PLACE into the base weights (one adapter per instance);
 * -1: no merge; PB_MERGE_ALL (-2): every adapter OUT OF PLACE into its own copy of each tensor it touches
 * (several adapters served at once; needs bufs.adapted and the STAGE policy when n_gpus > 1),
 * sequences then pick their adapter in pb_prefill_enqueue_ex. */
#define PB_MERGE_ALL (-2)
PB_API pb_status pb_merge_lora(pb_ctx* ctx, int32_t adapter_id);

/* a4 — arm this rank's receive list (here over NVLink): for each chunk, wait (device-side) for
 * the loader's readiness word (merged or landed), then copy peer HBM -> local HBM (copy engine, stream_nvlink).
 * Stage-needed chunks first, then rotation (g+i) mod N. With the trial fully armed this call
 * STARTS ISSUING it: a per-rank issuer thread enqueues the copy groups, the merges of each chunk as it lands
 * and the receive copies (pro rata to the load) without waiting for a prompt, so load -> merge -> gather ->
 * pb_sync reaches T_full on its own. A prompt posted later (pb_prefill_enqueue) joins the same issuer: its
 * compute items are interleaved with the loads still in flight (the prefill starts as soon as its layers are
 * resident, "begins serving ... while asynchronously loading the remaining parts"). Async. */
PB_API pb_status pb_gather_layers(pb_ctx* ctx);

/* a5 — pipelined first-token prefill. Every rank calls it (SPMD). tokens: host
 * [batch][seq] int32 (read on rank 0 only; other ranks may pass NULL); the
 * stages run layers as they become resident (no wait for the full model).
 * Rank 0 receives the first tokens (host [batch], lowest index wins exact ties)
 * and optionally the fp32 logits (host [batch][vocab] or NULL).
 * pb_prefill_enqueue only enqueues; pb_prefill_wait blocks until this rank's work
 * (and on rank 0 the token D2H) is complete; pb_prefill_first_token = both.
 * Errors: PB_EINVAL (batch/seq out of range, a token outside [0, vocab)), PB_EPROTOCOL, PB_ECUDA, PB_ENUMERIC. */
PB_API pb_status pb_prefill_enqueue(pb_ctx* ctx, const int32_t* tokens, int32_t batch, int32_t seq);
/* Same, with the adapter of every sequence (host [batch], read on every rank; needs PB_MERGE_ALL). The batch
 * then runs as `batch` single-sequence pipeline microbatches, each reading its adapter's merged copies. */
PB_API pb_status pb_prefill_enqueue_ex(pb_ctx* ctx, const int32_t* tokens, const int32_t* adapter_of_seq,
                                       int32_t batch, int32_t seq);
PB_API pb_status pb_prefill_wait(pb_ctx* ctx, float* logits_out, int32_t* tokens_out);
PB_API pb_status pb_prefill_first_token(pb_ctx* ctx, const int32_t* tokens, int32_t batch, int32_t seq,
                                 float* logits_out, int32_t* tokens_out);

/* f3 — pipelined decode. Compute the next token of every sequence
 * of the batch this context last prefilled (pb_prefill_enqueue / pb_prefill_replay): the position after the
 * prompt and the tokens decoded so far, fed with the previous step's argmax (already on the device, no host
 * round trip), attending over the KV cache the prefill and earlier steps left in the workspace (one q|k|v
 * slot per layer). Pipelined like the prefill: stage g runs its layers on the new position and hands the
 * activation to stage g+1; every rank calls it (SPMD) with the same new epoch. Complete with pb_prefill_wait
 * (tokens_out = the new tokens, on rank 0 or on a replica). Needs max_seq > prompt + decoded steps.
 * Errors: PB_EPROTOCOL (nothing prefilled, or prefilled in the other mode), PB_EINVAL (epoch, max_seq),
 * PB_EUNSUPPORTED (PB_MERGE_ALL microbatches). */
PB_API pb_status pb_decode_step(pb_ctx* ctx, uint32_t epoch);

/* f3 — seamless strategy switch: "Once all GPUs ... have fully loaded the complete model, PipeBoost
 * can seamlessly switch to ... single-GPU independent inference ... batches of requests submitted after the
 * switching point are executed using the new inference parallelism strategy." on = 1: this GPU serves its own
 * batches with the WHOLE model it holds after T_full (every layer, local head, no cross-rank traffic):
 * pb_prefill_replay (tokens on every replica) and pb_decode_step then run independently per rank. Requires a
 * completed cold start whose merges and receive copies have finished (pb_sync). on = 0: back to the pipeline.
 * Errors: PB_EPROTOCOL (no cold start / T_full not reached), PB_EUNSUPPORTED (PB_MERGE_ALL). */
PB_API pb_status pb_ctx_set_replica(pb_ctx* ctx, int32_t on);

/* f2 — epoch-based adapter switching (§4.3.2). Replace the adapter merged
 * into this rank's STAGE layers by `adapter_id` (or by none: -1): every adapted tensor of the stage is restored
 * from its pristine base copy (bufs.backup, saved by the cold start's merges) and the new adapter is merged
 * from it — W = RNE_bf16(W_base + s B A), so any sequence of switches gives exactly the weights a cold start
 * with that adapter gives (no drift). LoRA factors the rank did not load are fetched from the host image.
 * Enqueued on the compute stream behind every prefill already enqueued on this rank: a stage switches only
 * after finishing the batches handed to it, so along the pipeline the stages switch one after another
 * ("Each GPU switches adapters only after completing the batch received from the preceding GPU").
 * Requires a completed cold start with an in-place adapter (pb_merge_lora(ctx, a >= 0) or -1) and
 * bufs.backup. Serve the next batch with pb_prefill_replay. Async; errors: PB_EINVAL, PB_EPROTOCOL,
 * PB_ENOMEM (no backup buffer), PB_EUNSUPPORTED (PB_MERGE_ALL mode: every adapter is already merged). */
PB_API pb_status pb_switch_adapter(pb_ctx* ctx, int32_t adapter_id);

/* f2 scheduling (SPEC lora-scheduler S:L340-405): which adapter's batch runs next. Host only.
 * One FIFO queue per adapter plus the base-model queue (adapter -1). While an epoch of epoch_ms lasts,
 * batches come from the active adapter ("prioritizes the scheduling of batches corresponding to the currently
 * activated adapter"); when it has expired, the next non-empty queue in round-robin order (ids ascending,
 * base first) takes over ("At regular intervals, PipeBoost switches adapters"), except that a queue left
 * waiting over more than starvation_epochs expirations goes first; an empty active queue hands over at once.
 * pb_epoch_next returns the batch (up to max_batch request ids, FIFO, written to ids[]) and switch_needed = 1
 * when the stages must pb_switch_adapter first; *adapter = -2 and *n = 0 when every queue is empty.
 * Errors: PB_EINVAL (null, bad config, unknown adapter). Not thread-safe per scheduler. */
typedef struct pb_epoch pb_epoch;
PB_API pb_status pb_epoch_create(int32_t n_adapters, double epoch_ms, int32_t starvation_epochs, pb_epoch** out);
PB_API pb_status pb_epoch_set_active(pb_epoch* sched, int32_t adapter, double now_ms);  /* what the stages hold */
PB_API pb_status pb_epoch_enqueue(pb_epoch* sched, int32_t adapter, int64_t request_id);
PB_API pb_status pb_epoch_next(pb_epoch* sched, double now_ms, int32_t max_batch, int32_t* adapter,
                               int32_t* switch_needed, int64_t* ids, int32_t* n);
PB_API void pb_epoch_free(pb_epoch* sched);

/* Warm re-run of the last trial's prefill on the now-resident merged weights (no load / merge / gather,
 * no readiness waits on weights): the single-GPU-resident regime after T_full. Used by bench.py
 * to time every prefill kernel with CUDA events away from the PCIe-saturated cold-start window. Every
 * rank calls it with the same new epoch; complete it with pb_prefill_wait. */
PB_API pb_status pb_prefill_replay(pb_ctx* ctx, uint32_t epoch, const int32_t* tokens, int32_t batch, int32_t seq);

/* Block until every stream of this rank is idle; surfaces async CUDA errors. */
PB_API pb_status pb_sync(pb_ctx* ctx);

/* Timeline of the last trial (valid after pb_sync / pb_prefill_wait), ms since t0
 * on this rank's device clock. Arrays are owned by the ctx; valid until the next trial. */
typedef struct {
    double t_ready_ms;       /* every layer of this rank's stage resident and merged ("ready to serve") */
    double t_full_ms;        /* this rank holds the whole merged model (strategy-switch point) */
    double ttft_ms;          /* device time of the first-token D2H completion (rank 0), else last prefill op */
    double load_done_ms;     /* last own chunk landed */
    int64_t load_bytes;      /* bytes this rank moved over PCIe in the trial */
    int64_t recv_bytes;      /* bytes this rank received over NVLink */
    int32_t n_chunks;
    const double* chunk_landed_ms;   /* [n_chunks], -1 where not loaded by this rank; per-chunk times only when the
                                      * context was created with PB_LANDED_TIMING=1 (timing events on the saturated
                                      * copy lane cost ~20 us each), else -1 (load_done_ms is always set) */
    const double* chunk_gathered_ms; /* [n_chunks], -1 where not received by this rank */
    int32_t n_launches;      /* kernels this rank launched in the trial */
    const double* chunk_merged_ms;   /* [n_chunks], own chunk's merges (and peer signal) done; timing mode only
                                      * (PB_LANDED_TIMING=1), else -1 */
    double stage_begin_ms;   /* first layer kernel of this rank's stage started (compute stream; -1 if no stage) */
    double stage_end_ms;     /* last layer of the stage done for every microbatch / prompt chunk */
    double ctx_create_ms;    /* host time pb_ctx_create took (tables, TMA maps, events, pinned staging): part of the
                              * init breakdown excluded from t0 ("Init Meta") */
} pb_timeline_t;
PB_API pb_status pb_timeline(pb_ctx* ctx, pb_timeline_t* out);

/* Optional per-launch kernel timing (CUDA events around every kernel this rank launches, recorded on
 * the launching stream). Off by default. pb_kernel_stats aggregates the LAST trial per kernel class:
 * launches, summed device duration, and the algorithmic flops / bytes of those launches (the work the
 * method must do: GEMM 2MNK, merge 4 bytes per weight element + operands, ...). Classes: "merge",
 * "gemm", "attention", "norm", "rope", "embed", "logits", "argmax", "signal". */
typedef struct {
    const char* name;
    int32_t launches;
    double total_ms, flops, bytes;
} pb_kernel_stat;
PB_API pb_status pb_ctx_set_profiling(pb_ctx* ctx, int32_t enable);
PB_API pb_status pb_kernel_stats(pb_ctx* ctx, pb_kernel_stat* out, int32_t cap, int32_t* n);
/* Per-launch trace of the last profiled trial: class index (order of pb_kernel_stats), start / end ms
 * since t0 on the device clock. Writes min(cap, launches) records; *n = launches. */
typedef struct {
    int32_t cls;
    float start_ms, end_ms;
} pb_kernel_event;
PB_API pb_status pb_kernel_trace(pb_ctx* ctx, pb_kernel_event* out, int32_t cap, int32_t* n);

PB_API const char* pb_last_error(void);
PB_API void pb_ctx_free(pb_ctx* ctx);

/* f1 support — abandon the current trial after a peer has died mid-load (the survivors re-plan and
 * resume). Cross-rank dependencies are device-side waits on readiness words only peers write, so a dead peer
 * would leave this rank's streams blocked forever. pb_ctx_abort stops the issuer thread at its next poll, then
 * forces every readiness word of this rank's workspace open (epoch + 2^30: the waits compare cyclically) so the blocked streams
 * drain (their remaining kernels compute on whatever bytes are there; nothing is published as valid), and
 * marks the ctx aborted: every later call except pb_ctx_free returns PB_EPROTOCOL. pb_ctx_free of an aborted
 * ctx waits at most a few seconds per stream instead of synchronizing the device. The weight / adapter buffers
 * (caller-owned) keep whatever chunks had landed; pb_timeline before the abort tells which (chunk_landed_ms),
 * and Plan.replan + a new ctx with those buffers resumes. Errors: PB_EINVAL (null), PB_ECUDA. */
PB_API pb_status pb_ctx_abort(pb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PIPEBOOST_H */
