// kernels.hpp — launchers of the device kernels (host-callable, asynchronous on `stream`).
// Every launcher returns cudaError_t of the launch; kernels never allocate.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

namespace pb {

// Launch with an optional programmatic-dependent-launch edge to the previous kernel of the stream (the kernel
// must call pdl_wait() before reading anything that kernel wrote).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                              Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the call costs microseconds of host
// time and the prefill issues thousands of launches, which would leave the GPU waiting on the issuer.
template <auto Fn>
inline cudaError_t smem_attr_once(int bytes) {
    static std::atomic<unsigned long long> done{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(Fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
    return e;
}

// ---------------------------------------------------------------- tensor maps (TMA)
// Resolved once from the driver (cudaGetDriverEntryPoint), no libcuda link dependency.
bool driver_init(char* err, size_t errlen);
// 2-D bf16 tensor map: rows x cols row-major with row pitch `ld_elems`, box {box_cols, box_rows},
// swizzle in bytes (0, 32, 64, 128). Returns false and fills err on failure.
bool make_map_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                   uint32_t box_rows, uint32_t box_cols, int swizzle_bytes, char* err, size_t errlen);

// 3-D bf16 tensor map: dims innermost first, strides (bytes) of dims 1 and 2, box innermost first.
bool make_map_bf16_3d(CUtensorMap* map, const void* base, const uint64_t dims[3], const uint64_t strides_bytes[2],
                      const uint32_t box[3], int swizzle_bytes, char* err, size_t errlen);

// Stream memory operations / cross-rank readiness words.
cudaError_t stream_wait_geq(cudaStream_t s, const uint32_t* dev_addr, uint32_t value);
cudaError_t stream_write(cudaStream_t s, uint32_t* dev_addr, uint32_t value);   // after all prior stream work
struct SignalTargets {
    uint32_t* addr[8];
    int n;
};
cudaError_t launch_signal(const SignalTargets& t, uint32_t value, cudaStream_t s);
// f3 decode: tokens[(*dyn) * B + b] = tok_out[b] (the previous step's argmax becomes this step's input).
cudaError_t launch_feed_tokens(int32_t* tokens, const int32_t* tok_out, const int* dyn, int B, cudaStream_t s);
// base[idx[i]] = value (release, system scope) for i < n; idx is a device array.
cudaError_t launch_set_words(uint32_t* base, const int32_t* idx, int n, uint32_t value, cudaStream_t s);

// ---------------------------------------------------------------- a3: LoRA merge (tcgen05)
// W[rows x cols] (row pitch ldw) <- RNE_bf16(W + scale * B[rows x r] * A[r x cols]), fp32 accumulate in TMEM.
// Maps: mapW box {64 cols, 128 rows} SW128; mapB box {rk, 128} with swizzle rk*2 bytes; mapA box {64, rk} SW128,
// rk = r rounded up to 16 / 32 / 64 (zero-filled by TMA out of bounds).
struct MergeMaps {
    CUtensorMap W, B, A, Wout;   // Wout: destination (== W in place; an adapter's copy out of place)
};
int merge_rk(int rank);  // padded K of the merge MMA (16, 32 or 64)
bool make_merge_maps(MergeMaps* m, void* W, int64_t ldw, int rows, int cols, const void* B, const void* A, int rank,
                     char* err, size_t errlen, void* Wout = nullptr);
// SM byte copy (16-B vectors; falls back to cudaMemcpyAsync for unaligned spans).
cudaError_t launch_copy(void* dst, const void* src, int64_t bytes, cudaStream_t s);
cudaError_t launch_merge(const MergeMaps& maps, int rows, int cols, int rank, float scale, cudaStream_t s);
// Up to kMaxMergeJobs merges of the same padded rank in ONE persistent launch (the tiles of all jobs are walked as
// one list): the adapted tensors of a DMA group merge in one kernel instead of one launch each.
constexpr int kMaxMergeJobs = 8;
struct MergeJobDesc {
    const MergeMaps* maps;
    int rows, cols, rank;
    float scale;
};
cudaError_t launch_merge_batch(const MergeJobDesc* jobs, int n, cudaStream_t s);

// ---------------------------------------------------------------- prefill GEMM (tcgen05)
// out = X[M x K] * W[N x K]^T with a fused epilogue. X rows [m_begin, m_end) are computed.
enum GemmEpi : int {
    EPI_BF16 = 0,      // out_bf16[m, n] = bf16((acc + bias[n]) * (n < scale_cols ? scale : 1)), optional ReLU
    EPI_RESID = 1,     // h_f32[m, n] += acc + bias[n]
    EPI_SILU_MUL = 2,  // W is [gate; up] (2*N_out x K); out_bf16[m, n] = bf16(silu(gate_n) * up_n), n < N_out
};
struct GemmArgs {
    int M_begin, M_end;   // rows of X / out computed
    int N, K;             // N = output columns (EPI_SILU_MUL: N_out), K = reduction length (multiple of 64)
    int epi;
    int relu;
    int scale_cols;
    float scale;
    const __nv_bfloat16* bias;  // [N] or null
    void* out;                  // bf16 [*, ldo] or fp32 [*, ldo]
    int ldo;
    int up_row0;                // EPI_SILU_MUL: first row of `up` in W (= N_out)
    int split_k;                // 0 = automatic (gemm_split_k), else the cluster split-K factor (1, 2, 4, 8)
    unsigned long long* trace;  // debug (pb_op_debug_gemm): 8 %globaltimer stamps per CTA of the split-K kernel, or null
    const int* m_dyn;           // f3 decode graphs: rows shift by (*m_dyn) * m_dyn_mul (device), or null
    int m_dyn_mul;
    int M_total;                // rows of the whole prompt batch (picks split_k; chunk-invariant), 0 = M_end-M_begin
    int pdl;                    // 1: programmatic dependent launch after the stream's previous kernel
    // plain pointers for the weight-streaming GEMV (M_total <= kGemvAutoRows: decode steps, tiny prompts);
    // null = tensor-core kernels only
    const __nv_bfloat16* X;     // [*, ldx] (rows as for mapX)
    int ldx;
    const __nv_bfloat16* W;     // [rows x K] row-major (rows as for mapW)
    // the same weights with 64-row boxes (64-column tiles, gemm_tile_n); null = 128-column tiles only (host pointer)
    const CUtensorMap* mapW64;
    // ... and with 32-row boxes (the persistent kernel's 160- / 224-column tiles); null = not used (host pointer)
    const CUtensorMap* mapW32;
    // Llama QKV (EPI_BF16): rotary embedding applied to the fp32 accumulator BEFORE the one bf16 rounding, so
    // q/k = RNE_bf16(rope(x Wqk^T)) exactly as the storage contract says. Columns [0, rope_cols)
    // are q and k heads of rope_hd columns each (head-aligned); output row r is at position
    // (r - rope_row0) / rope_B; rope = [positions][rope_hd / 2] (cos, sin) table. null = no rotation.
    const float2* rope;
    int rope_cols, rope_hd, rope_row0, rope_B;
};
int gemm_tile_n(int N, int K, int epi, int M_total);
constexpr int kGemvAutoRows = 2;   // rows up to which launch_gemm picks the GEMV
int gemm_split_k(int N, int K, int epi, int M_total);

// Maps: X box {64, 128} SW128 over [max_rows x K]; W box {64, 128} (EPI_SILU_MUL: {64, 64}) SW128 over [rows x K].
cudaError_t launch_gemm(const CUtensorMap& mapX, const CUtensorMap& mapW, const GemmArgs& a, cudaStream_t s);
// logits[b, v0:v1] (fp32, row pitch ldl) = y[b] . E[v0:v1]^T for large batches (tcgen05, S = 1)
// logits[b, v0:v1] for B <= 2 sequences through the weight-streaming GEMV (zeroed fp32 slice, then y . E^T)
cudaError_t launch_logits_gemv(const __nv_bfloat16* y, int B, int d, const __nv_bfloat16* E, int v0, int v1,
                               float* logits, int ldl, cudaStream_t s, bool pdl);
cudaError_t launch_logits_tc(const __nv_bfloat16* y, int B, int d, const __nv_bfloat16* E, int v0, int v1, float* logits,
                             int ldl, cudaStream_t s);


// ---------------------------------------------------------------- SIMT kernels
// Row norm over d of fp32 rows -> bf16: LayerNorm (beta != null) or RMSNorm (beta == null).
// dyn (f3 decode graphs): input rows shift by (*dyn) * dyn_in and output rows by (*dyn) * dyn_out (device).
cudaError_t launch_norm(const float* h, int ldh, __nv_bfloat16* out, int ldo, int rows, int d, const __nv_bfloat16* gamma,
                        const __nv_bfloat16* beta, float eps, cudaStream_t s, bool pdl = false,
                        const int* dyn = nullptr, int dyn_in = 0, int dyn_out = 0);

struct EmbedSrc {
    const void* base[8];           // embedding table of each owner (peer pointers allowed); bf16 or fp32
    int slice_begin[9];            // vocab rows [slice_begin[i], slice_begin[i+1]) live on owner i
    int n;
};
// h[row, :] = E[tok[row]] (+ P[pos(row) + 2]) as fp32, rows [r0, r1), row = t * B + b.
cudaError_t launch_embed(const EmbedSrc& E, const __nv_bfloat16* pos, const int32_t* tok, float* h, int d, int r0,
                         int r1, int B, cudaStream_t s, bool pdl = false, const int* dyn = nullptr);

// RoPE cos/sin table [T x hd/2] (float2), angles t * theta^(-2i/hd) computed in fp64.
cudaError_t launch_rope_table(float2* table, int T, int hd, double theta, cudaStream_t s);
// In-place rotate_half RoPE on q (n_q heads at col 0) and k (n_k heads at col q_cols) of rows [r0, r1).
cudaError_t launch_rope(__nv_bfloat16* qkv, int ld, int r0, int r1, int B, int n_q, int n_k, int hd, int k_col0,
                        const float2* table, cudaStream_t s, bool pdl = false, const int* dyn = nullptr);

// Causal attention for query rows [t0, t1) (token-major rows t*B+b) against keys [0, t] of the same
// sequence; q at col h*hd, k at k_col0 + (h/group)*hd, v at v_col0 + (h/group)*hd of `qkv`.
// hd = 64 or 128: tensor-core kernel (attention.cu); other head sizes: the SIMT kernel (simt.cu).
// dyn (f3 decode graphs): positions shift by *dyn; t_extent then bounds the keys' TMA view (>= every t1 + *dyn).
cudaError_t launch_attention(const __nv_bfloat16* qkv, int ld, __nv_bfloat16* out, int ldo, int t0, int t1, int B,
                             int n_heads, int n_kv_heads, int hd, int k_col0, int v_col0, float score_scale,
                             cudaStream_t s, bool pdl = false, const int* dyn = nullptr, int t_extent = 0,
                             int seq_stride = 0);
// seq_stride > 0: sequence-major rows (sequence b at rows b * seq_stride + t: the multi-adapter microbatches, all of
// them in one launch); 0: token-major rows t * B + b.
// One query position per sequence (decode): keys [0, t1 - 1 (+ *dyn)] of (head, sequence), contract-exact P rounding;
// max_keys bounds the keys (shared memory for the scores).
cudaError_t launch_decode_attention(const __nv_bfloat16* qkv, int ld, __nv_bfloat16* out, int ldo, int t1, int B,
                                    int n_heads, int n_kv_heads, int hd, int k_col0, int v_col0, float score_scale,
                                    cudaStream_t s, bool pdl, const int* dyn, int max_keys);
cudaError_t launch_attention_simt(const __nv_bfloat16* qkv, int ld, __nv_bfloat16* out, int ldo, int t0, int t1,
                                  int B, int n_heads, int n_kv_heads, int hd, int k_col0, int v_col0,
                                  float score_scale, cudaStream_t s);

// logits[b, v] = sum_c y[b, c] * E[v, c] for v in [v0, v1) (fp32 out, row pitch ldl).
cudaError_t launch_logits(const __nv_bfloat16* y, int B, int d, const __nv_bfloat16* E, int v0, int v1, float* logits,
                          int ldl, cudaStream_t s, bool pdl = false);
// tokens[b] = argmax_v logits[b, v] (lowest index on ties); *nan_flag |= 1 if any logit is not finite.
cudaError_t launch_argmax(const float* logits, int B, int V, int ldl, int32_t* tokens, int32_t* nan_flag,
                          cudaStream_t s, bool pdl = false);

// Load every kernel of the library into the current context (CUDA lazy module loading otherwise loads a
// function at its first launch; concurrent first launches from several issuer threads were measured to
// deadlock). Called once per device from pb_ctx_create.
cudaError_t warm_merge_kernels();
cudaError_t warm_gemm_kernels();
cudaError_t warm_simt_kernels();
cudaError_t warm_attention_kernels();
cudaError_t warm_f32_kernels();

// ---------------------------------------------------------------- fp32 debug-parity path (f32.cu)
// Same operations as above with fp32 weights and activations on CUDA-core FFMA (PB_DTYPE_F32; not timed).
cudaError_t launch_merge_f32(const float* W, float* Wout, int64_t ldw, int rows, int cols, const float* B,
                             const float* A, int rank, float scale, cudaStream_t s);
cudaError_t launch_gemm_f32(const float* X, int ldx, int M_begin, int M_end, const float* W, int N, int K, int epi,
                            const float* bias, int relu, float scale, int scale_cols, float* out, int ldo, int up_row0,
                            cudaStream_t s);
cudaError_t launch_norm_f32(const float* h, int ldh, float* out, int ldo, int rows, int d, const float* gamma,
                            const float* beta, float eps, cudaStream_t s);
cudaError_t launch_embed_f32(const EmbedSrc& E, const float* pos, const int32_t* tok, float* h, int d, int r0, int r1,
                             int B, cudaStream_t s);
cudaError_t launch_rope_f32(float* qkv, int ld, int r0, int r1, int B, int n_q, int n_k, int hd, int k_col0,
                            const float2* table, cudaStream_t s);
cudaError_t launch_attention_f32(const float* qkv, int ld, float* out, int ldo, int t0, int t1, int B, int n_heads,
                                 int n_kv_heads, int hd, int k_col0, int v_col0, float score_scale, cudaStream_t s);
cudaError_t launch_logits_f32(const float* y, int B, int d, const float* E, int v0, int v1, float* logits, int ldl,
                              cudaStream_t s);

}  // namespace pb
