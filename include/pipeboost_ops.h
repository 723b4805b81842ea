/*
 * pipeboost_ops.h — the individual device kernels of the cold-start path, exposed for parity tests
 * and micro-benchmarks. These are the SAME kernels pb_merge_lora / pb_prefill_* launch.
 *
 * All pointers are DEVICE pointers on the current CUDA device unless stated; `stream` is a
 * cudaStream_t (NULL = legacy default stream). Calls are asynchronous; tensor maps are encoded on the
 * host per call (so these entry points cost a few microseconds of host time more than the path).
 * Returns PB_OK, PB_EINVAL (shape/alignment not supported) or PB_ECUDA (launch failed).
 * Layouts are row-major; bf16 = IEEE bfloat16 bits (uint16).
 */
#ifndef PIPEBOOST_OPS_H
#define PIPEBOOST_OPS_H

#include "pipeboost.h"

#ifdef __cplusplus
extern "C" {
#endif

/* a3 merge: W[rows x cols] (row pitch ldw elems) <- RNE_bf16(W + scale * B * A),
 * B [rows x rank] (pitch rank), A [rank x cols] (pitch cols); rank % 8 == 0, rank <= 64, cols % 8 == 0,
 * 16-byte aligned bases. tcgen05.mma with fp32 TMEM accumulation. */
PB_API pb_status pb_op_merge(void* W, int64_t ldw, int32_t rows, int32_t cols, const void* B, const void* A,
                             int32_t rank, float scale, void* stream);

/* n <= 8 merges of the same rank in ONE persistent launch (their 128x128 tiles walked as one list): job i is
 * W[i] [rows[i] x cols[i]] (pitch ldw[i]) <- RNE_bf16(W[i] + scale[i] * B[i] * A[i]) with the layouts of pb_op_merge.
 * The path merges the adapted chunks of one DMA group this way. */
PB_API pb_status pb_op_merge_batch(int32_t n, void* const* W, const int64_t* ldw, const int32_t* rows,
                                   const int32_t* cols, const void* const* B, const void* const* A, int32_t rank,
                                   const float* scale, void* stream);

/* Prefill GEMM: X [*, K] bf16 (rows [m_begin, m_end) used; the map spans x_rows rows), W [n_rows x K] bf16.
 * epi 0: out bf16 [*, ldo] = (X W^T + bias) * (col < scale_cols ? scale : 1), ReLU if relu;
 * epi 1: out fp32 [*, ldo] += X W^T + bias;
 * epi 2: W = [gate; up] with N = d_ffn outputs: out bf16 = silu(X gate^T) * (X up^T).
 * K % 64 == 0. bias may be NULL. m_end - m_begin <= 2 (f3 decode sizes): the weight-streaming GEMV (CUDA cores,
 * fixed-order fp32 sums); otherwise the tcgen05 kernels. */
PB_API pb_status pb_op_gemm(const void* X, int32_t x_rows, int32_t m_begin, int32_t m_end, int32_t K, const void* W,
                            int32_t n_rows, int32_t N, int32_t epi, const void* bias, int32_t relu, float scale,
                            int32_t scale_cols, void* out, int32_t ldo, void* stream);
/* Same with an explicit cluster split-K factor (0 = the path's automatic choice, else 1, 2, 4 or 8). */
PB_API pb_status pb_op_gemm_split(const void* X, int32_t x_rows, int32_t m_begin, int32_t m_end, int32_t K,
                                  const void* W, int32_t n_rows, int32_t N, int32_t epi, const void* bias, int32_t relu,
                                  float scale, int32_t scale_cols, void* out, int32_t ldo, int32_t split_k,
                                  void* stream);

/* Debug / measurement only: every following pb_op_gemm* launch of the split-K kernel writes 8 %globaltimer stamps
 * per CTA to trace (device, uint64 [grid CTAs][8]: entry, prologue done, activation wait passed, last load issued,
 * first stage landed, last MMA done, partial staged + cluster barrier, epilogue done), or none (trace = NULL); pdl != 0
 * launches them with programmatic dependent launch, as the prefill path does. Process-wide; not thread-safe. */
PB_API pb_status pb_op_debug_gemm(void* trace, int32_t pdl);

/* Llama QKV projection with the rotary embedding fused into the epilogue (DESIGN.md §3 storage contract:
 * q/k = RNE_bf16(rope(X Wqkv^T)), one rounding): epi 0 without bias / scale, then columns [0, rope_cols) (q and k
 * heads of hd = 64 or 128, head-aligned) rotated HF rotate_half style at position (row - row0) / B with
 * theta^(-2i/hd) angles; columns >= rope_cols (v) plain. table: device scratch of T*hd/2*8 bytes (filled here,
 * positions < T). split_k as in pb_op_gemm_split; M <= 2 rows take the GEMV. */
PB_API pb_status pb_op_gemm_rope(const void* X, int32_t x_rows, int32_t m_begin, int32_t m_end, int32_t K,
                                 const void* W, int32_t N, void* out, int32_t ldo, int32_t rope_cols, int32_t hd,
                                 int32_t row0, int32_t B, int32_t T, float theta, void* table, int32_t split_k,
                                 void* stream);

/* LayerNorm (beta != NULL) or RMSNorm (beta == NULL): fp32 h [rows x d] -> bf16 out [rows x d]. */
PB_API pb_status pb_op_norm(const float* h, int32_t rows, int32_t d, const void* gamma, const void* beta, float eps,
                            void* out, void* stream);

/* Causal attention (token-major rows t*B+b of qkv, row pitch ld): queries [t0, t1) of every sequence.
 * q at col h*hd, k at k_col0 + kvh*hd, v at v_col0 + kvh*hd; out bf16 [*, ldo] at col h*hd. */
PB_API pb_status pb_op_attention(const void* qkv, int32_t ld, void* out, int32_t ldo, int32_t t0, int32_t t1,
                                 int32_t B, int32_t n_heads, int32_t n_kv_heads, int32_t hd, int32_t k_col0,
                                 int32_t v_col0, float score_scale, void* stream);

/* RoPE (rotate_half, theta) in place on q heads [0, n_q) at col 0 and k heads at k_col0, rows [r0, r1).
 * table: device scratch of T*hd/2*8 bytes (filled here). */
PB_API pb_status pb_op_rope(void* qkv, int32_t ld, int32_t r0, int32_t r1, int32_t B, int32_t T, int32_t n_q,
                            int32_t n_k, int32_t hd, int32_t k_col0, float theta, void* table, void* stream);

/* logits[b, v] (fp32, pitch ldl) = y[b] . E[v] for v in [v0, v1); y bf16 [B x d], E bf16 [V x d] (the LM head,
 * P:L99-107 final projection). B <= 2: the weight-streaming GEMV into a zeroed slice; 3-15: warp-per-row kernel, 8
 * sequences per launch; >= 16: the tensor-core GEMM. Each output is summed in an order independent of [v0, v1), so
 * vocab slices reproduce the whole head bit for bit. Errors: PB_EINVAL (d % 8), PB_ECUDA. */
PB_API pb_status pb_op_logits(const void* y, int32_t B, int32_t d, const void* E, int32_t v0, int32_t v1,
                              float* logits, int32_t ldl, void* stream);

/* tokens[b] = argmax_v logits[b, v], lowest index on ties; nan_flag |= 1 on non-finite logits. */
PB_API pb_status pb_op_argmax(const float* logits, int32_t B, int32_t V, int32_t ldl, int32_t* tokens,
                              int32_t* nan_flag, void* stream);

/* Embedding: h[row] = E[tok[row]] (+ pos[t + 2] when pos != NULL), rows [r0, r1), t = row / B. */
PB_API pb_status pb_op_embed(const void* E, const void* pos, const int32_t* tok, float* h, int32_t d, int32_t r0,
                             int32_t r1, int32_t B, void* stream);


#ifdef __cplusplus
}
#endif
#endif
