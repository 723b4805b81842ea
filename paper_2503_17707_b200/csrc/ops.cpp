// ops.cpp — pb_op_*: the path's kernels behind the C ABI, one call = one kernel (for parity tests).
#include <cuda_runtime.h>

#include "../../include/pipeboost_ops.h"
#include "errors.hpp"
#include "kernels.hpp"

using namespace pb;

static pb_status cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return PB_OK;
    return fail(PB_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" pb_status pb_op_merge(void* W, int64_t ldw, int32_t rows, int32_t cols, const void* B, const void* A,
                                 int32_t rank, float scale, void* stream) {
    if (!W || !B || !A) return fail(PB_EINVAL, "pb_op_merge: null pointer");
    if (rank < 8 || rank > 64 || rank % 8 || cols % 8 || ldw % 8 || rows < 0 || cols < 0)
        return fail(PB_EINVAL, "pb_op_merge: need rank%%8==0, rank<=64, cols%%8==0 (rank=%d cols=%d)", rank, cols);
    if (!aligned16(W) || !aligned16(B) || !aligned16(A)) return fail(PB_EINVAL, "pb_op_merge: bases must be 16-B aligned");
    if (rows == 0 || cols == 0) return PB_OK;
    MergeMaps m;
    char err[512];
    if (!make_merge_maps(&m, W, ldw, rows, cols, B, A, rank, err, sizeof err)) return fail(PB_EINVAL, "%s", err);
    return cuda_status(launch_merge(m, rows, cols, rank, scale, (cudaStream_t)stream), "merge");
}

extern "C" pb_status pb_op_merge_batch(int32_t n, void* const* W, const int64_t* ldw, const int32_t* rows,
                                       const int32_t* cols, const void* const* B, const void* const* A, int32_t rank,
                                       const float* scale, void* stream) {
    if (n < 0 || n > kMaxMergeJobs) return fail(PB_EINVAL, "pb_op_merge_batch: n = %d (1..%d)", n, kMaxMergeJobs);
    if (n == 0) return PB_OK;
    if (!W || !ldw || !rows || !cols || !B || !A || !scale) return fail(PB_EINVAL, "pb_op_merge_batch: null array");
    if (rank < 8 || rank > 64 || rank % 8) return fail(PB_EINVAL, "pb_op_merge_batch: rank %d", rank);
    MergeMaps maps[kMaxMergeJobs];
    MergeJobDesc jobs[kMaxMergeJobs];
    char err[512];
    for (int i = 0; i < n; ++i) {
        if (!W[i] || !B[i] || !A[i]) return fail(PB_EINVAL, "pb_op_merge_batch: null pointer in job %d", i);
        if (cols[i] % 8 || ldw[i] % 8 || rows[i] < 0 || cols[i] < 0)
            return fail(PB_EINVAL, "pb_op_merge_batch: job %d needs cols %% 8 == 0", i);
        if (!aligned16(W[i]) || !aligned16(B[i]) || !aligned16(A[i]))
            return fail(PB_EINVAL, "pb_op_merge_batch: job %d bases must be 16-B aligned", i);
        if (rows[i] && cols[i] && !make_merge_maps(&maps[i], W[i], ldw[i], rows[i], cols[i], B[i], A[i], rank, err,
                                                   sizeof err))
            return fail(PB_EINVAL, "%s", err);
        jobs[i] = MergeJobDesc{&maps[i], rows[i], cols[i], rank, scale[i]};
    }
    return cuda_status(launch_merge_batch(jobs, n, (cudaStream_t)stream), "merge batch");
}

extern "C" pb_status pb_op_gemm(const void* X, int32_t x_rows, int32_t m_begin, int32_t m_end, int32_t K,
                                const void* W, int32_t n_rows, int32_t N, int32_t epi, const void* bias, int32_t relu,
                                float scale, int32_t scale_cols, void* out, int32_t ldo, void* stream) {
    return pb_op_gemm_split(X, x_rows, m_begin, m_end, K, W, n_rows, N, epi, bias, relu, scale, scale_cols, out, ldo, 0,
                            stream);
}

// debug state of pb_op_debug_gemm (process-wide; the op tests and tools/gemm_phases.py set it)
static unsigned long long* g_gemm_trace = nullptr;
static int g_gemm_pdl = 0;

extern "C" pb_status pb_op_debug_gemm(void* trace, int32_t pdl) {
    g_gemm_trace = static_cast<unsigned long long*>(trace);
    g_gemm_pdl = pdl != 0;
    return PB_OK;
}

static pb_status gemm_op(const void* X, int32_t x_rows, int32_t m_begin, int32_t m_end, int32_t K, const void* W,
                         int32_t n_rows, int32_t N, int32_t epi, const void* bias, int32_t relu, float scale,
                         int32_t scale_cols, void* out, int32_t ldo, int32_t split_k, void* stream);

extern "C" pb_status pb_op_gemm_split(const void* X, int32_t x_rows, int32_t m_begin, int32_t m_end, int32_t K,
                                      const void* W, int32_t n_rows, int32_t N, int32_t epi, const void* bias,
                                      int32_t relu, float scale, int32_t scale_cols, void* out, int32_t ldo,
                                      int32_t split_k, void* stream) {
    if (split_k < 0 || split_k > 8 || (split_k & (split_k - 1)) || (split_k > 0 && split_k > (K + 63) / 64))
        return fail(PB_EINVAL, "pb_op_gemm_split: split_k %d out of range", split_k);
    return gemm_op(X, x_rows, m_begin, m_end, K, W, n_rows, N, epi, bias, relu, scale, scale_cols, out, ldo, split_k,
                   stream);
}

static pb_status gemm_op(const void* X, int32_t x_rows, int32_t m_begin, int32_t m_end, int32_t K, const void* W,
                         int32_t n_rows, int32_t N, int32_t epi, const void* bias, int32_t relu, float scale,
                         int32_t scale_cols, void* out, int32_t ldo, int32_t split_k, void* stream) {
    if (!X || !W || !out) return fail(PB_EINVAL, "pb_op_gemm: null pointer");
    if (K % 8 || K <= 0 || epi < 0 || epi > 2 || m_begin < 0 || m_end > x_rows)
        return fail(PB_EINVAL, "pb_op_gemm: bad shape (K=%d epi=%d)", K, epi);
    CUtensorMap mx, mw;
    char err[512];
    if (!make_map_bf16(&mx, X, x_rows, K, K, 128, 64, 128, err, sizeof err) ||
        !make_map_bf16(&mw, W, n_rows, K, K, epi == EPI_SILU_MUL ? 64 : 128, 64, 128, err, sizeof err))
        return fail(PB_EINVAL, "%s", err);
    GemmArgs a{};
    a.M_begin = m_begin;
    a.M_end = m_end;
    a.N = N;
    a.K = K;
    a.epi = epi;
    a.relu = relu;
    a.scale = scale;
    a.scale_cols = scale_cols;
    a.bias = static_cast<const __nv_bfloat16*>(bias);
    a.out = out;
    a.ldo = ldo;
    a.up_row0 = N;
    a.split_k = split_k;
    a.trace = g_gemm_trace;
    a.pdl = g_gemm_pdl;
    a.M_total = m_end - m_begin;
    CUtensorMap mw64, mw32;
    if (epi != EPI_SILU_MUL) {
        if (!make_map_bf16(&mw64, W, n_rows, K, K, 64, 64, 128, err, sizeof err) ||
            !make_map_bf16(&mw32, W, n_rows, K, K, 32, 64, 128, err, sizeof err))
            return fail(PB_EINVAL, "%s", err);
        a.mapW64 = &mw64;   // 64-column tiles where gemm_tile_n picks them
        a.mapW32 = &mw32;   // the persistent kernel's 160- / 224-column tiles where gemm_big_tile_n picks them
    }
    a.X = static_cast<const __nv_bfloat16*>(X);   // M <= 2 with split_k == 0: the weight-streaming GEMV
    a.ldx = K;
    a.W = static_cast<const __nv_bfloat16*>(W);
    return cuda_status(launch_gemm(mx, mw, a, (cudaStream_t)stream), "gemm");
}

extern "C" pb_status pb_op_gemm_rope(const void* X, int32_t x_rows, int32_t m_begin, int32_t m_end, int32_t K,
                                     const void* W, int32_t N, void* out, int32_t ldo, int32_t rope_cols, int32_t hd,
                                     int32_t row0, int32_t B, int32_t T, float theta, void* table, int32_t split_k,
                                     void* stream) {
    if (!X || !W || !out || !table) return fail(PB_EINVAL, "pb_op_gemm_rope: null pointer");
    if (K % 8 || K <= 0 || m_begin < 0 || m_end > x_rows || B < 1 || T < 1 || (hd != 64 && hd != 128) ||
        rope_cols % hd || rope_cols > N || row0 > m_begin || (m_end - 1 - row0) / B >= T)
        return fail(PB_EINVAL, "pb_op_gemm_rope: bad shape");
    if (split_k < 0 || split_k > 8 || (split_k & (split_k - 1)))
        return fail(PB_EINVAL, "pb_op_gemm_rope: split_k %d out of range", split_k);
    cudaStream_t s = (cudaStream_t)stream;
    pb_status st = cuda_status(launch_rope_table(static_cast<float2*>(table), T, hd, theta, s), "rope table");
    if (st) return st;
    CUtensorMap mx, mw;
    char err[512];
    if (!make_map_bf16(&mx, X, x_rows, K, K, 128, 64, 128, err, sizeof err) ||
        !make_map_bf16(&mw, W, N, K, K, 128, 64, 128, err, sizeof err))
        return fail(PB_EINVAL, "%s", err);
    GemmArgs a{};
    a.M_begin = m_begin;
    a.M_end = m_end;
    a.N = N;
    a.K = K;
    a.epi = EPI_BF16;
    a.scale = 1.0f;
    a.out = out;
    a.ldo = ldo;
    a.up_row0 = N;
    a.split_k = split_k;
    a.M_total = m_end - m_begin;
    a.X = static_cast<const __nv_bfloat16*>(X);
    a.ldx = K;
    a.W = static_cast<const __nv_bfloat16*>(W);
    a.rope = static_cast<const float2*>(table);
    a.rope_cols = rope_cols;
    a.rope_hd = hd;
    a.rope_row0 = row0;
    a.rope_B = B;
    return cuda_status(launch_gemm(mx, mw, a, s), "gemm rope");
}

extern "C" pb_status pb_op_norm(const float* h, int32_t rows, int32_t d, const void* gamma, const void* beta, float eps,
                                void* out, void* stream) {
    if (!h || !gamma || !out) return fail(PB_EINVAL, "pb_op_norm: null pointer");
    return cuda_status(launch_norm(h, d, static_cast<__nv_bfloat16*>(out), d, rows, d,
                                   static_cast<const __nv_bfloat16*>(gamma), static_cast<const __nv_bfloat16*>(beta),
                                   eps, (cudaStream_t)stream),
                       "norm");
}

extern "C" pb_status pb_op_attention(const void* qkv, int32_t ld, void* out, int32_t ldo, int32_t t0, int32_t t1,
                                     int32_t B, int32_t n_heads, int32_t n_kv_heads, int32_t hd, int32_t k_col0,
                                     int32_t v_col0, float score_scale, void* stream) {
    if (!qkv || !out) return fail(PB_EINVAL, "pb_op_attention: null pointer");
    if (n_kv_heads <= 0 || n_heads % n_kv_heads) return fail(PB_EINVAL, "pb_op_attention: bad heads");
    return cuda_status(launch_attention(static_cast<const __nv_bfloat16*>(qkv), ld, static_cast<__nv_bfloat16*>(out),
                                        ldo, t0, t1, B, n_heads, n_kv_heads, hd, k_col0, v_col0, score_scale,
                                        (cudaStream_t)stream),
                       "attention");
}

extern "C" pb_status pb_op_rope(void* qkv, int32_t ld, int32_t r0, int32_t r1, int32_t B, int32_t T, int32_t n_q,
                                int32_t n_k, int32_t hd, int32_t k_col0, float theta, void* table, void* stream) {
    if (!qkv || !table) return fail(PB_EINVAL, "pb_op_rope: null pointer");
    cudaError_t e = launch_rope_table(static_cast<float2*>(table), T, hd, theta, (cudaStream_t)stream);
    if (e == cudaSuccess)
        e = launch_rope(static_cast<__nv_bfloat16*>(qkv), ld, r0, r1, B, n_q, n_k, hd, k_col0,
                        static_cast<const float2*>(table), (cudaStream_t)stream);
    return cuda_status(e, "rope");
}

extern "C" pb_status pb_op_logits(const void* y, int32_t B, int32_t d, const void* E, int32_t v0, int32_t v1,
                                  float* logits, int32_t ldl, void* stream) {
    if (!y || !E || !logits) return fail(PB_EINVAL, "pb_op_logits: null pointer");
    return cuda_status(launch_logits(static_cast<const __nv_bfloat16*>(y), B, d, static_cast<const __nv_bfloat16*>(E),
                                     v0, v1, logits, ldl, (cudaStream_t)stream),
                       "logits");
}

extern "C" pb_status pb_op_argmax(const float* logits, int32_t B, int32_t V, int32_t ldl, int32_t* tokens,
                                  int32_t* nan_flag, void* stream) {
    if (!logits || !tokens || !nan_flag) return fail(PB_EINVAL, "pb_op_argmax: null pointer");
    return cuda_status(launch_argmax(logits, B, V, ldl, tokens, nan_flag, (cudaStream_t)stream), "argmax");
}

extern "C" pb_status pb_op_embed(const void* E, const void* pos, const int32_t* tok, float* h, int32_t d, int32_t r0,
                                 int32_t r1, int32_t B, void* stream) {
    if (!E || !tok || !h) return fail(PB_EINVAL, "pb_op_embed: null pointer");
    EmbedSrc src{};
    src.base[0] = static_cast<const __nv_bfloat16*>(E);
    src.slice_begin[0] = 0;
    src.slice_begin[1] = 0x7fffffff;
    src.n = 1;
    return cuda_status(launch_embed(src, static_cast<const __nv_bfloat16*>(pos), tok, h, d, r0, r1, B,
                                    (cudaStream_t)stream),
                       "embed");
}

