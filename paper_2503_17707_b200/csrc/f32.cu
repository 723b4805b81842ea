// f32.cu — the fp32 debug-parity path (pb_model_desc.dtype = PB_DTYPE_F32): the same cold start with fp32
// weights, LoRA factors and activations, every product on CUDA-core FFMA.
//
// It exists for the north star's second tolerance gate ("1e-4 (fp32) for merged weights and first-token
// logits", SURVEY.md §8(c) "Tolerances"): with fp32 storage the only differences from the oracle's fp64
// arithmetic are fp32 roundings, so merged weights and logits must agree to 1e-4 relative. Not timed and
// not tuned — plain tiled SIMT kernels, one launcher per step of the layer:
//   merge   W' = fl(W + s * sum_k B[i,k] A[k,j])
//   gemm    out = X W^T (+ bias, q-scale, ReLU | residual add | SiLU(gate) * up)
//   norm    LayerNorm / RMSNorm rows -> fp32
//   embed   h = E[tok] (+ P[pos + 2])
//   rope    rotate_half in place on fp32 q / k
//   attention causal, online softmax, one warp per (query, head)
//   logits  y . E[v] for a vocab slice
#include <math_constants.h>

#include "kernels.hpp"

namespace pb {

namespace {

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ merge
__global__ void merge_f32_kernel(const float* __restrict__ W, float* __restrict__ Wout, int64_t ldw, int rows,
                                 int cols, const float* __restrict__ B, const float* __restrict__ A, int r,
                                 float scale) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (j >= cols || i >= rows) return;
    float acc = 0.f;
    for (int k = 0; k < r; ++k) acc = fmaf(B[(size_t)i * r + k], A[(size_t)k * cols + j], acc);
    Wout[(size_t)i * ldw + j] = fmaf(scale, acc, W[(size_t)i * ldw + j]);
}

// ------------------------------------------------------------------ GEMM: 64 x 64 tile, 256 threads, 4 x 4 each
constexpr int TM = 64, TN = 64, TK = 16;
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ X, int ldx, int M_begin, int M_end,
                                                       const float* __restrict__ W, int N, int K, int epi,
                                                       const float* __restrict__ bias, int relu, float scale,
                                                       int scale_cols, float* __restrict__ out, int ldo,
                                                       int up_row0) {
    __shared__ float sX[TK][TM + 1];
    __shared__ float sW[TK][TN + 1];
    __shared__ float sU[TK][TN + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = M_begin + blockIdx.y * TM, n0 = blockIdx.x * TN;
    float acc[4][4] = {}, accu[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += TK) {
        for (int e = threadIdx.x; e < TK * TM; e += 256) {
            const int kk = e % TK, mm = e / TK;
            const int row = m0 + mm, k = k0 + kk;
            sX[kk][mm] = (row < M_end && k < K) ? X[(size_t)row * ldx + k] : 0.f;
            const int n = n0 + mm;
            sW[kk][mm] = (n < N && k < K) ? W[(size_t)n * K + k] : 0.f;
            if (epi == EPI_SILU_MUL) sU[kk][mm] = (n < N && k < K) ? W[(size_t)(up_row0 + n) * K + k] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            float xa[4], wb[4], ub[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                xa[i] = sX[kk][ty * 4 + i];
                wb[i] = sW[kk][tx * 4 + i];
                ub[i] = epi == EPI_SILU_MUL ? sU[kk][tx * 4 + i] : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[i][q] = fmaf(xa[i], wb[q], acc[i][q]);
                    if (epi == EPI_SILU_MUL) accu[i][q] = fmaf(xa[i], ub[q], accu[i][q]);
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + ty * 4 + i;
        if (row >= M_end) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int n = n0 + tx * 4 + q;
            if (n >= N) continue;
            float v = acc[i][q];
            float* o = out + (size_t)row * ldo + n;
            if (epi == EPI_SILU_MUL) {
                *o = v / (1.0f + expf(-v)) * accu[i][q];
                continue;
            }
            if (bias) v += bias[n];
            if (epi == EPI_RESID) {
                *o += v;
                continue;
            }
            if (n < scale_cols) v *= scale;
            if (relu) v = fmaxf(v, 0.f);
            *o = v;
        }
    }
}

// ------------------------------------------------------------------ norm: one CTA per row
__global__ void __launch_bounds__(256) norm_f32_kernel(const float* __restrict__ h, int ldh, float* __restrict__ out,
                                                       int ldo, int d, const float* __restrict__ gamma,
                                                       const float* __restrict__ beta, float eps) {
    __shared__ float red[8];
    const float* x = h + (size_t)blockIdx.x * ldh;
    auto block_sum = [&](float v) {
        v = warp_sum_f(v);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += red[w];
        __syncthreads();
        return t;
    };
    float mu = 0.f;
    if (beta) {
        float s = 0.f;
        for (int c = threadIdx.x; c < d; c += 256) s += x[c];
        mu = block_sum(s) / d;
    }
    float s2 = 0.f;
    for (int c = threadIdx.x; c < d; c += 256) {
        const float v = x[c] - mu;
        s2 += v * v;
    }
    const float rstd = rsqrtf(block_sum(s2) / d + eps);
    float* o = out + (size_t)blockIdx.x * ldo;
    for (int c = threadIdx.x; c < d; c += 256) o[c] = (x[c] - mu) * rstd * gamma[c] + (beta ? beta[c] : 0.f);
}

// ------------------------------------------------------------------ embed
__global__ void embed_f32_kernel(EmbedSrc E, const float* __restrict__ pos, const int32_t* __restrict__ tok,
                                 float* __restrict__ h, int d, int r0, int B) {
    const int row = r0 + blockIdx.x;
    const int v = tok[row];
    int o = 0;
    while (o + 1 < E.n && v >= E.slice_begin[o + 1]) ++o;
    // every owner's table pointer is the base of the WHOLE table (same offsets on every GPU); rows [slice) live there
    const float* e = static_cast<const float*>(E.base[o]) + (size_t)v * d;
    const float* p = pos ? pos + (size_t)(row / B + 2) * d : nullptr;
    for (int c = threadIdx.x; c < d; c += blockDim.x) h[(size_t)row * d + c] = e[c] + (p ? p[c] : 0.f);
}

// ------------------------------------------------------------------ RoPE (rotate_half), angles from the fp64 table
__global__ void rope_f32_kernel(float* qkv, int ld, int r0, int B, int n_q, int n_k, int hd, int k_col0,
                                const float2* __restrict__ table) {
    const int row = r0 + blockIdx.x, t = row / B, half = hd / 2;
    for (int e = threadIdx.x; e < (n_q + n_k) * half; e += blockDim.x) {
        const int hh = e / half, i = e % half;
        float* x = qkv + (size_t)row * ld + (hh < n_q ? hh * hd : k_col0 + (hh - n_q) * hd);
        const float2 cs = table[(size_t)t * half + i];
        const float a = x[i], b = x[i + half];
        x[i] = a * cs.x - b * cs.y;
        x[i + half] = b * cs.x + a * cs.y;
    }
}

// ------------------------------------------------------------------ attention: one warp per (query t, head h, seq b)
__global__ void attention_f32_kernel(const float* __restrict__ qkv, int ld, float* __restrict__ out, int ldo, int t0,
                                     int t1, int B, int H, int group, int hd, int k_col0, int v_col0, float scale) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nq = t1 - t0;
    if (warp >= nq * H * B) return;
    const int t = t0 + warp % nq, h = (warp / nq) % H, b = warp / (nq * H), kvh = h / group;
    const float* q = qkv + ((size_t)t * B + b) * ld + h * hd;
    float m = -CUDART_INF_F, l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};   // hd <= 128: 4 dims per lane
    for (int j = 0; j <= t; ++j) {
        const float* kr = qkv + ((size_t)j * B + b) * ld + k_col0 + kvh * hd;
        float s = 0.f;
        for (int c = lane; c < hd; c += 32) s = fmaf(q[c], kr[c], s);
        s = warp_sum_f(s) * scale;
        const float m_new = fmaxf(m, s);
        const float corr = expf(m - m_new), p = expf(s - m_new);
        l = l * corr + p;
        const float* vr = qkv + ((size_t)j * B + b) * ld + v_col0 + kvh * hd;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = lane + 32 * e;
            acc[e] = acc[e] * corr + (c < hd ? p * vr[c] : 0.f);
        }
        m = m_new;
    }
    float* o = out + ((size_t)t * B + b) * ldo + h * hd;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int c = lane + 32 * e;
        if (c < hd) o[c] = acc[e] / l;
    }
}

// ------------------------------------------------------------------ logits: one warp per vocab row
__global__ void logits_f32_kernel(const float* __restrict__ y, int B, int d, const float* __restrict__ E, int v0,
                                  int v1, float* __restrict__ logits, int ldl) {
    const int v = v0 + (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
    if (v >= v1) return;
    const float* e = E + (size_t)v * d;
    for (int b = 0; b < B; ++b) {
        float s = 0.f;
        for (int c = lane; c < d; c += 32) s = fmaf(y[(size_t)b * d + c], e[c], s);
        s = warp_sum_f(s);
        if (lane == 0) logits[(size_t)b * ldl + v] = s;
    }
}

}  // namespace

cudaError_t launch_merge_f32(const float* W, float* Wout, int64_t ldw, int rows, int cols, const float* B,
                             const float* A, int rank, float scale, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    merge_f32_kernel<<<dim3((cols + 255) / 256, rows), 256, 0, s>>>(W, Wout, ldw, rows, cols, B, A, rank, scale);
    return cudaGetLastError();
}

cudaError_t launch_gemm_f32(const float* X, int ldx, int M_begin, int M_end, const float* W, int N, int K, int epi,
                            const float* bias, int relu, float scale, int scale_cols, float* out, int ldo, int up_row0,
                            cudaStream_t s) {
    if (M_end <= M_begin || N <= 0) return cudaSuccess;
    const dim3 grid((N + TN - 1) / TN, (M_end - M_begin + TM - 1) / TM);
    gemm_f32_kernel<<<grid, 256, 0, s>>>(X, ldx, M_begin, M_end, W, N, K, epi, bias, relu, scale, scale_cols, out,
                                         ldo, up_row0);
    return cudaGetLastError();
}

cudaError_t launch_norm_f32(const float* h, int ldh, float* out, int ldo, int rows, int d, const float* gamma,
                            const float* beta, float eps, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    norm_f32_kernel<<<rows, 256, 0, s>>>(h, ldh, out, ldo, d, gamma, beta, eps);
    return cudaGetLastError();
}

cudaError_t launch_embed_f32(const EmbedSrc& E, const float* pos, const int32_t* tok, float* h, int d, int r0, int r1,
                             int B, cudaStream_t s) {
    if (r1 <= r0) return cudaSuccess;
    embed_f32_kernel<<<r1 - r0, 256, 0, s>>>(E, pos, tok, h, d, r0, B);
    return cudaGetLastError();
}

cudaError_t launch_rope_f32(float* qkv, int ld, int r0, int r1, int B, int n_q, int n_k, int hd, int k_col0,
                            const float2* table, cudaStream_t s) {
    if (r1 <= r0) return cudaSuccess;
    rope_f32_kernel<<<r1 - r0, 256, 0, s>>>(qkv, ld, r0, B, n_q, n_k, hd, k_col0, table);
    return cudaGetLastError();
}

cudaError_t launch_attention_f32(const float* qkv, int ld, float* out, int ldo, int t0, int t1, int B, int n_heads,
                                 int n_kv_heads, int hd, int k_col0, int v_col0, float score_scale, cudaStream_t s) {
    if (t1 <= t0) return cudaSuccess;
    if (hd > 128) return cudaErrorInvalidValue;
    const long warps = (long)(t1 - t0) * n_heads * B;
    attention_f32_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(
        qkv, ld, out, ldo, t0, t1, B, n_heads, n_heads / n_kv_heads, hd, k_col0, v_col0, score_scale);
    return cudaGetLastError();
}

cudaError_t launch_logits_f32(const float* y, int B, int d, const float* E, int v0, int v1, float* logits, int ldl,
                              cudaStream_t s) {
    if (v1 <= v0) return cudaSuccess;
    logits_f32_kernel<<<(unsigned)(((long)(v1 - v0) * 32 + 255) / 256), 256, 0, s>>>(y, B, d, E, v0, v1, logits, ldl);
    return cudaGetLastError();
}

cudaError_t warm_f32_kernels() {
    cudaFuncAttributes a;
    const void* fns[] = {(const void*)merge_f32_kernel,  (const void*)gemm_f32_kernel,      (const void*)norm_f32_kernel,
                         (const void*)embed_f32_kernel,  (const void*)rope_f32_kernel,      (const void*)attention_f32_kernel,
                         (const void*)logits_f32_kernel};
    for (const void* f : fns) {
        cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace pb
