// simt.cu — the non-GEMM prefill kernels (CUDA cores): norms, embedding gather, RoPE, causal attention,
// vocab-parallel logits, argmax, and the cross-rank readiness signal.
//
// All are memory- or latency-bound row kernels: coalesced 16-byte accesses, fp32 statistics with
// warp-shuffle reductions, one CTA (or one warp) per row.
#include <cuda_bf16.h>
#include <math_constants.h>

#include <cstdlib>

#include "kernels.hpp"
#include "rownorm.cuh"
#include "sm100.cuh"

namespace pb {
using namespace sm100;

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float t = (l < NT / 32) ? red[l] : 0.f;
    return warp_sum(t);
}

// ------------------------------------------------------------------ LayerNorm / RMSNorm
// One CTA of 256 threads per row, the row held in registers: thread t owns the 8-element groups t, t + 256, ...
// (G groups, d <= 256 * 8 * G), read as two 16-byte fp32 vectors and written as one 16-byte bf16 vector; gamma /
// beta arrive as 16-byte bf16 vectors requested before the programmatic-dependency wait (they are weights,
// resident before the kernel is enqueued). Two-pass fp32 statistics (rownorm.cuh): mean, then the mean of squared
// deviations, each summed per thread in element order, then by a warp butterfly and over the 8 warps.
template <int G>
__global__ void __launch_bounds__(256, G >= 3 ? 4 : 1) norm_kernel(const float* __restrict__ h, int ldh, __nv_bfloat16* __restrict__ out,
                                                   int ldo, int d, const __nv_bfloat16* __restrict__ gamma,
                                                   const __nv_bfloat16* __restrict__ beta, float eps, const int* dyn,
                                                   int dyn_in, int dyn_out) {
    constexpr int NT = 256;
    static_assert(NT == rownorm::kVT, "8 warps per row (rownorm::combine8)");
    pdl_launch_dependents();   // a PDL-launched GEMM may start its weight prefetch
    const int ng = d >> 3;     // 8-element groups in the row
    // Small rows (G <= 2, the latency-bound small-M regime): gamma / beta in registers before the dependency wait.
    // Large rows (G >= 3, e.g. d = 8192 at M = 2048, bandwidth-bound): fetched at the output (L2-resident, shared by
    // every row), which frees 8 G registers per thread for 4 resident CTAs per SM (more row loads in flight).
    constexpr bool kPreGB = G <= 2;
    uint4 gm[kPreGB ? G : 1], bt[kPreGB ? G : 1];
    if constexpr (kPreGB) {
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const int g = threadIdx.x + i * NT;
            gm[i] = g < ng ? __ldg(reinterpret_cast<const uint4*>(gamma) + g) : make_uint4(0, 0, 0, 0);
            bt[i] = g < ng && beta ? __ldg(reinterpret_cast<const uint4*>(beta) + g) : make_uint4(0, 0, 0, 0);
        }
    }
    pdl_wait();                // PDL-launched: the previous kernel's output is visible from here on
    __shared__ float red[32];
    long long row = blockIdx.x, orow = blockIdx.x;
    if (dyn != nullptr) {
        const long long t = *dyn;
        row += t * dyn_in;
        orow += t * dyn_out;
    }
    const float4* x = reinterpret_cast<const float4*>(h + row * (long long)ldh);
    float v[G][8];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int g = threadIdx.x + i * NT;
        float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
        if (g < ng) {
            lo = x[2 * g];
            hi = x[2 * g + 1];
        }
        v[i][0] = lo.x; v[i][1] = lo.y; v[i][2] = lo.z; v[i][3] = lo.w;
        v[i][4] = hi.x; v[i][5] = hi.y; v[i][6] = hi.z; v[i][7] = hi.w;
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    float mean = 0.f;
    if (beta) {
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < G; ++i)
            if (threadIdx.x + i * NT < ng) {
#pragma unroll
                for (int e = 0; e < 8; ++e) s = rownorm::acc_sum(s, v[i][e]);
            }
        s = rownorm::warp_sum(s);
        if (l == 0) red[w] = s;
        __syncthreads();
        mean = rownorm::mean_of(rownorm::combine8(red, l), d);
        __syncthreads();
    }
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < G; ++i)
        if (threadIdx.x + i * NT < ng) {
#pragma unroll
            for (int e = 0; e < 8; ++e) q = rownorm::acc_sq(q, v[i][e], mean);
        }
    q = rownorm::warp_sum(q);
    if (l == 0) red[w] = q;
    __syncthreads();
    const float rstd = rownorm::rstd_of(rownorm::combine8(red, l), d, eps);
    uint4* o = reinterpret_cast<uint4*>(out + orow * (long long)ldo);
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int g = threadIdx.x + i * NT;
        if (g >= ng) continue;
        uint4 gq, bq;
        if constexpr (kPreGB) {
            gq = gm[i];
            bq = bt[i];
        } else {
            gq = __ldg(reinterpret_cast<const uint4*>(gamma) + g);
            bq = beta ? __ldg(reinterpret_cast<const uint4*>(beta) + g) : make_uint4(0, 0, 0, 0);
        }
        const __nv_bfloat16* gp = reinterpret_cast<const __nv_bfloat16*>(&gq);
        const __nv_bfloat16* bp = reinterpret_cast<const __nv_bfloat16*>(&bq);
        uint4 r;
        uint16_t* rp = reinterpret_cast<uint16_t*>(&r);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const __nv_bfloat16 y = rownorm::out_f(v[i][e], mean, rstd, __bfloat162float(gp[e]),
                                                   __bfloat162float(bp[e]), beta != nullptr);
            rp[e] = *reinterpret_cast<const uint16_t*>(&y);
        }
        o[g] = r;
    }
}

// ------------------------------------------------------------------ embedding (+ OPT learned positions)
__global__ void embed_kernel(EmbedSrc E, const __nv_bfloat16* __restrict__ pos, const int32_t* __restrict__ tok,
                             float* __restrict__ h, int d, int r0, int B, const int* dyn) {
    pdl_launch_dependents();
    pdl_wait();
    const int row = r0 + blockIdx.x + (dyn ? *dyn * B : 0);
    const int t = row / B;
    const int id = tok[row];
    int owner = 0;
    while (owner + 1 < E.n && id >= E.slice_begin[owner + 1]) ++owner;
    const __nv_bfloat16* e = static_cast<const __nv_bfloat16*>(E.base[owner]) + (size_t)id * d;
    const __nv_bfloat16* p = pos ? pos + (size_t)(t + 2) * d : nullptr;   // HF OPT position offset 2
    float* o = h + (size_t)row * d;
    for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
        uint4 ev = *reinterpret_cast<const uint4*>(e + c);
        const __nv_bfloat16* eb = reinterpret_cast<const __nv_bfloat16*>(&ev);
        float f[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(eb[i]);
        if (p) {
            uint4 pv = *reinterpret_cast<const uint4*>(p + c);
            const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&pv);
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] += __bfloat162float(pb[i]);
        }
        reinterpret_cast<float4*>(o + c)[0] = make_float4(f[0], f[1], f[2], f[3]);
        reinterpret_cast<float4*>(o + c)[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
}

// ------------------------------------------------------------------ RoPE
__global__ void rope_table_kernel(float2* table, int T, int hd, double theta) {
    const int half = hd / 2;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= T * half) return;
    const int t = idx / half, i = idx % half;
    const double inv_freq = pow(theta, -2.0 * i / (double)hd);
    double sv, cv;
    sincos((double)t * inv_freq, &sv, &cv);
    table[idx] = make_float2((float)cv, (float)sv);
}

// x'_i = x_i cos - x_{i+hd/2} sin ; x'_{i+hd/2} = x_{i+hd/2} cos + x_i sin   (HF rotate_half)
__global__ void rope_kernel(__nv_bfloat16* qkv, int ld, int r0, int B, int n_q, int n_k, int hd, int k_col0,
                            const float2* __restrict__ table, const int* dyn) {
    pdl_launch_dependents();   // a PDL-launched GEMM may start its weight prefetch
    pdl_wait();                // PDL-launched: the previous kernel's output is visible from here on
    const int row = r0 + blockIdx.x + (dyn ? *dyn * B : 0);
    const int t = row / B;
    const int half = hd / 2;
    const int total = (n_q + n_k) * half;
    __nv_bfloat16* base = qkv + (size_t)row * ld;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int head = idx / half, i = idx % half;
        __nv_bfloat16* x = head < n_q ? base + head * hd : base + k_col0 + (head - n_q) * hd;
        const float2 cs = table[t * half + i];
        const float a = __bfloat162float(x[i]), b = __bfloat162float(x[i + half]);
        x[i] = __float2bfloat16_rn(a * cs.x - b * cs.y);
        x[i + half] = __float2bfloat16_rn(b * cs.x + a * cs.y);
    }
}

// ------------------------------------------------------------------ causal attention (flash-style, SIMT)
// CTA = (32 query positions, head, sequence); 8 warps x 4 queries. Keys/values streamed through shared
// memory 32 at a time (K transposed for conflict-free lane-per-key dot products); online softmax in fp32.
template <int HD>
__global__ void __launch_bounds__(256, 2) attention_kernel(const __nv_bfloat16* __restrict__ qkv, int ld,
                                                        __nv_bfloat16* __restrict__ out, int ldo, int t0, int t1,
                                                        int B, int group, int k_col0, int v_col0,
                                                        float score_scale) {
    pdl_launch_dependents();   // a PDL-launched GEMM may start its weight prefetch
    pdl_wait();                // PDL-launched: the previous kernel's output is visible from here on
    constexpr int KT = 32, QT = 32, DPL = HD / 32;   // dims per lane
    extern __shared__ float attn_smem[];
    float (*sQ)[HD] = reinterpret_cast<float (*)[HD]>(attn_smem);
    float (*sKt)[KT + 1] = reinterpret_cast<float (*)[KT + 1]>(attn_smem + QT * HD);
    float (*sV)[HD] = reinterpret_cast<float (*)[HD]>(attn_smem + QT * HD + HD * (KT + 1));
    const int b = blockIdx.z, h = blockIdx.y, kvh = h / group;
    const int q0 = t0 + blockIdx.x * QT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q_hi = min(q0 + QT, t1);   // exclusive
    // load Q tile
    for (int i = threadIdx.x; i < QT * HD; i += 256) {
        const int qi = i / HD, c = i % HD;
        const int t = q0 + qi;
        sQ[qi][c] = t < t1 ? __bfloat162float(qkv[(size_t)(t * B + b) * ld + h * HD + c]) * score_scale : 0.f;
    }
    float m[4], l[4], acc[4][DPL];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        m[i] = -CUDART_INF_F;
        l[i] = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[i][e] = 0.f;
    }
    const int n_keys = q_hi;   // keys [0, q_hi) cover every query in the tile
    const int qw0 = q0 + warp * 4;   // this warp's 4 queries (independent FMA chains -> ILP)
    for (int k0 = 0; k0 < n_keys; k0 += KT) {
        __syncthreads();
        for (int i = threadIdx.x; i < KT * HD; i += 256) {
            const int kj = i / HD, c = i % HD;
            const int t = k0 + kj;
            float kv = 0.f, vv = 0.f;
            if (t < n_keys) {
                const __nv_bfloat16* r = qkv + (size_t)(t * B + b) * ld;
                kv = __bfloat162float(r[k_col0 + kvh * HD + c]);
                vv = __bfloat162float(r[v_col0 + kvh * HD + c]);
            }
            sKt[c][kj] = kv;
            sV[kj][c] = vv;
        }
        __syncthreads();
        if (qw0 >= q_hi || k0 > qw0 + 3) continue;   // warp-uniform: no live query or keys all in the future
        const int key = k0 + lane;
        float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
        for (int c = 0; c < HD; ++c) {
            const float kt = sKt[c][lane];
#pragma unroll
            for (int i = 0; i < 4; ++i) sc[i] = fmaf(sQ[warp * 4 + i][c], kt, sc[i]);
        }
        float p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int t = qw0 + i;
            float sv = (key > t || t >= q_hi) ? -CUDART_INF_F : sc[i];
            const float mx = warp_max(sv);
            const float m_new = fmaxf(m[i], mx);
            if (m_new == -CUDART_INF_F) {   // nothing visible yet for this query
                p[i] = 0.f;
                continue;
            }
            p[i] = __expf(sv - m_new);
            const float corr = __expf(m[i] - m_new);
            l[i] = l[i] * corr + warp_sum(p[i]);
            m[i] = m_new;
#pragma unroll
            for (int e = 0; e < DPL; ++e) acc[i][e] *= corr;
        }
#pragma unroll 4
        for (int j = 0; j < KT; ++j) {
            float vj[DPL];
#pragma unroll
            for (int e = 0; e < DPL; ++e) vj[e] = sV[j][lane + 32 * e];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float pj = __shfl_sync(0xffffffffu, p[i], j);
#pragma unroll
                for (int e = 0; e < DPL; ++e) acc[i][e] = fmaf(pj, vj[e], acc[i][e]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int t = q0 + warp * 4 + i;
        if (t >= q_hi) continue;
        const float inv = 1.f / l[i];
        __nv_bfloat16* o = out + (size_t)(t * B + b) * ldo + h * HD;
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[lane + 32 * e] = __float2bfloat16_rn(acc[i][e] * inv);
    }
}

// ------------------------------------------------------------------ vocab-parallel logits
// One warp per vocabulary row; y (B <= 8 rows) staged in shared memory as fp32.
__global__ void __launch_bounds__(256) logits_kernel(const __nv_bfloat16* __restrict__ y, int B, int d,
                                                     const __nv_bfloat16* __restrict__ E, int v0, int v1,
                                                     float* __restrict__ logits, int ldl) {
    // One warp per vocabulary row. Lane l accumulates columns l*8 + 256 k in ascending order; the row's 16-B
    // vectors are requested in groups of 8 before any is used, the first group before the programmatic-dependency
    // wait (the head weights are resident; y is the previous kernel's output). y (B x d bf16, a few KB) is read
    // through L1.
    pdl_launch_dependents();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int v = v0 + blockIdx.x * 8 + warp;
    constexpr int G = 8;
    const int nvec = d / 8;   // 16-B vectors per row
    const __nv_bfloat16* e = E + (size_t)(v < v1 ? v : v0) * d;
    uint4 ev[G];
    auto load_group = [&](int k0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int vec = (k0 + g) * 32 + lane;
            ev[g] = vec < nvec ? __ldg(reinterpret_cast<const uint4*>(e) + vec) : make_uint4(0, 0, 0, 0);
        }
    };
    load_group(0);
    pdl_wait();
    if (v >= v1) return;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k0 = 0; k0 * 32 < nvec; k0 += G) {
        if (k0 > 0) load_group(k0);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int vec = (k0 + g) * 32 + lane;
            if (vec >= nvec) break;
            const __nv_bfloat16* eb = reinterpret_cast<const __nv_bfloat16*>(&ev[g]);
            float f[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(eb[i]);
            for (int b = 0; b < B; ++b) {
                const uint4 yv = __ldg(reinterpret_cast<const uint4*>(y + (size_t)b * d) + vec);
                const __nv_bfloat16* yb = reinterpret_cast<const __nv_bfloat16*>(&yv);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[b] = fmaf(f[i], __bfloat162float(yb[i]), acc[b]);
            }
        }
    }
    for (int b = 0; b < B; ++b) {
        const float s2 = warp_sum(acc[b]);
        if (lane == 0) logits[(size_t)b * ldl + v] = s2;
    }
}

// ------------------------------------------------------------------ argmax (lowest index wins ties)
// A cluster of AM_CTAS CTAs per sequence: CTA c scans the c-th slice of the row with 8 loads in flight per thread,
// reduces it (butterfly per warp, then over the warps), and CTA 0 combines the slices' (value, index) pairs through
// distributed shared memory. The (value, lowest index) maximum does not depend on the visiting order.
constexpr int AM_CTAS = 8;

__device__ __forceinline__ void am_better(float& best, int& bi, float ov, int oi) {
    if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
    }
}

__global__ void __launch_bounds__(1024) argmax_kernel(const float* __restrict__ logits, int V, int ldl,
                                                      int32_t* tokens, int32_t* nan_flag) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ float sv[32];
    __shared__ int si[32];
    __shared__ float cv;   // this CTA's slice result, read by CTA 0 of the cluster
    __shared__ int ci;
    uint32_t crank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const float* x = logits + (size_t)blockIdx.y * ldl;
    const int per = (V + AM_CTAS - 1) / AM_CTAS, lo = (int)crank * per, hi = min(V, lo + per);
    float best = -CUDART_INF_F;
    int bi = 0x7fffffff;
    bool bad = false;
    constexpr int U = 8;
    for (int v = lo + threadIdx.x; v < hi; v += U * blockDim.x) {
        float f[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int vv = v + u * blockDim.x;
            f[u] = vv < hi ? x[vv] : -CUDART_INF_F;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int vv = v + u * blockDim.x;
            if (vv >= hi) break;
            if (!isfinite(f[u])) bad = true;
            am_better(best, bi, f[u], vv);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        am_better(best, bi, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bi, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sv[w] = best; si[w] = bi; }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nan_flag, 1);
    if (w == 0) {
        best = l < (blockDim.x >> 5) ? sv[l] : -CUDART_INF_F;
        bi = l < (blockDim.x >> 5) ? si[l] : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            am_better(best, bi, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bi, o));
        if (l == 0) { cv = best; ci = bi; }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (crank == 0 && w == 0) {
        float ov = -CUDART_INF_F;
        int oi = 0x7fffffff;
        if (l < AM_CTAS) {
            uint32_t av, ai;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(av) : "r"((uint32_t)__cvta_generic_to_shared(&cv)), "r"(l));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ai) : "r"((uint32_t)__cvta_generic_to_shared(&ci)), "r"(l));
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(ov) : "r"(av) : "memory");
            asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(oi) : "r"(ai) : "memory");
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            am_better(ov, oi, __shfl_xor_sync(0xffffffffu, ov, o), __shfl_xor_sync(0xffffffffu, oi, o));
        if (l == 0) tokens[blockIdx.y] = oi == 0x7fffffff ? 0 : oi;
    }
    // keep every CTA's shared slice result alive until CTA 0 has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ------------------------------------------------------------------ cross-rank readiness words
__global__ void signal_kernel(SignalTargets t, uint32_t value) {
    const int i = threadIdx.x;
    if (i < t.n) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(t.addr[i]), "r"(value) : "memory");
    }
}

// Re-plan resume: publish `value` into words base[idx[i]] (a peer's chunk readiness words for the chunks this
// rank already holds), one thread per word.
__global__ void set_words_kernel(uint32_t* base, const int32_t* __restrict__ idx, int n, uint32_t value) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(base + idx[i]), "r"(value) : "memory");
    }
}

__global__ void feed_tokens_kernel(int32_t* tokens, const int32_t* __restrict__ tok_out, const int* dyn, int B) {
    const int b = threadIdx.x;
    if (b < B) tokens[*dyn * B + b] = tok_out[b];
}

}  // namespace

cudaError_t launch_feed_tokens(int32_t* tokens, const int32_t* tok_out, const int* dyn, int B, cudaStream_t s) {
    feed_tokens_kernel<<<1, 32, 0, s>>>(tokens, tok_out, dyn, B);
    return cudaGetLastError();
}

cudaError_t launch_set_words(uint32_t* base, const int32_t* idx, int n, uint32_t value, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    set_words_kernel<<<(n + 255) / 256, 256, 0, s>>>(base, idx, n, value);
    return cudaGetLastError();
}

cudaError_t warm_simt_kernels() {
    cudaFuncAttributes a;
    const void* fns[] = {(const void*)norm_kernel<1>, (const void*)norm_kernel<2>, (const void*)norm_kernel<3>,
                         (const void*)norm_kernel<4>, (const void*)norm_kernel<5>, (const void*)embed_kernel,
                         (const void*)rope_table_kernel, (const void*)rope_kernel, (const void*)attention_kernel<32>,
                         (const void*)attention_kernel<64>, (const void*)attention_kernel<128>,
                         (const void*)logits_kernel, (const void*)argmax_kernel, (const void*)signal_kernel,
                         (const void*)set_words_kernel, (const void*)feed_tokens_kernel};
    for (const void* f : fns) {
        cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_norm(const float* h, int ldh, __nv_bfloat16* out, int ldo, int rows, int d,
                        const __nv_bfloat16* gamma, const __nv_bfloat16* beta, float eps, cudaStream_t s, bool pdl,
                        const int* dyn, int dyn_in, int dyn_out) {
    if (rows <= 0) return cudaSuccess;
    // 16-byte vectors: d % 8 == 0 and 16-byte aligned rows / gamma / beta (every path buffer is)
    if (d % 8 || ldh % 4 || ldo % 8 || (reinterpret_cast<uintptr_t>(h) & 15) || (reinterpret_cast<uintptr_t>(out) & 15) ||
        (reinterpret_cast<uintptr_t>(gamma) & 15) || (reinterpret_cast<uintptr_t>(beta) & 15))
        return cudaErrorInvalidValue;
    const int groups = (d / 8 + 255) / 256;
#define PB_NORM_CASE(G)                                                                                                \
    case G:                                                                                                            \
        return launch_pdl(norm_kernel<G>, rows, 256, 0, s, pdl, h, ldh, out, ldo, d, gamma, beta, eps, dyn, dyn_in,   \
                          dyn_out);
    switch (groups) {
        PB_NORM_CASE(1)
        PB_NORM_CASE(2)
        PB_NORM_CASE(3)
        PB_NORM_CASE(4)
        PB_NORM_CASE(5)
    }
#undef PB_NORM_CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_embed(const EmbedSrc& E, const __nv_bfloat16* pos, const int32_t* tok, float* h, int d, int r0,
                         int r1, int B, cudaStream_t s, bool pdl, const int* dyn) {
    if (r1 <= r0) return cudaSuccess;
    if (d % 8) return cudaErrorInvalidValue;
    return launch_pdl(embed_kernel, r1 - r0, 128, 0, s, pdl, E, pos, tok, h, d, r0, B, dyn);
}

cudaError_t launch_rope_table(float2* table, int T, int hd, double theta, cudaStream_t s) {
    const int n = T * (hd / 2);
    if (n <= 0) return cudaSuccess;
    rope_table_kernel<<<(n + 255) / 256, 256, 0, s>>>(table, T, hd, theta);
    return cudaGetLastError();
}

cudaError_t launch_rope(__nv_bfloat16* qkv, int ld, int r0, int r1, int B, int n_q, int n_k, int hd, int k_col0,
                        const float2* table, cudaStream_t s, bool pdl, const int* dyn) {
    if (r1 <= r0) return cudaSuccess;
    return launch_pdl(rope_kernel, r1 - r0, 256, 0, s, pdl, qkv, ld, r0, B, n_q, n_k, hd, k_col0, table, dyn);
}

// ------------------------------------------------------------------ decode attention (one query position)
// One new position per sequence (f3 decode steps): a 128-query tensor-core tile would be 127/128 padding and
// its two passes over the key tiles are a chain of MMA / softmax handshakes per tile. Here a cluster of CL CTAs of 16
// warps serves one (head, sequence), CTA r taking the contiguous key block r of CL, with the storage contract's
// exact normalised-P rounding:
//   scores  s_j = q . k_j (fp32, one thread per key, the key's vectors all requested before the FMAs), kept in smem;
//   m = max s over the cluster, E_j = exp2(s_j c - m c), l = sum E (block sums, then the CL block values added in rank
//   order through distributed shared memory: every CTA gets the same l);
//   O = sum_j RNE_bf16(E_j / l) v_j (warps take keys w, w + 16, ... of the block, lanes the head dims; 16 warp
//   partials added in warp order, then the CL block partials in rank order — CTA r finishing dims r of CL);
//   out = RNE_bf16(O). dyn (decode graphs): positions read on the device. Keys [0, t] of the position t = t1 - 1.
constexpr int DA_WARPS = 16, kDecodeMaxKeys = 12288;

__device__ __forceinline__ uint32_t da_cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void da_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float da_ld_remote(const float* p, uint32_t rank) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p)), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
    return v;
}

template <int HD, int CL>
__global__ void __launch_bounds__(DA_WARPS * 32) decode_attention_kernel(const __nv_bfloat16* __restrict__ qkv, int ld,
                                                                         __nv_bfloat16* __restrict__ out, int ldo,
                                                                         int t1, int B, int group, int k_col0,
                                                                         int v_col0, float scale_log2, const int* dyn) {
    pdl_launch_dependents();
    extern __shared__ float da_smem[];
    constexpr int NT = DA_WARPS * 32, VPR = HD / 8, DPL = HD / 32;   // 16-B vectors per row, dims per lane
    float* red = da_smem;                        // [DA_WARPS]
    float* xch = da_smem + DA_WARPS;             // [2]: this CTA's block max / block sum (read by the cluster)
    float* opart = da_smem + 32;                 // [DA_WARPS][HD]; row 0 then holds the CTA's block partial of O
    float* sq = opart + DA_WARPS * HD;           // [HD] query
    float* sc = sq + HD;                         // [keys of this block]
    const int h = blockIdx.x / CL, b = blockIdx.y, kvh = h / group;
    const uint32_t rank = CL > 1 ? da_cluster_rank() : 0u;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (dyn) t1 += *dyn;
    pdl_wait();
    const int t = t1 - 1, nk = t + 1;
    const int j0 = (int)((long long)nk * rank / CL), j1 = (int)((long long)nk * (rank + 1) / CL), nb = j1 - j0;
    const __nv_bfloat16* qrow = qkv + ((size_t)t * B + b) * ld + h * HD;
    for (int d = tid; d < HD; d += NT) sq[d] = __bfloat162float(qrow[d]);
    __syncthreads();
    // ---- scores of this block: thread per key
    for (int jj = tid; jj < nb; jj += NT) {
        const uint4* krow = reinterpret_cast<const uint4*>(qkv + ((size_t)(j0 + jj) * B + b) * ld + k_col0 + kvh * HD);
        uint4 kv[VPR];
#pragma unroll
        for (int v = 0; v < VPR; ++v) kv[v] = __ldg(krow + v);
        float acc = 0.f;
#pragma unroll
        for (int v = 0; v < VPR; ++v) {
            const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(&kv[v]);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(sq[v * 8 + e], __bfloat162float(kb[e]), acc);
        }
        sc[jj] = acc;
    }
    __syncthreads();
    // ---- m = max s (exact in any order): block, then cluster
    float mx = -CUDART_INF_F;
    for (int jj = tid; jj < nb; jj += NT) mx = fmaxf(mx, sc[jj]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int w = 1; w < DA_WARPS; ++w) mx = fmaxf(mx, red[w]);
    if (CL > 1) {
        if (tid == 0) xch[0] = mx;
        da_cluster_sync();
        mx = da_ld_remote(xch, 0);
#pragma unroll
        for (uint32_t r = 1; r < CL; ++r) mx = fmaxf(mx, da_ld_remote(xch, r));
    }
    const float m = mx * scale_log2;
    __syncthreads();
    // ---- l = sum E: block sum in a fixed order, then the CL block sums in rank order
    float ls = 0.f;
    for (int jj = tid; jj < nb; jj += NT) {
        const float e = exp2f(fmaf(sc[jj], scale_log2, -m));
        sc[jj] = e;
        ls += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    if (lane == 0) red[warp] = ls;
    __syncthreads();
    float l = red[0];
#pragma unroll
    for (int w = 1; w < DA_WARPS; ++w) l += red[w];
    if (CL > 1) {
        if (tid == 0) xch[1] = l;
        da_cluster_sync();
        l = da_ld_remote(xch + 1, 0);
#pragma unroll
        for (uint32_t r = 1; r < CL; ++r) l += da_ld_remote(xch + 1, r);
    }
    const float inv_l = 1.f / l;
    // ---- this block's O = sum_j RNE_bf16(E_j / l) v_j: warp w takes keys w, w + 16, ...; lane the dims lane*DPL ..
    float o[DPL];
#pragma unroll
    for (int d = 0; d < DPL; ++d) o[d] = 0.f;
    constexpr int U = 4;
    for (int jb = warp; jb < nb; jb += DA_WARPS * U) {
        float vv[U][DPL], pp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int jj = jb + u * DA_WARPS;
            pp[u] = 0.f;
#pragma unroll
            for (int d = 0; d < DPL; ++d) vv[u][d] = 0.f;
            if (jj < nb) {
                const __nv_bfloat16* vrow = qkv + ((size_t)(j0 + jj) * B + b) * ld + v_col0 + kvh * HD + lane * DPL;
                if (DPL == 4) {
                    const uint2 w2 = __ldg(reinterpret_cast<const uint2*>(vrow));
                    const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&w2);
#pragma unroll
                    for (int d = 0; d < 4; ++d) vv[u][d] = __bfloat162float(vb[d]);
                } else {
                    const uint32_t w1 = __ldg(reinterpret_cast<const uint32_t*>(vrow));
                    const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&w1);
#pragma unroll
                    for (int d = 0; d < DPL; ++d) vv[u][d] = __bfloat162float(vb[d]);
                }
                pp[u] = __bfloat162float(__float2bfloat16_rn(sc[jj] * inv_l));   // P rounded after normalisation
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int d = 0; d < DPL; ++d) o[d] = fmaf(pp[u], vv[u][d], o[d]);
    }
#pragma unroll
    for (int d = 0; d < DPL; ++d) opart[warp * HD + lane * DPL + d] = o[d];
    __syncthreads();
    for (int d = tid; d < HD; d += NT) {   // the block partial: the 16 warp partials in warp order, into row 0
        float acc = opart[d];
#pragma unroll
        for (int w = 1; w < DA_WARPS; ++w) acc += opart[w * HD + d];
        opart[d] = acc;
    }
    __nv_bfloat16* orow = out + ((size_t)t * B + b) * ldo + h * HD;
    if (CL == 1) {
        __syncthreads();
        for (int d = tid; d < HD; d += NT) orow[d] = __float2bfloat16_rn(opart[d]);
        return;
    }
    da_cluster_sync();   // every block partial is complete
    for (int d = (int)rank * (HD / CL) + tid; d < (int)(rank + 1) * (HD / CL); d += NT) {
        float acc = da_ld_remote(opart + d, 0);
#pragma unroll
        for (uint32_t r = 1; r < CL; ++r) acc += da_ld_remote(opart + d, r);
        orow[d] = __float2bfloat16_rn(acc);
    }
    da_cluster_sync();   // peers stay alive until every remote read of their smem is done
}

template <int HD, int CL>
cudaError_t launch_decode_cl(const __nv_bfloat16* qkv, int ld, __nv_bfloat16* out, int ldo, int t1, int B, int H,
                             int group, int k_col0, int v_col0, float scale_log2, cudaStream_t s, bool pdl,
                             const int* dyn, int max_keys) {
    const int blk = (max_keys + CL - 1) / CL + 1;
    const int sm = (32 + DA_WARPS * HD + HD + blk) * (int)sizeof(float);
    const int sm_max = (32 + DA_WARPS * HD + HD + kDecodeMaxKeys / CL + 1) * (int)sizeof(float);   // set once
    cudaError_t e = smem_attr_once<decode_attention_kernel<HD, CL>>(sm_max);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(H * CL, B);
    cfg.blockDim = dim3(DA_WARPS * 32);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (CL > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CL;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, decode_attention_kernel<HD, CL>, qkv, ld, out, ldo, t1, B, group, k_col0, v_col0,
                              scale_log2, dyn);
}

// Cluster size from the context bound: ~250-400 keys per CTA, at most 8 (portable clusters). Measured
// (profiles/r02_decode_attention_ab.txt): C2 (<= 160 keys) CL 1 1.01 ms per token vs CL 2 1.08; C4 (~1060 keys)
// CL 4 5.83 ms vs CL 8 6.10, CL 2 6.42, tensor cores 6.80.
int decode_attention_cluster(int max_keys) {
    static const int forced = getenv("PB_DECODE_CL") ? atoi(getenv("PB_DECODE_CL")) : 0;   // experiments
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8) return forced;
    return max_keys <= 384 ? 1 : max_keys <= 768 ? 2 : max_keys <= 1600 ? 4 : 8;
}

cudaError_t launch_decode_attention(const __nv_bfloat16* qkv, int ld, __nv_bfloat16* out, int ldo, int t1, int B,
                                    int n_heads, int n_kv_heads, int hd, int k_col0, int v_col0, float score_scale,
                                    cudaStream_t s, bool pdl, const int* dyn, int max_keys) {
    if (max_keys > kDecodeMaxKeys) return cudaErrorInvalidValue;
    const int group = n_heads / n_kv_heads;
    const float scale_log2 = score_scale * 1.4426950408889634f;
    const int cl = decode_attention_cluster(max_keys);
#define PB_DEC(HDV, CLV)                                                                                           \
    if (hd == HDV && cl == CLV)                                                                                    \
        return launch_decode_cl<HDV, CLV>(qkv, ld, out, ldo, t1, B, n_heads, group, k_col0, v_col0, scale_log2, s, \
                                          pdl, dyn, max_keys);
    PB_DEC(64, 1) PB_DEC(64, 2) PB_DEC(64, 4) PB_DEC(64, 8)
    PB_DEC(128, 1) PB_DEC(128, 2) PB_DEC(128, 4) PB_DEC(128, 8)
#undef PB_DEC
    return cudaErrorNotSupported;
}

cudaError_t launch_attention_simt(const __nv_bfloat16* qkv, int ld, __nv_bfloat16* out, int ldo, int t0, int t1,
                                  int B, int n_heads, int n_kv_heads, int hd, int k_col0, int v_col0,
                                  float score_scale, cudaStream_t s) {
    if (t1 <= t0) return cudaSuccess;
    dim3 grid((t1 - t0 + 31) / 32, n_heads, B);
    const int group = n_heads / n_kv_heads;
    const int sm = (32 * hd + hd * 33 + 32 * hd) * (int)sizeof(float);
#define PB_ATTN(HD)                                                                                        \
    case HD: {                                                                                             \
        cudaError_t e = smem_attr_once<attention_kernel<HD>>(sm);                                            \
        if (e != cudaSuccess) return e;                                                                    \
        attention_kernel<HD><<<grid, 256, sm, s>>>(qkv, ld, out, ldo, t0, t1, B, group, k_col0, v_col0, score_scale); \
        break;                                                                                             \
    }
    switch (hd) {
        PB_ATTN(32)
        PB_ATTN(64)
        PB_ATTN(128)
        default: return cudaErrorInvalidValue;
    }
#undef PB_ATTN
    return cudaGetLastError();
}

cudaError_t launch_logits(const __nv_bfloat16* y, int B, int d, const __nv_bfloat16* E, int v0, int v1, float* logits,
                          int ldl, cudaStream_t s, bool pdl) {
    if (v1 <= v0) return cudaSuccess;
    if (d % 8) return cudaErrorInvalidValue;
    // a large batch (the paper's 64 x 64 workload) is a GEMM: the tensor cores read the head once
    // (C2p: 1.3 ms on the CUDA cores, 8 sequences per pass)
    if (B >= 16 && d % 64 == 0) return launch_logits_tc(y, B, d, E, v0, v1, logits, ldl, s);
    // one or two sequences (the cold start's first token, decode steps): the weight-streaming GEMV
    static const bool gemv_off = getenv("PB_LOGITS_GEMV") && atoi(getenv("PB_LOGITS_GEMV")) == 0;   // A/B
    if (B <= kGemvAutoRows && !gemv_off) return launch_logits_gemv(y, B, d, E, v0, v1, logits, ldl, s, pdl);
    // up to 8 sequences per launch (the warp's accumulators); larger batches (the paper's 64 x 64 workload)
    // stream the head once per group of 8
    for (int b0 = 0; b0 < B; b0 += 8) {
        const cudaError_t e = launch_pdl(logits_kernel, (v1 - v0 + 7) / 8, 256, 0, s, pdl, y + (size_t)b0 * d,
                                         std::min(8, B - b0), d, E, v0, v1, logits + (size_t)b0 * ldl, ldl);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_argmax(const float* logits, int B, int V, int ldl, int32_t* tokens, int32_t* nan_flag,
                          cudaStream_t s, bool pdl) {
    if (B <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(AM_CTAS, B);
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = AM_CTAS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, argmax_kernel, logits, V, ldl, tokens, nan_flag);
}

cudaError_t launch_signal(const SignalTargets& t, uint32_t value, cudaStream_t s) {
    if (t.n <= 0) return cudaSuccess;
    signal_kernel<<<1, 32, 0, s>>>(t, value);
    return cudaGetLastError();
}

}  // namespace pb
