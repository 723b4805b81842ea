// gemm.cu — prefill projections on the tensor cores: out = X[M x K] * W[N x K]^T + fused epilogue.
//
// Used for the QKV, O, FC1/FC2 (OPT) and QKV, O, gate|up, down (Llama) projections of every layer
// (the per-layer prefill compute of P:L102-107). Both operands are K-major bf16 (activations row-major,
// HF [out, in] weights row-major), fed by TMA with 128-byte swizzle into a shared-memory ring of 6 stages
// (3 when the grid needs two CTAs per SM). With programmatic dependent launch (GemmArgs::pdl) the producer
// requests the first ring of WEIGHT tiles before waiting for the previous kernel (weights do not depend on
// it), so the weight stream of one projection starts under the tail of the kernel before it.
//
// CTA tile 128 x 128, BK = 64; 128 threads:
//   warp 0 / lane 0 : TMA producer   (full[s] <- expect_tx; empty[s] released by tcgen05.commit)
//   warp 1 / lane 0 : MMA issuer     (4 x tcgen05.mma M128 N128 K16 per stage, fp32 accumulator in TMEM)
//   warps 0-3       : epilogue
// Split-K over a thread-block cluster (1 x 1 x S): at prefill sizes (M = B*T = 128 rows at C2) a projection
// has only N/128 = 16..64 output tiles, far fewer than 148 SMs, and streams its weights once (arithmetic
// intensity = M flop/byte, HBM-bound). The S CTAs of a cluster each accumulate 1/S of K in their own TMEM,
// stage the fp32 partial tile in shared memory, and after a cluster barrier CTA s reduces rows
// [s*128/S, (s+1)*128/S) over the S partials through distributed shared memory in a FIXED order, applies the
// fused epilogue (bias / q-scale / ReLU / SiLU*up / fp32 residual add) and writes coalesced rows.
// S is chosen from (N, K) only — never from M — so a prompt split into chunks gives bit-identical results.
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>


#include "kernels.hpp"
#include "sm100.cuh"

namespace pb {
using namespace sm100;

namespace {

constexpr int BM = 128, BN = 128, BK = 64, MAX_STAGES = 6;
constexpr int kStageA = BM * BK * 2;  // 16 KB
constexpr int kStageB = BN * BK * 2;  // 16 KB
constexpr int kStage = kStageA + kStageB;
constexpr int kBarBytes = 256;
static_assert(BM * BN * 4 <= 2 * kStage, "partial tile must fit in a 2-stage ring");
// The split-K kernel also runs with 64-column tiles (TBN = 64; bias / residual epilogues) when a projection has so
// few 128-column tiles that fewer than half the SMs would stream its weights (gemm_tile_n).
constexpr int kMaxStagesAny = 8;
template <int TBN> __host__ __device__ constexpr int stage_bytes() { return kStageA + TBN * BK * 2; }
template <int TBN> __host__ __device__ constexpr int max_stages() { return TBN == 128 ? MAX_STAGES : 8; }
template <int TBN> __host__ __device__ constexpr int smem_bytes_t(int stages) {
    return stages * stage_bytes<TBN>() + kBarBytes + 1024;
}
static_assert(BM * 64 * 4 <= 2 * (kStageA + 64 * BK * 2), "64-column partial tile must fit in a 2-stage ring");

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// HF rotate_half RoPE on fp32 values (x1 = columns ci.., x2 = columns ci + hd/2.. of one head, both already summed):
// x1' = x1 cos - x2 sin, x2' = x2 cos + x1 sin, angle = position * theta^(-2i/hd) from the fp64-built table.
template <int NV>
__device__ __forceinline__ void rope_rotate(const GemmArgs& a, int row, int ci, float (&x1)[NV], float (&x2)[NV]) {
    const int half = a.rope_hd >> 1;
    const int pos = (row - a.rope_row0) / a.rope_B;
    const float2* tb = a.rope + (size_t)pos * half + ci;
#pragma unroll
    for (int e = 0; e < NV; ++e) {
        const float2 cs = tb[e];
        const float u = x1[e], w = x2[e];
        x1[e] = fmaf(u, cs.x, -w * cs.y);
        x2[e] = fmaf(w, cs.x, u * cs.y);
    }
}
__device__ __forceinline__ void rope_rotate4(const GemmArgs& a, int row, int ci, float (&x1)[4], float (&x2)[4]) {
    rope_rotate<4>(a, row, ci, x1, x2);
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_cluster(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

// Partial tile: [128 rows][TBN/4 float4 chunks], chunk c of row r stored at slot c ^ (r % (TBN/4)) (row-per-thread
// writes and chunk-per-thread reads spread over the banks).
template <int TBN>
__device__ __forceinline__ uint32_t part_off(int row, int chunk) {
    return (uint32_t)(row * (TBN * 4) + ((chunk ^ (row & (TBN / 4 - 1))) << 4));
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Phase stamps of the debug trace (pb_op_debug_gemm): slot k of CTA (x, y, z) in a.trace[cta * 8 + k].
#define PB_GEMM_STAMP(k)                                                                                              \
    do {                                                                                                              \
        if (a.trace)                                                                                                  \
            a.trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 8 + (k)] = gtimer();          \
    } while (0)

// S = split-K factor = cluster size along z (compile-time so the S remote loads of the reduction are issued
// back to back, then summed in the fixed order 0..S-1).
template <int EPI, int S, int TBN = BN>
__global__ void __launch_bounds__(128, 1) gemm_kernel(const __grid_constant__ CUtensorMap mapX,
                                                      const __grid_constant__ CUtensorMap mapW, const GemmArgs a,
                                                      const int stages) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = smem;
    static_assert(TBN == BN || (TBN == 64 && EPI != EPI_SILU_MUL), "64-column tiles: bias / residual epilogues");
    constexpr int kStageT = stage_bytes<TBN>();
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStageT);
    uint64_t* empty = full + kMaxStagesAny;
    uint64_t* done = empty + kMaxStagesAny;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int split = S > 1 ? (int)cluster_rank() : 0;
    const int m_shift = a.m_dyn ? *a.m_dyn * a.m_dyn_mul : 0;   // f3 decode graphs: rows known on the device
    const int m0 = a.M_begin + m_shift + blockIdx.y * BM;
    const int m_end = a.M_end + m_shift;
    // EPI_SILU_MUL: tile = 64 gate columns + the matching 64 up columns -> 64 outputs.
    const int n_out0 = blockIdx.x * (EPI == EPI_SILU_MUL ? BN / 2 : TBN);
    const int nk = (a.K + BK - 1) / BK;            // K tail: TMA zero-fills out-of-bounds columns
    const int kb0 = (int)((long)nk * split / S), kb1 = (int)((long)nk * (split + 1) / S);
    const int my_k = kb1 - kb0;                    // >= 1 (host guarantees S <= nk)

    if (tid == 0) PB_GEMM_STAMP(0);
    pdl_launch_dependents();
    if (tid == 0) {
        tma_prefetch_desc(&mapX);
        tma_prefetch_desc(&mapW);
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<TBN>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) PB_GEMM_STAMP(1);

    auto load_w = [&](int i) {
        const int s = i % stages, kc = (kb0 + i) * BK;
        uint8_t* sB = ring + s * kStageT + kStageA;
        if (EPI == EPI_SILU_MUL) {
            tma_load_2d(sB, &mapW, &full[s], kc, n_out0);
            tma_load_2d(sB + kStageB / 2, &mapW, &full[s], kc, a.up_row0 + n_out0);
        } else {
            tma_load_2d(sB, &mapW, &full[s], kc, n_out0);
        }
    };
    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer. The weights do not depend on the previous kernel: the first ring's
        // worth is requested before the programmatic-dependency wait, X (the previous kernel's output) after.
        const int pre = my_k < stages ? my_k : stages;
        for (int i = 0; i < pre; ++i) {
            mbar_arrive_expect_tx(&full[i], kStageT);
            load_w(i);
        }
        pdl_wait();
        PB_GEMM_STAMP(2);
        for (int i = 0; i < pre; ++i) tma_load_2d(ring + i * kStageT, &mapX, &full[i], (kb0 + i) * BK, m0);
        for (int i = pre; i < my_k; ++i) {
            const int s = i % stages;
            mbar_wait(&empty[s], ((i / stages) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], kStageT);
            tma_load_2d(ring + s * kStageT, &mapX, &full[s], (kb0 + i) * BK, m0);
            load_w(i);
        }
        PB_GEMM_STAMP(3);
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = idesc_bf16_f32(BM, TBN, 0, 0);
        for (int i = 0; i < my_k; ++i) {
            const int s = i % stages;
            mbar_wait(&full[s], (i / stages) & 1);
            if (i == 0) PB_GEMM_STAMP(4);
            tc_fence_after();
            const uint32_t a_base = smem_u32(ring + s * kStageT), b_base = a_base + kStageA;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = smem_desc(a_base + k * 32, 16, 1024, kSw128);
                const uint64_t bd = smem_desc(b_base + k * 32, 16, 1024, kSw128);
                umma_bf16(tmem, ad, bd, idesc, (i | k) != 0 ? 1u : 0u);
            }
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    } else {
        pdl_wait();
    }
    __syncwarp();
    mbar_wait(done, 0);
    tc_fence_after();
    if (tid == 0) PB_GEMM_STAMP(5);

    // ---------------- stage the fp32 tile (this CTA's K-partial) in shared memory; all MMAs and TMA loads
    // have completed, so the stage ring is free. Two batches of 64 columns (4 loads in flight, one wait).
    {
        const int row = warp * 32 + lane;
        const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
        for (int half = 0; half < TBN / 64; ++half) {
            uint32_t r0[32], r1[32];
            tmem_ld32_async(t_row + half * 64, r0);
            tmem_ld32_async(t_row + half * 64 + 32, r1);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                *reinterpret_cast<uint4*>(smem + part_off<TBN>(row, half * 16 + q)) =
                    make_uint4(r0[4 * q], r0[4 * q + 1], r0[4 * q + 2], r0[4 * q + 3]);
                *reinterpret_cast<uint4*>(smem + part_off<TBN>(row, half * 16 + 8 + q)) =
                    make_uint4(r1[4 * q], r1[4 * q + 1], r1[4 * q + 2], r1[4 * q + 3]);
            }
        }
    }
    tc_fence_before();
    if (S > 1) cluster_sync();
    else __syncthreads();
    if (tid == 0) PB_GEMM_STAMP(6);

    // ---------------- reduce rows [r_lo, r_hi) over the S partials (fixed order 0..S-1) + fused epilogue
    const int r_lo = BM * split / S, r_hi = BM * (split + 1) / S;
    const uint32_t base = smem_u32(smem);
    const int chunks = EPI == EPI_SILU_MUL ? 16 : TBN / 4;
    auto sum_chunk = [&](int r, int c) {
        if constexpr (S == 1) {
            return *reinterpret_cast<const float4*>(smem + part_off<TBN>(r, c));
        } else {
            float4 p[S];
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) p[s2] = ld_cluster_f4(map_cluster(base + part_off<TBN>(r, c), s2));
            float4 acc = p[0];
#pragma unroll
            for (int s2 = 1; s2 < S; ++s2) {
                acc.x += p[s2].x;
                acc.y += p[s2].y;
                acc.z += p[s2].z;
                acc.w += p[s2].w;
            }
            return acc;
        }
    };
    for (int idx = tid; idx < (r_hi - r_lo) * chunks; idx += 128) {
        const int r = r_lo + idx / chunks, ch = idx % chunks;
        const int row = m0 + r;
        if (row >= m_end) continue;
        if (EPI == EPI_SILU_MUL) {
            const int n = n_out0 + ch * 4;
            if (n >= a.N) continue;
            const float4 g = sum_chunk(r, ch), u = sum_chunk(r, ch + 16);
            const float o[4] = {silu(g.x) * u.x, silu(g.y) * u.y, silu(g.z) * u.z, silu(g.w) * u.w};
            __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.ldo + n;
            if (n + 4 <= a.N) {
                uint2 w;
                w.x = bf16x2_bits(o[0], o[1]);
                w.y = bf16x2_bits(o[2], o[3]);
                *reinterpret_cast<uint2*>(out) = w;
            } else {
                for (int c = 0; c < 4 && n + c < a.N; ++c) out[c] = __float2bfloat16_rn(o[c]);
            }
            continue;
        }
        const int n = n_out0 + ch * 4;
        if (n >= a.N) continue;
        if (EPI == EPI_BF16 && a.rope && n < a.rope_cols) {
            // rotary pair (i, i + hd/2) of one head, both halves in this tile (128-column tiles, head-aligned): the
            // thread owning the first half rotates and writes both, from the fp32 sums
            const int half = a.rope_hd >> 1, ci = n % a.rope_hd;
            if (ci >= half) continue;
            const float4 p1 = sum_chunk(r, ch), p2 = sum_chunk(r, ch + (half >> 2));
            float x1[4] = {p1.x, p1.y, p1.z, p1.w}, x2[4] = {p2.x, p2.y, p2.z, p2.w};
            rope_rotate4(a, row, ci, x1, x2);
            __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.ldo + n;
            uint2 w1, w2;
            w1.x = bf16x2_bits(x1[0], x1[1]);
            w1.y = bf16x2_bits(x1[2], x1[3]);
            w2.x = bf16x2_bits(x2[0], x2[1]);
            w2.y = bf16x2_bits(x2[2], x2[3]);
            *reinterpret_cast<uint2*>(out) = w1;
            *reinterpret_cast<uint2*>(out + half) = w2;
            continue;
        }
        const float4 acc = sum_chunk(r, ch);
        float v[4] = {acc.x, acc.y, acc.z, acc.w};
        const int nv = min(4, a.N - n);
        if (a.bias) {
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] += c < nv ? __bfloat162float(a.bias[n + c]) : 0.f;
        }
        if (EPI == EPI_BF16) {
            if (n < a.scale_cols) {
#pragma unroll
                for (int c = 0; c < 4; ++c) v[c] *= (n + c < a.scale_cols) ? a.scale : 1.0f;
            }
            if (a.relu) {
#pragma unroll
                for (int c = 0; c < 4; ++c) v[c] = fmaxf(v[c], 0.0f);
            }
            __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.ldo + n;
            if (nv == 4) {
                uint2 w;
                w.x = bf16x2_bits(v[0], v[1]);
                w.y = bf16x2_bits(v[2], v[3]);
                *reinterpret_cast<uint2*>(out) = w;
            } else {
                for (int c = 0; c < nv; ++c) out[c] = __float2bfloat16_rn(v[c]);
            }
        } else {  // EPI_RESID: h += acc + bias (fp32)
            float* h = reinterpret_cast<float*>(a.out) + (size_t)row * a.ldo + n;
            // 16-byte vectors where aligned (every residual stream; a vocab slice of the logits may start anywhere)
            if (nv == 4 && (reinterpret_cast<uintptr_t>(h) & 15) == 0) {
                float4 x = *reinterpret_cast<float4*>(h);
                x.x += v[0];
                x.y += v[1];
                x.z += v[2];
                x.w += v[3];
                *reinterpret_cast<float4*>(h) = x;
            } else {
                for (int c = 0; c < nv; ++c) h[c] += v[c];
            }
        }
    }
    if (S > 1) cluster_sync();   // keep this CTA's partial alive until every peer has read it
    if (tid == 0) PB_GEMM_STAMP(7);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<TBN>(tmem);
    }
}

template <int EPI, int S, int TBN = BN>
cudaError_t launch_es(const CUtensorMap& mapX, const CUtensorMap& mapW, const GemmArgs& a, cudaStream_t s) {
    const int per = EPI == EPI_SILU_MUL ? BN / 2 : TBN;
    const dim3 grid((a.N + per - 1) / per, (a.M_end - a.M_begin + BM - 1) / BM, S);
    // Deep ring when the grid fits one CTA per SM; otherwise 3 stages (96 KB) so two CTAs share an SM.
    const int ctas = grid.x * grid.y * grid.z;
    static const int forced = getenv("PB_GEMM_STAGES") ? atoi(getenv("PB_GEMM_STAGES")) : 0;   // experiments
    const int stages = forced >= 2 && forced <= max_stages<TBN>() ? forced : ctas <= 148 ? max_stages<TBN>() : 3;
    const int smem = smem_bytes_t<TBN>(stages);
    cudaError_t e = smem_attr_once<gemm_kernel<EPI, S, TBN>>(smem_bytes_t<TBN>(max_stages<TBN>()));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (S > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 1;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = S;
        ++na;
    }
    if (a.pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, gemm_kernel<EPI, S, TBN>, mapX, mapW, a, stages);
}

template <int EPI>
cudaError_t launch_epi(const CUtensorMap& mapX, const CUtensorMap& mapW, const GemmArgs& a, int S, int tbn,
                       cudaStream_t s) {
    if constexpr (EPI != EPI_SILU_MUL) {
        if (tbn == 64) {
            switch (S) {
                case 1: return launch_es<EPI, 1, 64>(mapX, *a.mapW64, a, s);
                case 2: return launch_es<EPI, 2, 64>(mapX, *a.mapW64, a, s);
                case 4: return launch_es<EPI, 4, 64>(mapX, *a.mapW64, a, s);
            }
            return cudaErrorInvalidValue;
        }
    }
    switch (S) {
        case 1: return launch_es<EPI, 1>(mapX, mapW, a, s);
        case 2: return launch_es<EPI, 2>(mapX, mapW, a, s);
        case 4: return launch_es<EPI, 4>(mapX, mapW, a, s);
        case 8: return launch_es<EPI, 8>(mapX, mapW, a, s);
    }
    return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------------------------
// Large-M path (the prompt batch spans several 128-row tiles; S = 1): persistent, warp-specialised, 128 x 256
// tiles (one tcgen05.mma M128 N256 K16 per 16-wide K step), a 4-stage TMA ring of 48 KB stages, and two
// 256-column TMEM accumulators so the epilogue of tile i overlaps the mainloop of tile i+1.
//   warp 0 lane 0 : TMA producer (X box 128 x 64; W as two 128-row boxes, SiLU: four 64-row boxes)
//   warp 1 lane 0 : MMA issuer
//   warps 2-5     : epilogue, one output row per thread (TMEM lane quadrant = warp % 4)
// Tiles are visited n-major (all M tiles of one N tile back to back) so each weight tile is read from HBM once
// and re-read from L2 by the other M tiles while the activations (M x K) stay L2-resident.
// ------------------------------------------------------------------------------------------------------------
constexpr int BIG_BN = 256, BIG_STAGES = 4;
constexpr int kBigA = BM * BK * 2, kBigB = BIG_BN * BK * 2;   // 16 KB activation box, 32 KB weight boxes per stage
// The same kernel with 128- to 224-column tiles (bias / residual epilogues) where 256-column tiles fill the last wave
// badly (gemm_big_tile_n): W arrives as a 128-row box plus 64- (mapW64) and 32-row (mapW32) boxes for the rest
// (160 = 128 + 32, 192 = 128 + 64, 224 = 128 + 64 + 32); as many stages as fit in 227 KB (4 to 6). (144 / 208 columns
// with 16-row boxes measured slower at the C4 shapes than the wave count predicts.)
template <int TBN> __host__ __device__ constexpr int big_stages() {
    return TBN == 256 ? BIG_STAGES : TBN >= 192 ? 5 : 6;
}
template <int TBN> __host__ __device__ constexpr int big_stage_bytes() { return kBigA + TBN * BK * 2; }
template <int TBN> __host__ __device__ constexpr int big_smem() {
    return big_stages<TBN>() * big_stage_bytes<TBN>() + 256 + 1024;
}

// Epilogue of CW accumulator columns [n, n + CW) of one output row: + bias, then (EPI_BF16) q-scale / ReLU and one
// RNE rounding to bf16, or (EPI_RESID) the fp32 residual add h += acc + bias.
template <int EPI, int CW>
__device__ __forceinline__ void big_epi_chunk(const GemmArgs& a, int row, int n, const uint32_t (&r)[CW]) {
    float v[CW];
#pragma unroll
    for (int e = 0; e < CW; ++e) {
        v[e] = __uint_as_float(r[e]);
        if (a.bias && n + e < a.N) v[e] += __bfloat162float(a.bias[n + e]);
    }
    const int nv = min(CW, a.N - n);
    if (EPI == EPI_BF16) {
#pragma unroll
        for (int e = 0; e < CW; ++e) {
            if (n + e < a.scale_cols) v[e] *= a.scale;
            if (a.relu) v[e] = fmaxf(v[e], 0.f);
        }
        __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.ldo + n;
        if (nv == CW) {
#pragma unroll
            for (int q = 0; q < CW / 8; ++q)
                *reinterpret_cast<uint4*>(out + 8 * q) =
                    make_uint4(bf16x2_bits(v[8 * q], v[8 * q + 1]), bf16x2_bits(v[8 * q + 2], v[8 * q + 3]),
                               bf16x2_bits(v[8 * q + 4], v[8 * q + 5]), bf16x2_bits(v[8 * q + 6], v[8 * q + 7]));
        } else {
#pragma unroll
            for (int e = 0; e < CW; ++e)
                if (e < nv) out[e] = __float2bfloat16_rn(v[e]);
        }
    } else {   // EPI_RESID: h += acc + bias
        float* h = reinterpret_cast<float*>(a.out) + (size_t)row * a.ldo + n;
        if (nv == CW) {
#pragma unroll
            for (int q = 0; q < CW / 4; ++q) {
                float4 x = *reinterpret_cast<float4*>(h + 4 * q);
                x.x += v[4 * q];
                x.y += v[4 * q + 1];
                x.z += v[4 * q + 2];
                x.w += v[4 * q + 3];
                *reinterpret_cast<float4*>(h + 4 * q) = x;
            }
        } else {
#pragma unroll
            for (int e = 0; e < CW; ++e)
                if (e < nv) h[e] += v[e];
        }
    }
}

template <int EPI, int TBN = BIG_BN>
__global__ void __launch_bounds__(192, 1) gemm_big_kernel(const __grid_constant__ CUtensorMap mapX,
                                                          const __grid_constant__ CUtensorMap mapW,
                                                          const __grid_constant__ CUtensorMap mapW64,
                                                          const __grid_constant__ CUtensorMap mapW32, const GemmArgs a) {
    static_assert(TBN == BIG_BN || (TBN % 32 == 0 && TBN >= 128 && TBN < 256 && EPI != EPI_SILU_MUL),
                  "128- to 224-column tiles: bias / residual epilogues");
    constexpr int NST = big_stages<TBN>(), kStg = big_stage_bytes<TBN>();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * kStg);
    uint64_t* empty = full + NST;
    uint64_t* acc_full = empty + NST;           // [2] MMA -> epilogue
    uint64_t* acc_empty = acc_full + 2;         // [2] epilogue -> MMA (128 arrivals)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int per = EPI == EPI_SILU_MUL ? BIG_BN / 2 : TBN;   // outputs per tile along N
    const int n_tiles = (a.N + per - 1) / per;
    const int m_tiles = (a.M_end - a.M_begin + BM - 1) / BM;
    const int tiles = n_tiles * m_tiles;
    const int nk = (a.K + BK - 1) / BK;

    pdl_launch_dependents();
    if (tid == 0) {
        tma_prefetch_desc(&mapX);
        tma_prefetch_desc(&mapW);
        if (TBN == 192 || TBN == 224) tma_prefetch_desc(&mapW64);
        if (TBN == 160 || TBN == 224) tma_prefetch_desc(&mapW32);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 128);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            int it = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int m0 = a.M_begin + (t % m_tiles) * BM, n0 = (t / m_tiles) * per;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % NST, kc = kb * BK;
                    if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
                    uint8_t* sA = smem + s * kStg;
                    uint8_t* sB = sA + kBigA;
                    mbar_arrive_expect_tx(&full[s], kStg);
                    tma_load_2d(sA, &mapX, &full[s], kc, m0);
                    if (EPI == EPI_SILU_MUL) {   // [gate 128 | up 128] rows as four 64-row boxes
                        tma_load_2d(sB, &mapW, &full[s], kc, n0);
                        tma_load_2d(sB + kBigB / 4, &mapW, &full[s], kc, n0 + 64);
                        tma_load_2d(sB + kBigB / 2, &mapW, &full[s], kc, a.up_row0 + n0);
                        tma_load_2d(sB + 3 * kBigB / 4, &mapW, &full[s], kc, a.up_row0 + n0 + 64);
                    } else {
                        tma_load_2d(sB, &mapW, &full[s], kc, n0);   // rows 128 B apart: row r at sB + 128 r
                        if (TBN == 256) tma_load_2d(sB + 128 * 128, &mapW, &full[s], kc, n0 + 128);
                        if (TBN == 192 || TBN == 224) tma_load_2d(sB + 128 * 128, &mapW64, &full[s], kc, n0 + 128);
                        if (TBN == 160) tma_load_2d(sB + 128 * 128, &mapW32, &full[s], kc, n0 + 128);
                        if (TBN == 224) tma_load_2d(sB + 192 * 128, &mapW32, &full[s], kc, n0 + 192);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer
            constexpr uint32_t idesc = idesc_bf16_f32(BM, TBN, 0, 0);
            int it = 0, local = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
                const int b = local & 1;
                const uint32_t acc = tmem + b * TBN;
                if (local >= 2) mbar_wait(&acc_empty[b], ((local >> 1) - 1) & 1);
                tc_fence_after();
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % NST;
                    mbar_wait(&full[s], (it / NST) & 1);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(smem + s * kStg), b_base = a_base + kBigA;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16(acc, smem_desc(a_base + k * 32, 16, 1024, kSw128),
                                  smem_desc(b_base + k * 32, 16, 1024, kSw128), idesc, (kb | k) != 0 ? 1u : 0u);
                    umma_commit(&empty[s]);
                }
                umma_commit(&acc_full[b]);
            }
        }
    } else {   // ---------------- epilogue warps 2..5: row = TMEM lane
        const int quad = warp & 3, row_in_tile = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        int local = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
            const int b = local & 1;
            const int m0 = a.M_begin + (t % m_tiles) * BM, n0 = (t / m_tiles) * per;
            mbar_wait(&acc_full[b], (local >> 1) & 1);
            tc_fence_after();
            const int row = m0 + row_in_tile;
            const bool row_ok = row < a.M_end;
            const uint32_t acc = tmem + b * TBN + lane_off;
            if (EPI == EPI_SILU_MUL) {
#pragma unroll 1
                for (int cb = 0; cb < 4; ++cb) {   // 32 gate columns + the matching 32 up columns
                    uint32_t g[32], u[32];
                    tmem_ld32_async(acc + cb * 32, g);
                    tmem_ld32_async(acc + 128 + cb * 32, u);
                    tmem_wait_ld();
                    const int n = n0 + cb * 32;
                    if (!row_ok || n >= a.N) continue;
                    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.ldo + n;
                    if (n + 32 <= a.N) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            float o[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                const float gv = __uint_as_float(g[8 * q + e]);
                                o[e] = silu(gv) * __uint_as_float(u[8 * q + e]);
                            }
                            *reinterpret_cast<uint4*>(out + 8 * q) =
                                make_uint4(bf16x2_bits(o[0], o[1]), bf16x2_bits(o[2], o[3]), bf16x2_bits(o[4], o[5]),
                                           bf16x2_bits(o[6], o[7]));
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (n + e < a.N)
                                out[e] = __float2bfloat16_rn(silu(__uint_as_float(g[e])) * __uint_as_float(u[e]));
                    }
                }
            } else {
#pragma unroll 1
                for (int cb = 0; cb < TBN / 32; ++cb) {
                    const int n = n0 + cb * 32;
                    if (EPI == EPI_BF16 && a.rope && n < a.rope_cols) {
                        // rotary pair blocks (cb, cb + hd/64) of one head (256- / 128-column tiles are head-aligned):
                        // rotate the fp32 accumulators, round once, write both halves
                        const int half = a.rope_hd >> 1, ci = n % a.rope_hd;
                        if (ci >= half) continue;
                        uint32_t r1[32], r2[32];
                        tmem_ld32_async(acc + cb * 32, r1);
                        tmem_ld32_async(acc + cb * 32 + half, r2);
                        tmem_wait_ld();
                        if (!row_ok) continue;
                        float x1[32], x2[32];
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            x1[e] = __uint_as_float(r1[e]);
                            x2[e] = __uint_as_float(r2[e]);
                        }
                        rope_rotate<32>(a, row, ci, x1, x2);
                        __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.ldo + n;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            *reinterpret_cast<uint4*>(out + 8 * q) =
                                make_uint4(bf16x2_bits(x1[8 * q], x1[8 * q + 1]), bf16x2_bits(x1[8 * q + 2], x1[8 * q + 3]),
                                           bf16x2_bits(x1[8 * q + 4], x1[8 * q + 5]),
                                           bf16x2_bits(x1[8 * q + 6], x1[8 * q + 7]));
                            *reinterpret_cast<uint4*>(out + half + 8 * q) =
                                make_uint4(bf16x2_bits(x2[8 * q], x2[8 * q + 1]), bf16x2_bits(x2[8 * q + 2], x2[8 * q + 3]),
                                           bf16x2_bits(x2[8 * q + 4], x2[8 * q + 5]),
                                           bf16x2_bits(x2[8 * q + 6], x2[8 * q + 7]));
                        }
                        continue;
                    }
                    uint32_t r[32];
                    tmem_ld32_async(acc + cb * 32, r);
                    tmem_wait_ld();
                    if (!row_ok || n >= a.N) continue;
                    big_epi_chunk<EPI, 32>(a, row, n, r);
                }
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int EPI, int TBN = BIG_BN>
cudaError_t launch_big(const CUtensorMap& mapX, const CUtensorMap& mapW, const CUtensorMap& mapW64,
                       const CUtensorMap& mapW32, const GemmArgs& a, cudaStream_t s) {
    cudaError_t e = smem_attr_once<gemm_big_kernel<EPI, TBN>>(big_smem<TBN>());
    if (e != cudaSuccess) return e;
    const int per = EPI == EPI_SILU_MUL ? BIG_BN / 2 : TBN;
    const int tiles = ((a.N + per - 1) / per) * ((a.M_end - a.M_begin + BM - 1) / BM);
    const int grid = tiles < 148 ? tiles : 148;
    return launch_pdl(gemm_big_kernel<EPI, TBN>, dim3(grid), dim3(192), big_smem<TBN>(), s, a.pdl != 0, mapX, mapW,
                      mapW64, mapW32, a);
}

// Tile width of the persistent kernel: 256, 224, 192, 160 or 128 columns, whichever minimises waves x (width + 32)
// (the +32 charges narrower tiles for their extra activation traffic and per-tile overhead); 256 unless another width
// is more than 5 % better. 160 / 224 need the 32-row weight boxes (fine = false: 256 / 192 / 128 only). C4: QKV and
// FC1 224, O / FC2 160; C3: QKV 192, O / down 128 (one wave); C5a: O / down 224 (QKV: rotary, 256).
// Depends on (N, epi, rows of the whole prompt) only.
int gemm_big_tile_n(int N, int epi, int M_total, bool fine) {
    if (epi == EPI_SILU_MUL) return BIG_BN;
    const long m_tiles = (M_total + BM - 1) / BM;
    auto cost = [&](int w) {
        const long tiles = (N + w - 1) / w * m_tiles;
        return (double)((tiles + 147) / 148) * (w + 32);
    };
    int best = BIG_BN;
    double best_cost = cost(BIG_BN) * 0.95;
    for (int w : {224, 192, 160, 128})
        if ((fine || w == 192 || w == 128) && cost(w) < best_cost) {
            best = w;
            best_cost = cost(w);
        }
    return best;
}

// ------------------------------------------------------------------------------------------------------------
// Weight-streaming GEMV for M <= 2 rows (f3 decode steps; tiny prompts). At M = 1 or 2 a projection is a pure
// weight stream (intensity <= 2 flop/B), the tensor core's 128-row tile would be >= 98 % padding, and the split-K
// cluster kernel's fixed latency (TMEM, cluster barriers, DSMEM reduction) dominates. Here a CTA of 8 warps owns
// 4 weight rows (EPI_SILU_MUL: 2 gate + the 2 matching up rows -> 2 outputs) and splits K across its warps;
// every lane streams 16-B weight vectors with no L1 allocation (ld.global.nc.L1::no_allocate), the M activation
// rows come through L1, fp32 FMAs in a fixed order, a butterfly per warp and the 8 warp sums added in order 0..7
// — deterministic, independent of which rows a launch covers. The first weight vectors are loaded before the
// programmatic-dependency wait (weights never depend on the previous kernel).
constexpr int GV_ROWS = 4, GV_WARPS = 8, GV_UNROLL = 2;

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}

template <int EPI, int MR>
__global__ void __launch_bounds__(GV_WARPS * 32) gemv_kernel(const GemmArgs a) {
    __shared__ float red[GV_WARPS][GV_ROWS][MR];
    pdl_launch_dependents();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int M = a.M_end - a.M_begin;
    // weight rows of this CTA; out-of-range rows read row 0 and are never stored
    int wrow[GV_ROWS];
    bool wok[GV_ROWS];
#pragma unroll
    for (int r = 0; r < GV_ROWS; ++r) {
        int n;
        if (EPI == EPI_SILU_MUL) {
            const int o = blockIdx.x * 2 + (r & 1);
            wok[r] = o < a.N;
            n = r < 2 ? o : a.up_row0 + o;
        } else if (EPI == EPI_BF16 && a.rope && (int)blockIdx.x * GV_ROWS < a.rope_cols) {
            // rotary CTA: rows {i, i+1} of a head's first half and their partners {i + hd/2, i + hd/2 + 1}
            const int half = a.rope_hd >> 1, per_head = half / 2;
            const int head = blockIdx.x / per_head, i0 = (blockIdx.x % per_head) * 2;
            n = head * a.rope_hd + (r >= 2 ? half : 0) + i0 + (r & 1);
            wok[r] = true;
        } else {
            n = blockIdx.x * GV_ROWS + r;
            wok[r] = n < a.N;
        }
        wrow[r] = wok[r] ? n : 0;
    }
    // K range of this warp, in 8-element vectors: vectors [v0, v1) of every row
    const int nvec = a.K / 8;
    const int per_w = (nvec + GV_WARPS - 1) / GV_WARPS;
    const int v0 = warp * per_w, v1 = min(nvec, v0 + per_w);
    float acc[GV_ROWS][MR];
#pragma unroll
    for (int r = 0; r < GV_ROWS; ++r)
#pragma unroll
        for (int m = 0; m < MR; ++m) acc[r][m] = 0.f;
    const int step = 32 * GV_UNROLL;
    int vb = v0;
    // first batch of weight vectors before the dependency wait
    uint4 wv[GV_UNROLL][GV_ROWS];
    auto load_w = [&](int base) {
#pragma unroll
        for (int u = 0; u < GV_UNROLL; ++u) {
            const int v = base + u * 32 + lane;
#pragma unroll
            for (int r = 0; r < GV_ROWS; ++r)
                wv[u][r] = v < v1 ? ld_stream16(a.W + (size_t)wrow[r] * a.K + (size_t)v * 8) : make_uint4(0, 0, 0, 0);
        }
    };
    if (vb < v1) load_w(vb);
    pdl_wait();
    const int m_shift = a.m_dyn ? *a.m_dyn * a.m_dyn_mul : 0;
    const int m0 = a.M_begin + m_shift;
    for (; vb < v1; vb += step) {
        if (vb != v0) load_w(vb);   // the first batch was requested before the dependency wait
#pragma unroll
        for (int u = 0; u < GV_UNROLL; ++u) {
            const int v = vb + u * 32 + lane;
            if (v >= v1) break;
            float wf[GV_ROWS][8];
#pragma unroll
            for (int r = 0; r < GV_ROWS; ++r) bf16x8_to_f32(wv[u][r], wf[r]);
            uint4 xv[MR];
#pragma unroll
            for (int m = 0; m < MR; ++m)
                if (m < M) xv[m] = __ldg(reinterpret_cast<const uint4*>(a.X + (size_t)(m0 + m) * a.ldx) + v);
#pragma unroll
            for (int m = 0; m < MR; ++m) {
                if (m >= M) break;
                float xf[8];
                bf16x8_to_f32(xv[m], xf);
#pragma unroll
                for (int r = 0; r < GV_ROWS; ++r)
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[r][m] = __fmaf_rn(wf[r][e], xf[e], acc[r][m]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < GV_ROWS; ++r)
#pragma unroll
        for (int m = 0; m < MR; ++m) {
            float v = acc[r][m];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[warp][r][m] = v;
        }
    __syncthreads();
    // epilogue: one thread per (output, row)
    const int outs = EPI == EPI_SILU_MUL ? 2 : GV_ROWS;
    const int t = threadIdx.x;
    if (t >= outs * M) return;
    const int r = t % outs, m = t / outs;
    auto total = [&](int rr) {
        float v = red[0][rr][m];
#pragma unroll
        for (int w = 1; w < GV_WARPS; ++w) v += red[w][rr][m];
        return v;
    };
    const int row = m0 + m;
    if (EPI == EPI_SILU_MUL) {
        if (!wok[r]) return;
        const int n = blockIdx.x * 2 + r;
        reinterpret_cast<__nv_bfloat16*>(a.out)[(size_t)row * a.ldo + n] =
            __float2bfloat16_rn(silu(total(r)) * total(r + 2));
        return;
    }
    if (!wok[r]) return;
    const int n = wrow[r];
    float v = total(r);
    if (a.bias) v += __bfloat162float(a.bias[n]);
    if (EPI == EPI_BF16 && a.rope && n < a.rope_cols) {   // rotary CTA: the partner row is r ^ 2
        float w = total(r ^ 2);
        if (a.bias) w += __bfloat162float(a.bias[wrow[r ^ 2]]);
        const int half = a.rope_hd >> 1, ci = n % a.rope_hd;
        float x1[1] = {r < 2 ? v : w}, x2[1] = {r < 2 ? w : v};
        rope_rotate<1>(a, row, ci % half, x1, x2);
        reinterpret_cast<__nv_bfloat16*>(a.out)[(size_t)row * a.ldo + n] = __float2bfloat16_rn(r < 2 ? x1[0] : x2[0]);
        return;
    }
    if (EPI == EPI_BF16) {
        if (n < a.scale_cols) v *= a.scale;
        if (a.relu) v = fmaxf(v, 0.0f);
        reinterpret_cast<__nv_bfloat16*>(a.out)[(size_t)row * a.ldo + n] = __float2bfloat16_rn(v);
    } else {
        float* h = reinterpret_cast<float*>(a.out) + (size_t)row * a.ldo + n;
        *h += v;
    }
}

template <int EPI>
cudaError_t launch_gemv_epi(const GemmArgs& a, cudaStream_t s) {
    const int M = a.M_end - a.M_begin;
    const int per = EPI == EPI_SILU_MUL ? 2 : GV_ROWS;
    const dim3 grid((a.N + per - 1) / per);
    const bool pdl = a.pdl != 0;
    static_assert(kGemvAutoRows <= 2, "instantiate gemv_kernel for more rows");
    if (M <= 1) return launch_pdl(gemv_kernel<EPI, 1>, grid, dim3(GV_WARPS * 32), 0, s, pdl, a);
    return launch_pdl(gemv_kernel<EPI, 2>, grid, dim3(GV_WARPS * 32), 0, s, pdl, a);
}

}  // namespace


// Split-K factor S (1, 2 or 4): the largest S <= 4 that keeps n_tiles x m_tiles x S <= 296 CTAs (two per SM
// on 148 SMs) with at least 4 K blocks of 64 per split. It depends on (N, K, M_total) only, where M_total is
// the row count of the WHOLE prompt batch (not of a prompt chunk), so a prompt split into chunks reduces
// every output in the same order and gives bit-identical results. Measured on B200 at M = 128
// (tools/gemm_bench.py, r01c): S = 4 is fastest for all four OPT-1.3B projections; clusters of 8 lose to
// cluster scheduling (one CTA per SM needs 8 free SMs in one GPC).
// Tile width of the split-K kernel: 64 columns when the projection has a single row tile and its 128-column tiles x
// S would keep fewer than half of the 148 SMs streaming weights (C2: O and FC2, N = 2048 -> 16 x 4 = 64 CTAs), so
// twice as many SMs share the weight stream. Depends on (N, K, epi, M_total) only, like S.
int gemm_tile_n(int N, int K, int epi, int M_total) {
    if (epi == EPI_SILU_MUL || M_total > BM) return BN;
    const long n_tiles = (N + BN - 1) / BN;
    return n_tiles * gemm_split_k(N, K, epi, M_total) <= 74 ? 64 : BN;
}

int gemm_split_k(int N, int K, int epi, int M_total) {
    const int per = epi == EPI_SILU_MUL ? BN / 2 : BN;
    const long n_tiles = (N + per - 1) / per;
    const long m_tiles = M_total > 0 ? (M_total + BM - 1) / BM : 1;
    const int nk = (K + BK - 1) / BK;
    static const long max_ctas = getenv("PB_GEMM_CTAS") ? atol(getenv("PB_GEMM_CTAS")) : 296;   // experiments
    int S = 1;
    while (S < 4 && n_tiles * m_tiles * 2 * S <= max_ctas && nk / (2 * S) >= 4) S *= 2;
    return S;
}

cudaError_t warm_gemm_kernels() {
    cudaFuncAttributes at;
    const void* fns[] = {(const void*)gemm_kernel<EPI_BF16, 1>,     (const void*)gemm_kernel<EPI_BF16, 2>,
                         (const void*)gemm_kernel<EPI_BF16, 4>,     (const void*)gemm_kernel<EPI_BF16, 8>,
                         (const void*)gemm_kernel<EPI_RESID, 1>,    (const void*)gemm_kernel<EPI_RESID, 2>,
                         (const void*)gemm_kernel<EPI_RESID, 4>,    (const void*)gemm_kernel<EPI_RESID, 8>,
                         (const void*)gemm_kernel<EPI_SILU_MUL, 1>, (const void*)gemm_kernel<EPI_SILU_MUL, 2>,
                         (const void*)gemm_kernel<EPI_SILU_MUL, 4>, (const void*)gemm_kernel<EPI_SILU_MUL, 8>,
                         (const void*)gemm_kernel<EPI_BF16, 1, 64>, (const void*)gemm_kernel<EPI_BF16, 2, 64>,
                         (const void*)gemm_kernel<EPI_BF16, 4, 64>, (const void*)gemm_kernel<EPI_RESID, 1, 64>,
                         (const void*)gemm_kernel<EPI_RESID, 2, 64>, (const void*)gemm_kernel<EPI_RESID, 4, 64>,
                         (const void*)gemm_big_kernel<EPI_BF16>,     (const void*)gemm_big_kernel<EPI_RESID>,
                         (const void*)gemm_big_kernel<EPI_SILU_MUL>,
                         (const void*)gemm_big_kernel<EPI_BF16, 192>, (const void*)gemm_big_kernel<EPI_RESID, 192>,
                         (const void*)gemm_big_kernel<EPI_BF16, 128>, (const void*)gemm_big_kernel<EPI_RESID, 128>,
                         (const void*)gemm_big_kernel<EPI_BF16, 160>, (const void*)gemm_big_kernel<EPI_RESID, 160>,
                         (const void*)gemm_big_kernel<EPI_BF16, 224>, (const void*)gemm_big_kernel<EPI_RESID, 224>,
                         (const void*)gemv_kernel<EPI_BF16, 1>,  (const void*)gemv_kernel<EPI_BF16, 2>,
                         (const void*)gemv_kernel<EPI_RESID, 1>, (const void*)gemv_kernel<EPI_RESID, 2>,
                         (const void*)gemv_kernel<EPI_SILU_MUL, 1>, (const void*)gemv_kernel<EPI_SILU_MUL, 2>};
    for (const void* f : fns) {
        cudaError_t e = cudaFuncGetAttributes(&at, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Vocabulary logits of one or two sequences as the weight-streaming GEMV (the head is a pure stream of V x d bf16 at
// M <= 2): logits[b, v0:v1] = y[b] . E[v0:v1]^T accumulated into a zeroed fp32 slice (EPI_RESID). Each output's sum
// is taken in the same order whatever rows a launch covers, so vocab slices give the same bits as the whole head.
cudaError_t launch_logits_gemv(const __nv_bfloat16* y, int B, int d, const __nv_bfloat16* E, int v0, int v1,
                               float* logits, int ldl, cudaStream_t s, bool pdl) {
    if (v1 <= v0 || B <= 0) return cudaSuccess;
    if (B > kGemvAutoRows || d % 8) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemset2DAsync(logits + v0, (size_t)ldl * 4, 0, (size_t)(v1 - v0) * 4, B, s);
    if (e != cudaSuccess) return e;
    GemmArgs a{};
    a.M_begin = 0;
    a.M_end = B;
    a.N = v1 - v0;
    a.K = d;
    a.epi = EPI_RESID;
    a.scale = 1.f;
    a.out = logits + v0;
    a.ldo = ldl;
    a.M_total = B;
    a.pdl = pdl ? 1 : 0;
    a.X = y;
    a.ldx = d;
    a.W = E + (size_t)v0 * d;
    return launch_gemv_epi<EPI_RESID>(a, s);
}

// Vocabulary logits of a large batch on the tensor cores: logits[b, v0:v1] = y[b] . E[v0:v1]^T (fp32), as the
// split-K kernel's fp32 epilogue over a zeroed slice. S = 1 (each output's K sum in one CTA, in k order), so a
// vocab slice of any width gives the same bits as the whole head (pipelined equals sequential).
cudaError_t launch_logits_tc(const __nv_bfloat16* y, int B, int d, const __nv_bfloat16* E, int v0, int v1, float* logits,
                             int ldl, cudaStream_t s) {
    if (v1 <= v0 || B <= 0) return cudaSuccess;
    CUtensorMap mx, mw;
    char err[256];
    if (!make_map_bf16(&mx, y, B, d, d, 128, 64, 128, err, sizeof err) ||
        !make_map_bf16(&mw, E + (size_t)v0 * d, v1 - v0, d, d, 128, 64, 128, err, sizeof err))
        return cudaErrorInvalidValue;
    cudaError_t e = cudaMemset2DAsync(logits + v0, (size_t)ldl * 4, 0, (size_t)(v1 - v0) * 4, B, s);
    if (e != cudaSuccess) return e;
    GemmArgs a{};
    a.M_begin = 0;
    a.M_end = B;
    a.N = v1 - v0;
    a.K = d;
    a.epi = EPI_RESID;
    a.scale = 1.f;
    a.out = logits + v0;
    a.ldo = ldl;
    a.split_k = 1;
    a.M_total = B;
    return launch_gemm(mx, mw, a, s);
}

cudaError_t launch_gemm(const CUtensorMap& mapX, const CUtensorMap& mapW, const GemmArgs& a, cudaStream_t s) {
    if (a.M_end <= a.M_begin || a.N <= 0) return cudaSuccess;
    if (a.K <= 0 || a.K % 8) return cudaErrorInvalidValue;
    if (a.rope && (a.epi != EPI_BF16 || (a.rope_hd != 64 && a.rope_hd != 128) || a.rope_cols % a.rope_hd ||
                   a.rope_B < 1 || a.bias || a.scale_cols > 0 || a.relu))
        return cudaErrorInvalidValue;
    // M_total <= 8 (a decode step or a tiny prompt; chosen from the whole batch, so chunks agree): weight-streaming GEMV
    // Measured on B200, C2 decode ms/step GEMV vs tensor-core path: B=1 1.07 vs 1.46, B=2 1.56 vs 1.56, B=4 1.95 vs
    // 1.73 (the GEMV's fp32 FMA work grows with M and its registers with it), hence M_total <= kGemvAutoRows.
    if (a.X && a.W && a.split_k <= 0 && a.M_total >= 1 && a.M_total <= kGemvAutoRows &&
        a.M_end - a.M_begin <= kGemvAutoRows) {
        switch (a.epi) {
            case EPI_BF16: return launch_gemv_epi<EPI_BF16>(a, s);
            case EPI_RESID: return launch_gemv_epi<EPI_RESID>(a, s);
            case EPI_SILU_MUL: return launch_gemv_epi<EPI_SILU_MUL>(a, s);
        }
    }
    const int S = a.split_k > 0 ? a.split_k : gemm_split_k(a.N, a.K, a.epi, a.M_total);
    // The kernel is chosen from the WHOLE prompt (M_total), never from the rows of this launch, so a prompt split
    // into chunks runs every output through the same kernel and the same summation order.
    if (S == 1 && a.split_k <= 0 && a.M_total > BM && !a.m_dyn) {
        static const bool fine_off = getenv("PB_GEMM_FINE_TILES") && atoi(getenv("PB_GEMM_FINE_TILES")) == 0;   // A/B
        const bool fine = a.mapW32 != nullptr && !fine_off;
        int tw = a.mapW64 ? gemm_big_tile_n(a.N, a.epi, a.M_total, fine) : BIG_BN;
        if (a.rope && tw % 128) tw = BIG_BN;   // rotary pairs need head-aligned tiles
        const CUtensorMap& m64 = a.mapW64 ? *a.mapW64 : mapW;
        const CUtensorMap& m32 = a.mapW32 ? *a.mapW32 : mapW;
#define PB_BIG(E, W) \
    if (tw == W) return launch_big<E, W>(mapX, mapW, m64, m32, a, s);
        switch (a.epi) {
            case EPI_BF16:
                PB_BIG(EPI_BF16, 224) PB_BIG(EPI_BF16, 192) PB_BIG(EPI_BF16, 160) PB_BIG(EPI_BF16, 128)
                return launch_big<EPI_BF16>(mapX, mapW, m64, m32, a, s);
            case EPI_RESID:
                PB_BIG(EPI_RESID, 224) PB_BIG(EPI_RESID, 192) PB_BIG(EPI_RESID, 160) PB_BIG(EPI_RESID, 128)
                return launch_big<EPI_RESID>(mapX, mapW, m64, m32, a, s);
            case EPI_SILU_MUL: return launch_big<EPI_SILU_MUL>(mapX, mapW, m64, m32, a, s);
        }
#undef PB_BIG
    }
    const int tbn = a.split_k <= 0 && a.mapW64 && !a.rope ? gemm_tile_n(a.N, a.K, a.epi, a.M_total) : BN;
    switch (a.epi) {
        case EPI_BF16: return launch_epi<EPI_BF16>(mapX, mapW, a, S, tbn, s);
        case EPI_RESID: return launch_epi<EPI_RESID>(mapX, mapW, a, S, tbn, s);
        case EPI_SILU_MUL: return launch_epi<EPI_SILU_MUL>(mapX, mapW, a, S, tbn, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace pb
