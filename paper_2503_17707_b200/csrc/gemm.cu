// gemm.cu — prefill projections on the tensor cores: out = X[M x K] * W[N x K]^T + fused epilogue.
//
// Used for the QKV, O, FC1/FC2 (OPT) and QKV, O, gate|up, down (Llama) projections of every layer
// (the per-layer prefill compute of P:L102-107). Both operands are K-major bf16 (activations row-major,
// HF [out, in] weights row-major), fed by TMA with 128-byte swizzle into a 6-stage shared-memory ring.
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

#include "kernels.hpp"
#include "sm100.cuh"

namespace pb {
using namespace sm100;

namespace {

constexpr int BM = 128, BN = 128, BK = 64, STAGES = 6;
constexpr int kStageA = BM * BK * 2;  // 16 KB
constexpr int kStageB = BN * BK * 2;  // 16 KB
constexpr int kBarOff = STAGES * (kStageA + kStageB);
constexpr int kSmem = kBarOff + 256 + 1024;
static_assert(BM * BN * 4 <= kBarOff, "partial tile must fit in the stage ring");

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

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
// Partial tile: [128 rows][32 float4 chunks], chunk c of row r stored at slot c ^ (r & 31) (conflict-free
// row-per-thread writes, and conflict-free chunk-per-thread reads).
__device__ __forceinline__ uint32_t part_off(int row, int chunk) {
    return (uint32_t)(row * 512 + ((chunk ^ (row & 31)) << 4));
}

template <int EPI>
__global__ void __launch_bounds__(128, 1) gemm_kernel(const __grid_constant__ CUtensorMap mapX,
                                                      const __grid_constant__ CUtensorMap mapW, const GemmArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * kStageA;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int S = gridDim.z;                       // split-K factor == cluster size along z
    const int split = S > 1 ? (int)cluster_rank() : 0;
    const int m0 = a.M_begin + blockIdx.y * BM;
    // EPI_SILU_MUL: tile = 64 gate columns + the matching 64 up columns -> 64 outputs.
    const int n_out0 = blockIdx.x * (EPI == EPI_SILU_MUL ? BN / 2 : BN);
    const int nk = (a.K + BK - 1) / BK;            // K tail: TMA zero-fills out-of-bounds columns
    const int kb0 = (int)((long)nk * split / S), kb1 = (int)((long)nk * (split + 1) / S);
    const int my_k = kb1 - kb0;                    // >= 1 (host guarantees S <= nk)

    if (tid == 0) {
        tma_prefetch_desc(&mapX);
        tma_prefetch_desc(&mapW);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<BN>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer
        for (int i = 0; i < my_k; ++i) {
            const int s = i % STAGES, kc = (kb0 + i) * BK;
            if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], kStageA + kStageB);
            tma_load_2d(sA + s * kStageA, &mapX, &full[s], kc, m0);
            if (EPI == EPI_SILU_MUL) {
                tma_load_2d(sB + s * kStageB, &mapW, &full[s], kc, n_out0);
                tma_load_2d(sB + s * kStageB + kStageB / 2, &mapW, &full[s], kc, a.up_row0 + n_out0);
            } else {
                tma_load_2d(sB + s * kStageB, &mapW, &full[s], kc, n_out0);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, 0, 0);
        for (int i = 0; i < my_k; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            tc_fence_after();
            const uint32_t a_base = smem_u32(sA + s * kStageA), b_base = smem_u32(sB + s * kStageB);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = smem_desc(a_base + k * 32, 16, 1024, kSw128);
                const uint64_t bd = smem_desc(b_base + k * 32, 16, 1024, kSw128);
                umma_bf16(tmem, ad, bd, idesc, (i | k) != 0 ? 1u : 0u);
            }
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    }
    __syncwarp();
    mbar_wait(done, 0);
    tc_fence_after();

    // ---------------- stage the fp32 tile (this CTA's K-partial) in shared memory; all MMAs and TMA loads
    // have completed, so the stage ring is free.
    {
        const int row = warp * 32 + lane;
        const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
        for (int cb = 0; cb < BN / 32; ++cb) {
            float v[32];
            tmem_ld32(t_row + cb * 32, v);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                *reinterpret_cast<float4*>(smem + part_off(row, cb * 8 + q)) =
                    make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
    }
    tc_fence_before();
    if (S > 1) cluster_sync();
    else __syncthreads();

    // ---------------- reduce rows [r_lo, r_hi) over the S partials (fixed order) + fused epilogue
    const int r_lo = BM * split / S, r_hi = BM * (split + 1) / S;
    const uint32_t base = smem_u32(smem);
    const int chunks = EPI == EPI_SILU_MUL ? 16 : 32;
    for (int idx = tid; idx < (r_hi - r_lo) * chunks; idx += 128) {
        const int r = r_lo + idx / chunks, ch = idx % chunks;
        const int row = m0 + r;
        auto sum_chunk = [&](int c) {
            float4 acc = *reinterpret_cast<const float4*>(smem + part_off(r, c));
            if (S > 1) {
                acc = ld_cluster_f4(map_cluster(base + part_off(r, c), 0));
                for (int s2 = 1; s2 < S; ++s2) {
                    const float4 p = ld_cluster_f4(map_cluster(base + part_off(r, c), s2));
                    acc.x += p.x;
                    acc.y += p.y;
                    acc.z += p.z;
                    acc.w += p.w;
                }
            }
            return acc;
        };
        if (row >= a.M_end) continue;
        if (EPI == EPI_SILU_MUL) {
            const int n = n_out0 + ch * 4;
            if (n >= a.N) continue;
            const float4 g = sum_chunk(ch), u = sum_chunk(ch + 16);
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
        const float4 acc = sum_chunk(ch);
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
            if (nv == 4) {
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
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<BN>(tmem);
    }
}

template <int EPI>
cudaError_t launch_epi(const CUtensorMap& mapX, const CUtensorMap& mapW, const GemmArgs& a, int S, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    if (S > 1) {
        e = cudaFuncSetAttribute(gemm_kernel<EPI>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    const int per = EPI == EPI_SILU_MUL ? BN / 2 : BN;
    const dim3 grid((a.N + per - 1) / per, (a.M_end - a.M_begin + BM - 1) / BM, S);
    if (S == 1) {   // no cluster: plain launch (lower launch latency)
        gemm_kernel<EPI><<<grid, 128, kSmem, s>>>(mapX, mapW, a);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = S;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_kernel<EPI>, mapX, mapW, a);
}

}  // namespace

// Split-K factor: fill the 148 SMs with (N tiles x S) CTAs, at most 4 (measured on B200 at M = 128:
// S = 8 loses to S = 4 on cluster scheduling + DSMEM reduction, tools/gemm_bench.py), at least eight
// 64-wide K blocks per split. Depends on N and K only (determinism across prompt chunkings).
int gemm_split_k(int N, int K, int epi) {
    const int per = epi == EPI_SILU_MUL ? BN / 2 : BN;
    const int n_tiles = (N + per - 1) / per;
    const int nk = (K + BK - 1) / BK;
    int S = 148 / (n_tiles > 0 ? n_tiles : 1);
    S = S < 1 ? 1 : (S > 4 ? 4 : S);
    while (S > 1 && nk / S < 8) --S;
    return S;
}

cudaError_t warm_gemm_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, gemm_kernel<EPI_BF16>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_kernel<EPI_RESID>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_kernel<EPI_SILU_MUL>);
    return e;
}

cudaError_t launch_gemm(const CUtensorMap& mapX, const CUtensorMap& mapW, const GemmArgs& a, cudaStream_t s) {
    if (a.M_end <= a.M_begin || a.N <= 0) return cudaSuccess;
    if (a.K <= 0 || a.K % 8) return cudaErrorInvalidValue;
    const int S = a.split_k > 0 ? a.split_k : gemm_split_k(a.N, a.K, a.epi);
    switch (a.epi) {
        case EPI_BF16: return launch_epi<EPI_BF16>(mapX, mapW, a, S, s);
        case EPI_RESID: return launch_epi<EPI_RESID>(mapX, mapW, a, S, s);
        case EPI_SILU_MUL: return launch_epi<EPI_SILU_MUL>(mapX, mapW, a, S, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace pb
