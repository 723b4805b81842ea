// gemm.cu — prefill projections on the tensor cores: out = X[M x K] * W[N x K]^T + fused epilogue.
//
// Used for the QKV, O, FC1/FC2 (OPT) and QKV, O, gate|up, down (Llama) projections of every layer
// (the per-layer prefill compute of P:L102-107). Both operands are K-major bf16 (activations row-major,
// HF [out, in] weights row-major), fed by TMA with 128-byte swizzle into a 4-stage shared-memory ring.
//
// CTA tile 128 x 128, BK = 64; 128 threads:
//   warp 0 / lane 0 : TMA producer   (full[s] <- expect_tx; empty[s] released by tcgen05.commit)
//   warp 1 / lane 0 : MMA issuer     (4 x tcgen05.mma M128 N128 K16 per stage, fp32 accumulator in TMEM)
//   warps 0-3       : epilogue       (tcgen05.ld, one output row per thread; bias / scale / ReLU /
//                                     SiLU*up / fp32 residual add fused, vectorised stores)
#include <cuda_bf16.h>

#include "kernels.hpp"
#include "sm100.cuh"

namespace pb {
using namespace sm100;

namespace {

constexpr int BM = 128, BN = 128, BK = 64, STAGES = 4;
constexpr int kStageA = BM * BK * 2;  // 16 KB
constexpr int kStageB = BN * BK * 2;  // 16 KB
constexpr int kSmem = STAGES * (kStageA + kStageB) + 256 + 1024;

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

template <int EPI>
__global__ void __launch_bounds__(128, 1) gemm_kernel(const __grid_constant__ CUtensorMap mapX,
                                                      const __grid_constant__ CUtensorMap mapW, const GemmArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * kStageA;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (kStageA + kStageB));
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = a.M_begin + blockIdx.y * BM;
    // EPI_SILU_MUL: tile = 64 gate columns + the matching 64 up columns -> 64 outputs.
    const int n_out0 = blockIdx.x * (EPI == EPI_SILU_MUL ? BN / 2 : BN);
    const int num_k = (a.K + BK - 1) / BK;   // K tail: TMA zero-fills out-of-bounds columns of X and W

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
        for (int kb = 0; kb < num_k; ++kb) {
            const int s = kb % STAGES;
            if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], kStageA + kStageB);
            tma_load_2d(sA + s * kStageA, &mapX, &full[s], kb * BK, m0);
            if (EPI == EPI_SILU_MUL) {
                tma_load_2d(sB + s * kStageB, &mapW, &full[s], kb * BK, n_out0);
                tma_load_2d(sB + s * kStageB + kStageB / 2, &mapW, &full[s], kb * BK, a.up_row0 + n_out0);
            } else {
                tma_load_2d(sB + s * kStageB, &mapW, &full[s], kb * BK, n_out0);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, 0, 0);
        for (int kb = 0; kb < num_k; ++kb) {
            const int s = kb % STAGES;
            mbar_wait(&full[s], (kb / STAGES) & 1);
            tc_fence_after();
            const uint32_t a_base = smem_u32(sA + s * kStageA), b_base = smem_u32(sB + s * kStageB);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = smem_desc(a_base + k * 32, 16, 1024, kSw128);
                const uint64_t bd = smem_desc(b_base + k * 32, 16, 1024, kSw128);
                umma_bf16(tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
            }
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    }
    __syncwarp();
    mbar_wait(done, 0);
    tc_fence_after();

    // ---------------- epilogue: one row per thread
    const int row = m0 + warp * 32 + lane;
    const bool row_ok = row < a.M_end;
    const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
    if (EPI == EPI_SILU_MUL) {
#pragma unroll 1
        for (int cb = 0; cb < 2; ++cb) {
            float g[32], u[32];
            tmem_ld32(t_row + cb * 32, g);
            tmem_ld32(t_row + 64 + cb * 32, u);
            const int n = n_out0 + cb * 32;
            if (row_ok && n < a.N) {
                __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.ldo + n;
                if (n + 32 <= a.N) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 v;
                        uint32_t* vv = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int c = q * 8 + 2 * e;
                            vv[e] = bf16x2_bits(silu(g[c]) * u[c], silu(g[c + 1]) * u[c + 1]);
                        }
                        reinterpret_cast<uint4*>(o)[q] = v;
                    }
                } else {
                    for (int c = 0; c < 32 && n + c < a.N; ++c) o[c] = __float2bfloat16_rn(silu(g[c]) * u[c]);
                }
            }
        }
    } else {
#pragma unroll 1
        for (int cb = 0; cb < BN / 32; ++cb) {
            float v[32];
            tmem_ld32(t_row + cb * 32, v);
            const int n = n_out0 + cb * 32;
            if (!row_ok || n >= a.N) continue;
            const int nv = min(32, a.N - n);
            if (a.bias) {
                for (int c = 0; c < 32; ++c) v[c] += c < nv ? __bfloat162float(a.bias[n + c]) : 0.f;
            }
            if (EPI == EPI_BF16) {
                if (n < a.scale_cols) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] *= (n + c < a.scale_cols) ? a.scale : 1.0f;
                }
                if (a.relu) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] = fmaxf(v[c], 0.0f);
                }
                __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.ldo + n;
                if (nv == 32) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 w;
                        uint32_t* ww = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                        for (int e = 0; e < 4; ++e) ww[e] = bf16x2_bits(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
                        reinterpret_cast<uint4*>(o)[q] = w;
                    }
                } else {
                    for (int c = 0; c < nv; ++c) o[c] = __float2bfloat16_rn(v[c]);
                }
            } else {  // EPI_RESID
                float* h = reinterpret_cast<float*>(a.out) + (size_t)row * a.ldo + n;
                if (nv == 32) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 x = reinterpret_cast<float4*>(h)[q];
                        x.x += v[q * 4 + 0];
                        x.y += v[q * 4 + 1];
                        x.z += v[q * 4 + 2];
                        x.w += v[q * 4 + 3];
                        reinterpret_cast<float4*>(h)[q] = x;
                    }
                } else {
                    for (int c = 0; c < nv; ++c) h[c] += v[c];
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<BN>(tmem);
    }
}

template <int EPI>
cudaError_t launch_epi(const CUtensorMap& mapX, const CUtensorMap& mapW, const GemmArgs& a, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    const int per = EPI == EPI_SILU_MUL ? BN / 2 : BN;
    dim3 grid((a.N + per - 1) / per, (a.M_end - a.M_begin + BM - 1) / BM);
    gemm_kernel<EPI><<<grid, 128, kSmem, s>>>(mapX, mapW, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm(const CUtensorMap& mapX, const CUtensorMap& mapW, const GemmArgs& a, cudaStream_t s) {
    if (a.M_end <= a.M_begin || a.N <= 0) return cudaSuccess;
    if (a.K <= 0 || a.K % 8) return cudaErrorInvalidValue;
    switch (a.epi) {
        case EPI_BF16: return launch_epi<EPI_BF16>(mapX, mapW, a, s);
        case EPI_RESID: return launch_epi<EPI_RESID>(mapX, mapW, a, s);
        case EPI_SILU_MUL: return launch_epi<EPI_SILU_MUL>(mapX, mapW, a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace pb
