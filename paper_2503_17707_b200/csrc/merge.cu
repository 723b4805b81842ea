// merge.cu — a3: merged-LoRA weight update on the tensor cores (tcgen05 / TMEM / TMA).
//
//   W'[i, j] = RNE_bf16( W[i, j] + s * sum_k B[i, k] * A[k, j] ),  s = alpha / r
//   (P:L111-114 LoRA definition; "parameters of the LoRA adapter are merged back into the base model")
//
// One CTA owns a 128 x 128 tile of W. The elected thread issues three TMA loads on two mbarriers:
// the tiny operands (B tile [128 x rk], A tile [rk x 128]) and the 32 KB W tile. As soon as the operands
// land it issues rk/16 tcgen05.mma (M=128, N=128, K=16) into a 128-column TMEM accumulator; the W tile
// keeps streaming meanwhile. The epilogue (4 warps, one W row per thread = one TMEM lane) reads 32
// accumulator columns at a time with tcgen05.ld, adds s*acc to W in fp32, rounds to bf16 in place in
// shared memory (128B-swizzled, conflict-free) and one thread TMA-stores the tile back.
//
// HBM-bound: 4 bytes/element (read + write W) against r/2 flop/byte; the tensor core turns the K=r
// contraction into a handful of instructions so the SMs only stream W.
#include <cuda_bf16.h>

#include <algorithm>

#include "kernels.hpp"
#include "sm100.cuh"

namespace pb {
using namespace sm100;

namespace {

constexpr int kTile = 128;
constexpr int kWBytes = kTile * kTile * 2;  // 32 KB, two 64-column SW128 boxes

template <int RK>
struct MergeSmem {
    static constexpr int kB = kTile * RK * 2;     // B tile [128 x RK], K-major, swizzle RK*2 bytes
    static constexpr int kA = RK * kTile * 2;     // A tile [RK x 128], MN-major, two SW128 boxes of RK rows
    static constexpr int offW = 0;
    static constexpr int offB = kWBytes;
    static constexpr int offA = offB + ((kB + 1023) / 1024) * 1024;
    static constexpr int offBar = offA + kA;
    static constexpr int kTotal = offBar + 64;
};

template <int RK>
__global__ void __launch_bounds__(128) merge_kernel(const __grid_constant__ CUtensorMap mapW,
                                                    const __grid_constant__ CUtensorMap mapB,
                                                    const __grid_constant__ CUtensorMap mapA,
                                                    const __grid_constant__ CUtensorMap mapWout, float scale) {
    using S = MergeSmem<RK>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sW = smem + S::offW;
    uint8_t* sB = smem + S::offB;
    uint8_t* sA = smem + S::offA;
    uint64_t* bar_ops = reinterpret_cast<uint64_t*>(smem + S::offBar);
    uint64_t* bar_w = bar_ops + 1;
    uint64_t* bar_mma = bar_ops + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_ops + 3);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n0 = blockIdx.x * kTile, m0 = blockIdx.y * kTile;

    if (tid == 0) {
        tma_prefetch_desc(&mapW);
        tma_prefetch_desc(&mapB);
        tma_prefetch_desc(&mapA);
        mbar_init(bar_ops, 1);
        mbar_init(bar_w, 1);
        mbar_init(bar_mma, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<128>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (tid == 0) {
        mbar_arrive_expect_tx(bar_ops, S::kB + S::kA);
        tma_load_2d(sB, &mapB, bar_ops, 0, m0);
        tma_load_2d(sA, &mapA, bar_ops, n0, 0);
        tma_load_2d(sA + RK * 128, &mapA, bar_ops, n0 + 64, 0);
        mbar_arrive_expect_tx(bar_w, kWBytes);
        tma_load_2d(sW, &mapW, bar_w, n0, m0);
        tma_load_2d(sW + kWBytes / 2, &mapW, bar_w, n0 + 64, m0);

        mbar_wait(bar_ops, 0);
        tc_fence_after();
        constexpr uint64_t kBSw = RK == 16 ? kSw32 : (RK == 32 ? kSw64 : kSw128);
        constexpr uint32_t idesc = idesc_bf16_f32(128, 128, /*a_mn=*/0, /*b_mn=*/1);
#pragma unroll
        for (int kk = 0; kk < RK / 16; ++kk) {
            // A operand = LoRA B tile, K-major: 8-row core groups RK*2*8 bytes apart; K slice advances 32 B.
            const uint64_t a_desc = smem_desc(smem_u32(sB) + kk * 32, 16, RK * 2 * 8, kBSw);
            // B operand = LoRA A tile, MN-major SW128: 64-column boxes RK*128 B apart (LBO),
            // 8-row K groups 1024 B apart (SBO); K slice of 16 rows advances 2048 B.
            const uint64_t b_desc = smem_desc(smem_u32(sA) + kk * 2048, RK * 128, 1024, kSw128);
            umma_bf16(tmem, a_desc, b_desc, idesc, kk > 0 ? 1u : 0u);
        }
        umma_commit(bar_mma);
    }
    __syncwarp();
    mbar_wait(bar_mma, 0);
    mbar_wait(bar_w, 0);
    tc_fence_after();

    // Epilogue: thread = W row (TMEM lane). Row r of a 64-col SW128 box: 16-B chunk j lives at chunk j ^ (r & 7).
    const int row = warp * 32 + lane;
#pragma unroll 1
    for (int cb = 0; cb < 4; ++cb) {
        float acc[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + cb * 32, acc);
        uint8_t* box = sW + (cb >> 1) * (kWBytes / 2) + row * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = (cb & 1) * 4 + q;
            uint4* p = reinterpret_cast<uint4*>(box + ((j ^ (row & 7)) << 4));
            uint4 w = *p;
            uint32_t* wv = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 pair = *reinterpret_cast<__nv_bfloat162*>(&wv[e]);
                float2 f = __bfloat1622float2(pair);
                wv[e] = bf16x2_bits(fmaf(scale, acc[q * 8 + 2 * e], f.x), fmaf(scale, acc[q * 8 + 2 * e + 1], f.y));
            }
            *p = w;
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        tma_store_2d(&mapWout, sW, n0, m0);                 // in place: mapWout == mapW
        tma_store_2d(&mapWout, sW + kWBytes / 2, n0 + 64, m0);
        tma_store_commit();
        tma_store_wait_all();
    }
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

template <int RK>
cudaError_t launch_rk(const MergeMaps& m, int rows, int cols, float scale, cudaStream_t s) {
    // >= 57 KB of shared memory keeps at most 4 CTAs per SM, so 4 x 128 TMEM columns never over-subscribe.
    int smem = MergeSmem<RK>::kTotal + 1024;
    if (smem < 57 * 1024) smem = 57 * 1024;
    cudaError_t e = cudaFuncSetAttribute(merge_kernel<RK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((cols + kTile - 1) / kTile, (rows + kTile - 1) / kTile);
    merge_kernel<RK><<<grid, 128, smem, s>>>(m.W, m.B, m.A, m.Wout, scale);
    return cudaGetLastError();
}

}  // namespace

int merge_rk(int rank) { return rank <= 16 ? 16 : (rank <= 32 ? 32 : 64); }

bool make_merge_maps(MergeMaps* m, void* W, int64_t ldw, int rows, int cols, const void* B, const void* A, int rank,
                     char* err, size_t errlen, void* Wout) {
    const int rk = merge_rk(rank);
    return make_map_bf16(&m->W, W, rows, cols, ldw, 128, 64, 128, err, errlen) &&
           make_map_bf16(&m->Wout, Wout ? Wout : W, rows, cols, ldw, 128, 64, 128, err, errlen) &&
           make_map_bf16(&m->B, B, rows, rank, rank, 128, rk, rk * 2, err, errlen) &&
           make_map_bf16(&m->A, A, rank, cols, cols, rk, 64, 128, err, errlen);
}

cudaError_t launch_merge(const MergeMaps& m, int rows, int cols, int rank, float scale, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    switch (merge_rk(rank)) {
        case 16: return launch_rk<16>(m, rows, cols, scale, s);
        case 32: return launch_rk<32>(m, rows, cols, scale, s);
        default: return launch_rk<64>(m, rows, cols, scale, s);
    }
}

// Device-to-device byte copy on the SMs (16-byte vectors, grid-stride): used for the rows of a tensor an
// adapter does not touch when building its out-of-place copy, so the copy engine stays free for the PCIe load.
__global__ void __launch_bounds__(256) copy16_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

cudaError_t launch_copy(void* dst, const void* src, int64_t bytes, cudaStream_t s) {
    if (bytes <= 0) return cudaSuccess;
    if ((bytes & 15) || (reinterpret_cast<uintptr_t>(dst) & 15) || (reinterpret_cast<uintptr_t>(src) & 15))
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s);
    const int64_t n = bytes / 16;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    copy16_kernel<<<blocks, 256, 0, s>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n);
    return cudaGetLastError();
}

// Force-load the module functions (CUDA lazy loading): see warm_kernels().
cudaError_t warm_merge_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, merge_kernel<16>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, merge_kernel<32>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, merge_kernel<64>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, copy16_kernel);
    return e;
}

}  // namespace pb
