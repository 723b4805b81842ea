// merge.cu — a3: merged-LoRA weight update on the tensor cores (tcgen05 / TMEM / TMA).
//
//   W'[i, j] = RNE_bf16( W[i, j] + s * sum_k B[i, k] * A[k, j] ),  s = alpha / r
//   (P:L111-114 LoRA definition; "parameters of the LoRA adapter are merged back into the base model")
//
// HBM-bound: 4 bytes/element (read + write W) against r/2 flop/byte, so the kernel is built to keep W streaming:
// a PERSISTENT grid (one CTA per SM, at most one per 128 x 128 tile) walks the W tiles t = blockIdx.x,
// blockIdx.x + gridDim.x, ... through a ring of shared-memory stages, three warp roles overlapping:
//   warp 0 lane 0  TMA producer: per tile one stage = W tile (32 KB, two SW128 boxes of 64 columns) + the LoRA
//                  B tile [128 x rk] (K-major) + A tile [rk x 128] (MN-major); the W load of tile i+stages-1 is in
//                  flight while tile i is merged.
//   warp 1 lane 0  MMA issuer: rk/16 tcgen05.mma M128 N128 K16 per tile into one of TWO 128-column TMEM
//                  accumulators (tile i+1's product is formed while tile i's epilogue drains the other).
//   warps 2-5      epilogue, one W row per thread (TMEM lane quadrant = warp % 4): tcgen05.ld 32 columns at a time,
//                  W + s*acc in fp32 rounded to bf16 in place in the stage (swizzle-aware, conflict-free), then one
//                  thread TMA-stores the tile; a stage is handed back to the producer only once the store has
//                  finished READING it (cp.async.bulk.wait_group.read), so stores drain under the next tiles.
// The arithmetic per element is one fp32 FMA of the fp32 TMEM sum and one RNE rounding (DESIGN.md §3 G2).
#include <cuda_bf16.h>

#include <algorithm>

#include "kernels.hpp"
#include "sm100.cuh"

namespace pb {
using namespace sm100;

namespace {

constexpr int kTile = 128;
constexpr int kWBytes = kTile * kTile * 2;  // 32 KB, two 64-column SW128 boxes
constexpr int kMergeThreads = 192;
constexpr int kMergeSmemBudget = 200 * 1024;
constexpr int kNumSms = 148;   // B200 (sm_100a): one persistent CTA per SM

template <int RK>
struct MergeSmem {
    static constexpr int kB = kTile * RK * 2;     // B tile [128 x RK], K-major, swizzle RK*2 bytes
    static constexpr int kA = RK * kTile * 2;     // A tile [RK x 128], MN-major, two SW128 boxes of RK rows
    static constexpr int offW = 0;
    static constexpr int offB = kWBytes;
    static constexpr int offA = offB + ((kB + 1023) / 1024) * 1024;
    static constexpr int kStage = ((offA + kA + 1023) / 1024) * 1024;
    static constexpr int kStages = std::min(6, (kMergeSmemBudget - 1024) / kStage);
    static constexpr int offBar = kStages * kStage;
    static constexpr int kTotal = offBar + 256;
};

template <int RK>
__global__ void __launch_bounds__(kMergeThreads, 1) merge_kernel(const __grid_constant__ CUtensorMap mapW,
                                                                 const __grid_constant__ CUtensorMap mapB,
                                                                 const __grid_constant__ CUtensorMap mapA,
                                                                 const __grid_constant__ CUtensorMap mapWout,
                                                                 int tiles_n, int n_tiles, float scale) {
    using S = MergeSmem<RK>;
    constexpr int NS = S::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_ops = reinterpret_cast<uint64_t*>(smem + S::offBar);   // [NS] B + A landed
    uint64_t* full_w = full_ops + NS;                                     // [NS] W landed
    uint64_t* empty = full_w + NS;                                        // [NS] stage free (store read it)
    uint64_t* acc_full = empty + NS;                                      // [2] product in TMEM
    uint64_t* acc_empty = acc_full + 2;                                   // [2] epilogue drained TMEM
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        tma_prefetch_desc(&mapW);
        tma_prefetch_desc(&mapB);
        tma_prefetch_desc(&mapA);
        tma_prefetch_desc(&mapWout);
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full_ops[s], 1);
            mbar_init(&full_w[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int my_tiles = n_tiles > (int)blockIdx.x ? (n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            for (int i = 0; i < my_tiles; ++i) {
                const int t = blockIdx.x + i * gridDim.x, m0 = (t / tiles_n) * kTile, n0 = (t % tiles_n) * kTile;
                const int s = i % NS;
                if (i >= NS) mbar_wait(&empty[s], ((i / NS) - 1) & 1);
                uint8_t* st = smem + s * S::kStage;
                mbar_arrive_expect_tx(&full_ops[s], S::kB + S::kA);
                tma_load_2d(st + S::offB, &mapB, &full_ops[s], 0, m0);
                tma_load_2d(st + S::offA, &mapA, &full_ops[s], n0, 0);
                tma_load_2d(st + S::offA + RK * 128, &mapA, &full_ops[s], n0 + 64, 0);
                mbar_arrive_expect_tx(&full_w[s], kWBytes);
                tma_load_2d(st + S::offW, &mapW, &full_w[s], n0, m0);
                tma_load_2d(st + S::offW + kWBytes / 2, &mapW, &full_w[s], n0 + 64, m0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            constexpr uint64_t kBSw = RK == 16 ? kSw32 : (RK == 32 ? kSw64 : kSw128);
            constexpr uint32_t idesc = idesc_bf16_f32(128, 128, /*a_mn=*/0, /*b_mn=*/1);
            for (int i = 0; i < my_tiles; ++i) {
                const int s = i % NS, b = i & 1;
                if (i >= 2) mbar_wait(&acc_empty[b], ((i >> 1) - 1) & 1);
                mbar_wait(&full_ops[s], (i / NS) & 1);
                tc_fence_after();
                const uint32_t sB = smem_u32(smem + s * S::kStage + S::offB);
                const uint32_t sA = smem_u32(smem + s * S::kStage + S::offA);
#pragma unroll
                for (int kk = 0; kk < RK / 16; ++kk) {
                    // A operand = LoRA B tile, K-major: 8-row core groups RK*2*8 bytes apart; K slice advances 32 B.
                    const uint64_t a_desc = smem_desc(sB + kk * 32, 16, RK * 2 * 8, kBSw);
                    // B operand = LoRA A tile, MN-major SW128: 64-column boxes RK*128 B apart (LBO),
                    // 8-row K groups 1024 B apart (SBO); K slice of 16 rows advances 2048 B.
                    const uint64_t b_desc = smem_desc(sA + kk * 2048, RK * 128, 1024, kSw128);
                    umma_bf16(tmem + b * 128, a_desc, b_desc, idesc, kk > 0 ? 1u : 0u);
                }
                umma_commit(&acc_full[b]);
            }
        }
    } else {
        // ---------------- epilogue (warps 2-5). Row r of a 64-col SW128 box: 16-B chunk j lives at chunk j ^ (r & 7).
        const int quad = warp & 3, row = quad * 32 + lane;
        const bool leader = warp == 2 && lane == 0;
        for (int i = 0; i < my_tiles; ++i) {
            const int t = blockIdx.x + i * gridDim.x, m0 = (t / tiles_n) * kTile, n0 = (t % tiles_n) * kTile;
            const int s = i % NS, b = i & 1;
            uint8_t* sW = smem + s * S::kStage + S::offW;
            mbar_wait(&acc_full[b], (i >> 1) & 1);
            mbar_wait(&full_w[s], (i / NS) & 1);
            tc_fence_after();
            const uint32_t t_row = tmem + b * 128 + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
            for (int cb = 0; cb < 4; ++cb) {
                float acc[32];
                tmem_ld32(t_row + cb * 32, acc);
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
                        wv[e] = bf16x2_bits(fmaf(scale, acc[q * 8 + 2 * e], f.x),
                                            fmaf(scale, acc[q * 8 + 2 * e + 1], f.y));
                    }
                    *p = w;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);     // TMEM buffer b may take tile i+2's product
            fence_proxy_async_smem();                       // generic smem writes -> visible to the TMA store
            named_bar_sync(1, 128);
            if (leader) {
                tma_store_2d(&mapWout, sW, n0, m0);         // in place: mapWout == mapW
                tma_store_2d(&mapWout, sW + kWBytes / 2, n0 + 64, m0);
                tma_store_commit();
                if (i >= 1) {
                    tma_store_wait_read_n<1>();              // tile i-1's store has read its stage
                    mbar_arrive(&empty[(i - 1) % NS]);
                }
            }
        }
        if (leader) tma_store_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

template <int RK>
cudaError_t launch_rk(const MergeMaps& m, int rows, int cols, float scale, cudaStream_t s) {
    constexpr int smem = MergeSmem<RK>::kTotal + 1024;
    cudaError_t e = smem_attr_once<merge_kernel<RK>>(smem);
    if (e != cudaSuccess) return e;
    const int tiles_n = (cols + kTile - 1) / kTile, tiles = tiles_n * ((rows + kTile - 1) / kTile);
    const int grid = std::min(tiles, kNumSms);
    merge_kernel<RK><<<grid, kMergeThreads, smem, s>>>(m.W, m.B, m.A, m.Wout, tiles_n, tiles, scale);
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
