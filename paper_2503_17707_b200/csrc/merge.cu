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

// The jobs of one launch: tensor maps (kernel parameters, as TMA requires) and each job's tile range.
struct MergeBatch {
    CUtensorMap W[kMaxMergeJobs], B[kMaxMergeJobs], A[kMaxMergeJobs], Wout[kMaxMergeJobs];
    int tiles_n[kMaxMergeJobs];    // 128-column tiles per row of tiles
    int tile_end[kMaxMergeJobs];   // exclusive end of the job's tiles in the launch's tile list
    float scale[kMaxMergeJobs];
    int n_jobs;
};

struct TileRef {
    int job, m0, n0;
};
__device__ __forceinline__ TileRef tile_ref(const MergeBatch& P, int t) {
    int j = 0;
    while (j + 1 < P.n_jobs && t >= P.tile_end[j]) ++j;
    const int lt = t - (j ? P.tile_end[j - 1] : 0);
    return {j, (lt / P.tiles_n[j]) * kTile, (lt % P.tiles_n[j]) * kTile};
}

template <int RK>
__global__ void __launch_bounds__(kMergeThreads, 1) merge_kernel(const __grid_constant__ MergeBatch P) {
    const int n_tiles = P.tile_end[P.n_jobs - 1];
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
        for (int j = 0; j < P.n_jobs; ++j) {
            tma_prefetch_desc(&P.W[j]);
            tma_prefetch_desc(&P.B[j]);
            tma_prefetch_desc(&P.A[j]);
            tma_prefetch_desc(&P.Wout[j]);
        }
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
                const TileRef tr = tile_ref(P, blockIdx.x + i * gridDim.x);
                const int m0 = tr.m0, n0 = tr.n0, j = tr.job;
                const int s = i % NS;
                if (i >= NS) mbar_wait(&empty[s], ((i / NS) - 1) & 1);
                uint8_t* st = smem + s * S::kStage;
                mbar_arrive_expect_tx(&full_ops[s], S::kB + S::kA);
                tma_load_2d(st + S::offB, &P.B[j], &full_ops[s], 0, m0);
                tma_load_2d(st + S::offA, &P.A[j], &full_ops[s], n0, 0);
                tma_load_2d(st + S::offA + RK * 128, &P.A[j], &full_ops[s], n0 + 64, 0);
                mbar_arrive_expect_tx(&full_w[s], kWBytes);
                tma_load_2d(st + S::offW, &P.W[j], &full_w[s], n0, m0);
                tma_load_2d(st + S::offW + kWBytes / 2, &P.W[j], &full_w[s], n0 + 64, m0);
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
            const TileRef tr = tile_ref(P, blockIdx.x + i * gridDim.x);
            const int m0 = tr.m0, n0 = tr.n0, j = tr.job;
            const float scale = P.scale[j];
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
                tma_store_2d(&P.Wout[j], sW, n0, m0);       // in place: Wout == W
                tma_store_2d(&P.Wout[j], sW + kWBytes / 2, n0 + 64, m0);
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
cudaError_t launch_rk(const MergeJobDesc* jobs, int n, cudaStream_t s) {
    constexpr int smem = MergeSmem<RK>::kTotal + 1024;
    cudaError_t e = smem_attr_once<merge_kernel<RK>>(smem);
    if (e != cudaSuccess) return e;
    MergeBatch P;
    int tiles = 0, nj = 0;
    for (int i = 0; i < n; ++i) {
        if (jobs[i].rows <= 0 || jobs[i].cols <= 0) continue;
        P.W[nj] = jobs[i].maps->W;
        P.B[nj] = jobs[i].maps->B;
        P.A[nj] = jobs[i].maps->A;
        P.Wout[nj] = jobs[i].maps->Wout;
        P.tiles_n[nj] = (jobs[i].cols + kTile - 1) / kTile;
        tiles += P.tiles_n[nj] * ((jobs[i].rows + kTile - 1) / kTile);
        P.tile_end[nj] = tiles;
        P.scale[nj] = jobs[i].scale;
        ++nj;
    }
    if (nj == 0) return cudaSuccess;
    P.n_jobs = nj;
    merge_kernel<RK><<<std::min(tiles, kNumSms), kMergeThreads, smem, s>>>(P);
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

cudaError_t launch_merge_batch(const MergeJobDesc* jobs, int n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (n > kMaxMergeJobs) return cudaErrorInvalidValue;
    const int rk = merge_rk(jobs[0].rank);
    for (int i = 1; i < n; ++i)
        if (merge_rk(jobs[i].rank) != rk) return cudaErrorInvalidValue;   // one padded rank per launch
    switch (rk) {
        case 16: return launch_rk<16>(jobs, n, s);
        case 32: return launch_rk<32>(jobs, n, s);
        default: return launch_rk<64>(jobs, n, s);
    }
}

cudaError_t launch_merge(const MergeMaps& m, int rows, int cols, int rank, float scale, cudaStream_t s) {
    const MergeJobDesc j{&m, rows, cols, rank, scale};
    return launch_merge_batch(&j, 1, s);
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
