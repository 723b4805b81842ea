// gemm_probe.cu — where does the M=128 weight-streaming GEMM lose time? Standalone timing probe (not part of
// the library): the prefill GEMM mainloop (TMA -> smem ring -> tcgen05.mma -> TMEM) with parts switched off.
//   LOADX=0 : X is loaded once (stage ring slot 0) and reused  -> W streaming only
//   MMA=0   : no tensor-core work                              -> TMA pipeline only
// Grid (N/128, 1, S): CTA (n, s) streams K blocks [s*nk/S, (s+1)*nk/S) of W rows [128n, 128n+128).
// Per-launch CUDA events; W rotated over buffers totalling > 2x L2 so every launch reads HBM.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2503_17707_b200/csrc \
//        tools/gemm_probe.cu -o gemm_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace pb::sm100;

constexpr int BM = 128, BN = 128, BK = 64;

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long g_stamps[1024][5];   // per CTA: start, first stage landed, mainloop done, end, smid

template <int STAGES, bool LOADX, bool MMA, bool MCAST>
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap mapX,
                                                const __grid_constant__ CUtensorMap mapW, int K, float* out) {
    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (threadIdx.x == 0 && cta < 1024) {
        g_stamps[cta][0] = gtimer();
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_stamps[cta][4] = smid;
    }
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int SA = BM * BK * 2, SB = BN * BK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * SA;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (SA + SB));
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int S = gridDim.z, split = blockIdx.z;
    const int nk = K / BK, kb0 = nk * split / S, kb1 = nk * (split + 1) / S, my = kb1 - kb0;
    const int n0 = blockIdx.x * BN;
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
    if (warp == 0) tmem_alloc<BN>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < my; ++i) {
            const int s = i % STAGES, kc = (kb0 + i) * BK;
            if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
            const bool lx = LOADX || i == 0;
            mbar_arrive_expect_tx(&full[s], (lx ? SA : 0) + SB);
            if (lx) tma_load_2d(sA + (LOADX ? s : 0) * SA, &mapX, &full[s], kc, 0);
            tma_load_2d(sB + s * SB, &mapW, &full[s], kc, n0);
            if (!MMA) {
                // no consumer: release the slot as soon as it lands
            }
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, 0, 0);
        for (int i = 0; i < my; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            if (i == 0 && cta < 1024) g_stamps[cta][1] = gtimer();
            tc_fence_after();
            if (MMA) {
                const uint32_t a = smem_u32(sA + (LOADX ? s : 0) * SA), b = smem_u32(sB + s * SB);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    umma_bf16(tmem, smem_desc(a + k * 32, 16, 1024, kSw128), smem_desc(b + k * 32, 16, 1024, kSw128),
                              idesc, (i | k) != 0);
                umma_commit(&empty[s]);
            } else {
                mbar_arrive(&empty[s]);
            }
        }
        if (MMA) umma_commit(done);
        else mbar_arrive(done);
    }
    __syncwarp();
    mbar_wait(done, 0);
    if (threadIdx.x == 0 && cta < 1024) g_stamps[cta][2] = gtimer();
    tc_fence_after();
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
    float acc = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += v[i];
    if (acc == 12345.f) out[tid] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<BN>(tmem);
    }
    if (threadIdx.x == 0 && cta < 1024) g_stamps[cta][3] = gtimer();
}

// Pure streaming reference: every CTA reads its contiguous byte range with ld.global.v4 (no TMA, no smem).
__global__ void stream_ld(const uint4* __restrict__ p, size_t n16, float* out) {
    uint32_t x = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(p + i);
        x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (x == 0x12345678u) out[0] = 1;
}

using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static Encode enc;
static CUtensorMap map2d(void* base, uint64_t rows, uint64_t cols, uint32_t brows, uint32_t bcols) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t str[1] = {cols * 2};
    cuuint32_t box[2] = {bcols, brows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

template <int STAGES, bool LOADX, bool MMA>
static void run(const char* tag, int N, int K, int S, const std::vector<void*>& Ws, void* X, float* out) {
    auto kern = probe<STAGES, LOADX, MMA, false>;
    const int smem = STAGES * (BM * BK * 2 + BN * BK * 2) + 1024 + 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    CUtensorMap mx = map2d(X, 128, K, 128, 64);
    std::vector<CUtensorMap> mw;
    for (void* w : Ws) mw.push_back(map2d(w, N, K, 128, 64));
    dim3 grid(N / BN, 1, S);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) kern<<<grid, 128, smem>>>(mx, mw[i % mw.size()], K, out);
    cudaDeviceSynchronize();
    float tot = 0;
    const int reps = 20;
    for (int i = 0; i < reps; ++i) {
        cudaEventRecord(a);
        kern<<<grid, 128, smem>>>(mx, mw[i % mw.size()], K, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        tot += ms;
    }
    {   // CTA timeline of one more launch: start spread, first-data latency, streaming time, epilogue, SM load
        kern<<<grid, 128, smem>>>(mx, mw[0], K, out);
        cudaDeviceSynchronize();
        static unsigned long long st[1024][5];
        cudaMemcpyFromSymbol(st, g_stamps, sizeof st);
        const int n = grid.x * grid.y * grid.z;
        unsigned long long t0 = ~0ull, tmax = 0;
        double s_first = 0, s_main = 0, s_epi = 0, start_max = 0;
        int per_sm[256] = {0}, sm_max = 0;
        for (int i = 0; i < n && i < 1024; ++i) t0 = st[i][0] < t0 ? st[i][0] : t0;
        for (int i = 0; i < n && i < 1024; ++i) {
            start_max = fmax(start_max, (double)(st[i][0] - t0));
            s_first += st[i][1] - st[i][0];
            s_main += st[i][2] - st[i][1];
            s_epi += st[i][3] - st[i][2];
            tmax = st[i][3] > tmax ? st[i][3] : tmax;
            if (++per_sm[st[i][4] & 255] > sm_max) sm_max = per_sm[st[i][4] & 255];
        }
        printf("    timeline: span %.2f us, CTA starts spread %.2f us, mean first-data %.2f us, mean stream %.2f us, "
               "mean epilogue %.2f us, max CTAs/SM %d\n", (tmax - t0) / 1e3, start_max / 1e3, s_first / n / 1e3,
               s_main / n / 1e3, s_epi / n / 1e3, sm_max);
    }
    const double us = tot * 1e3 / reps, wb = (double)N * K * 2;
    printf("%-10s N%5d K%5d S%2d stages%d loadX%d mma%d: %7.2f us  W %6.0f GB/s  CTAs %d\n", tag, N, K, S, STAGES,
           (int)LOADX, (int)MMA, us, wb / us / 1e3, grid.x * grid.z);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    float* out;
    cudaMalloc(&out, 4096);
    void* X;
    cudaMalloc(&X, 128 * 8192 * 2);
    cudaMemset(X, 0, 128 * 8192 * 2);
    struct Shape { const char* tag; int N, K; };
    Shape shapes[] = {{"qkv", 6144, 2048}, {"o", 2048, 2048}, {"fc1", 8192, 2048}, {"fc2", 2048, 8192}};
    for (auto& sh : shapes) {
        const size_t wb = (size_t)sh.N * sh.K * 2;
        const int nbuf = (int)(400e6 / wb) + 2;
        std::vector<void*> Ws(nbuf);
        for (auto& w : Ws) {
            cudaMalloc(&w, wb);
            cudaMemset(w, 0, wb);
        }
        // streaming reference over one buffer at a time
        {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int grid : {148, 296, 592, 1184}) {
                float tot = 0;
                for (int i = 0; i < 20; ++i) {
                    cudaEventRecord(a);
                    stream_ld<<<grid, 512>>>((const uint4*)Ws[i % nbuf], wb / 16, out);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    tot += ms;
                }
                printf("%-10s ld.v4 stream grid %4d: %7.2f us  %6.0f GB/s\n", sh.tag, grid, tot * 1e3 / 20,
                       wb / (tot * 1e3 / 20) / 1e3);
            }
        }
        const int nt = sh.N / BN, nk = sh.K / BK;
        for (int S : {1, 2, 3, 4, 6, 8}) {
            if (S > nk || nt * S > 600) continue;
            run<6, true, true>(sh.tag, sh.N, sh.K, S, Ws, X, out);
            run<6, false, false>(sh.tag, sh.N, sh.K, S, Ws, X, out);
            run<3, true, true>(sh.tag, sh.N, sh.K, S, Ws, X, out);
        }
        for (auto& w : Ws) cudaFree(w);
    }
    return 0;
}
