// launch_probe.cu — fixed per-launch cost of a TMA-streaming kernel, timed the way bench.py times kernels
// (CUDA events around every launch, back to back on one stream, no host sync in between).
//   empty   : <<<148,128>>> doing nothing
//   setup   : mbarrier init + TMEM alloc/dealloc (the GEMM's prologue/epilogue skeleton)
//   stream  : TMA W-only streaming of B bytes over `ctas` CTAs, `stages` x 16 KB in flight per CTA
//   pair    : a tiny SIMT kernel (no smem) before each stream launch, with / without max smem carveout
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2503_17707_b200/csrc \
//        tools/launch_probe.cu -o tools/launch_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace pb::sm100;

__global__ void empty_kernel(float* out) {
    if (threadIdx.x == 1000) out[0] = 1;
}

__global__ void small_kernel(float* out) {   // a "norm-like" kernel: 128 CTAs, no smem
    if (threadIdx.x == 0) out[blockIdx.x] += 1.0f;
}

__global__ void setup_kernel(float* out) {
    __shared__ uint64_t bar[4];
    __shared__ uint32_t slot;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc<128>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<128>(slot);
    if (threadIdx.x == 1000) out[0] = 1;
}

// W [rows x K] bf16, box {64, 128}: CTA c streams boxes c, c + ctas, ... (row tile = box / nk, k = box % nk).
template <int STAGES>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap mapW, int nk, int nboxes,
                                                        float* out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * 16384);
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&mapW);
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int i = 0;
        for (int b = blockIdx.x; b < nboxes; b += gridDim.x, ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) mbar_wait(&full[s], ((i / STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], 16384);
            tma_load_2d(smem + s * 16384, &mapW, &full[s], (b % nk) * 64, (b / nk) * 128);
        }
        for (int j = i > STAGES ? i - STAGES : 0; j < i; ++j) mbar_wait(&full[j % STAGES], (j / STAGES) & 1);
        if (smem[5] == 123 && smem[77] == 45) out[0] = 1;
    }
}

using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static Encode enc;
static CUtensorMap map2d(void* base, uint64_t rows, uint64_t cols) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t str[1] = {cols * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
}

struct Timer {
    std::vector<cudaEvent_t> ev;
    explicit Timer(int n) : ev(2 * n) {
        for (auto& e : ev) cudaEventCreate(&e);
    }
    template <class F>
    double run(int n, F f) {   // back-to-back, events around every launch, one sync at the end
        for (int i = 0; i < n; ++i) {
            cudaEventRecord(ev[2 * i]);
            f(i);
            cudaEventRecord(ev[2 * i + 1]);
        }
        cudaDeviceSynchronize();
        double tot = 0;
        for (int i = 0; i < n; ++i) {
            float ms;
            cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
            tot += ms;
        }
        return tot * 1e3 / n;
    }
};

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    float* out;
    cudaMalloc(&out, 1 << 20);
    cudaMemset(out, 0, 1 << 20);
    const int n = 40;
    Timer T(2 * n);
    for (int rep = 0; rep < 2; ++rep) {
        printf("empty  <<<148,128>>>            : %6.2f us\n", T.run(n, [&](int) { empty_kernel<<<148, 128>>>(out); }));
        printf("small  <<<128,256>>>            : %6.2f us\n", T.run(n, [&](int) { small_kernel<<<128, 256>>>(out); }));
        printf("setup  <<<148,128>>> tmem+mbar  : %6.2f us\n", T.run(n, [&](int) { setup_kernel<<<148, 128>>>(out); }));
    }
    // W buffers: rotate so every launch reads HBM
    const size_t total = 640ull << 20;
    void* W;
    cudaMalloc(&W, total);
    cudaMemset(W, 1, total);
    const int K = 2048;
    for (size_t mb : {8, 16, 33, 64}) {
        const size_t bytes = mb << 20;
        const int rows = (int)(bytes / (K * 2)) / 128 * 128;
        const int nk = K / 64, nboxes = rows / 128 * nk;
        const int nbuf = (int)(total / bytes);
        std::vector<CUtensorMap> maps;
        for (int b = 0; b < nbuf; ++b) maps.push_back(map2d((char*)W + b * bytes, rows, K));
        for (int stages : {6, 12}) {
            for (int ctas : {148, 296}) {
                auto kern = stages == 6 ? stream_kernel<6> : stream_kernel<12>;
                const int sm = stages * 16384 + 1024 + 256;
                if (ctas == 296 && sm > 110000) continue;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
                double us = T.run(n, [&](int i) { kern<<<ctas, 128, sm>>>(maps[i % nbuf], nk, nboxes, out); });
                printf("stream %3zu MB stages %2d ctas %3d        : %6.2f us  %6.0f GB/s\n", mb, stages, ctas, us,
                       rows * (double)K * 2 / us / 1e3);
                // with a small no-smem kernel in front (carveout reconfiguration?)
                for (int carve : {-1, 100}) {
                    cudaFuncSetAttribute(small_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
                    double us2 = T.run(2 * n, [&](int i) {
                        if (i & 1) kern<<<ctas, 128, sm>>>(maps[(i / 2) % nbuf], nk, nboxes, out);
                        else small_kernel<<<128, 256>>>(out);
                    });
                    printf("   alternating with small kernel (carveout %4d): avg of pair members %6.2f us\n", carve, us2);
                }
            }
        }
        // the whole sequence without per-launch events: steady-state throughput
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaFuncSetAttribute(stream_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384 + 1280);
        cudaEventRecord(a);
        for (int i = 0; i < n; ++i) stream_kernel<6><<<148, 128, 6 * 16384 + 1280>>>(maps[i % nbuf], nk, nboxes, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("stream %3zu MB back-to-back, no events  : %6.2f us/launch  %6.0f GB/s\n", mb, ms * 1e3 / n,
               rows * (double)K * 2 * n / (ms * 1e-3) / 1e9);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
