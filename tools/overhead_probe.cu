// overhead_probe.cu — what makes a short kernel "long" on B200: event-timed duration (back to back, events around
// each launch, no host sync) of an empty 148x128 kernel with each GEMM-like ingredient added: 197 KB dynamic smem,
// TMEM alloc/dealloc, a (1,1,4) cluster, __grid_constant__ tensor-map-sized params, 2 CTAs/SM worth of grid.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2503_17707_b200/csrc tools/overhead_probe.cu -o tools/overhead_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"
using namespace pb::sm100;

struct Big {
    char b[384];
};

template <bool TMEM>
__global__ void k(const __grid_constant__ Big p, float* out) {
    __shared__ uint32_t slot;
    if (TMEM) {
        if (threadIdx.x < 32) tmem_alloc<128>(&slot);
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (threadIdx.x < 32) tmem_dealloc<128>(slot);
    }
    if (threadIdx.x == 1000) out[0] = p.b[threadIdx.x & 255];
}

int main() {
    float* out;
    cudaMalloc(&out, 64);
    Big p{};
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int n = 50;
    cudaEvent_t ev[2 * n];
    for (auto& e : ev) cudaEventCreate(&e);
    struct V { const char* name; bool tmem; int smem; int cluster; int grid; };
    V vs[] = {{"empty", false, 0, 1, 148},          {"smem197K", false, 197 * 1024, 1, 148},
              {"tmem", true, 0, 1, 148},            {"cluster4", false, 0, 4, 148},
              {"smem+tmem", true, 197 * 1024, 1, 148}, {"smem+tmem+cl4", true, 197 * 1024, 4, 148},
              {"grid296 smem96K", true, 96 * 1024, 4, 296}, {"grid64 smem197K cl4", true, 197 * 1024, 4, 64}};
    for (int rep = 0; rep < 2; ++rep)
        for (auto& v : vs) {
            auto kern = v.tmem ? k<true> : k<false>;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(v.grid / v.cluster, 1, v.cluster);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = v.smem;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = v.cluster;
            cfg.attrs = at;
            cfg.numAttrs = v.cluster > 1 ? 1 : 0;
            for (int i = 0; i < n; ++i) {
                cudaEventRecord(ev[2 * i], s);
                cudaLaunchKernelEx(&cfg, kern, p, out);
                cudaEventRecord(ev[2 * i + 1], s);
            }
            cudaError_t e = cudaStreamSynchronize(s);
            double tot = 0;
            for (int i = 5; i < n; ++i) {
                float ms;
                cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
                tot += ms;
            }
            // back-to-back without events
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, s);
            for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, kern, p, out);
            cudaEventRecord(b, s);
            cudaStreamSynchronize(s);
            float ms2;
            cudaEventElapsedTime(&ms2, a, b);
            if (rep) printf("%-22s events %6.2f us/launch   no-events %6.2f us/launch  %s\n", v.name, tot * 1e3 / (n - 5),
                            ms2 * 1e3 / n, cudaGetErrorString(e));
        }
    return 0;
}
