// pdl_probe.cu — cost of a kernel boundary on B200: a chain of 200 dependent small kernels (148 CTAs, ~1 us of
// work each) launched (a) plainly, (b) with programmatic dependent launch, (c) plainly inside a CUDA graph,
// (d) with PDL inside a CUDA graph. Prints us per kernel for each. Also a chain whose kernels use 200 KB of
// dynamic shared memory (like the GEMM) to see whether occupancy blocks the early launch.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/pdl_probe.cu -o tools/pdl_probe
#include <cuda_runtime.h>

#include <cstdio>

__global__ void work(float* buf, int iters) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    extern __shared__ float sm[];
    float x = buf[blockIdx.x * blockDim.x + threadIdx.x];
    for (int i = 0; i < iters; ++i) x = x * 1.0000001f + 1e-7f;
    if (threadIdx.x == 0 && sm != nullptr && iters < 0) sm[0] = x;
    buf[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

static cudaError_t launch(cudaStream_t s, bool pdl, float* buf, int iters, int smem) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, work, buf, iters);
}

int main() {
    float* buf;
    cudaMalloc(&buf, 148 * 128 * 4);
    cudaMemset(buf, 0, 148 * 128 * 4);
    cudaFuncSetAttribute(work, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int n = 200;
    for (int smem : {0, 200 * 1024}) {
        for (int iters : {0, 1000}) {
            for (int mode = 0; mode < 4; ++mode) {
                const bool pdl = mode & 1, graph = mode & 2;
                cudaGraphExec_t ge = nullptr;
                if (graph) {
                    cudaGraph_t g;
                    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
                    for (int i = 0; i < n; ++i) launch(s, pdl, buf, iters, smem);
                    cudaStreamEndCapture(s, &g);
                    cudaGraphInstantiate(&ge, g, 0);
                    cudaGraphLaunch(ge, s);
                } else {
                    for (int i = 0; i < 10; ++i) launch(s, pdl, buf, iters, smem);
                }
                cudaStreamSynchronize(s);
                // queue the whole chain behind a host-side wait so the launch rate of the host does not matter
                cudaEventRecord(e0, s);
                if (graph) cudaGraphLaunch(ge, s);
                else
                    for (int i = 0; i < n; ++i) launch(s, pdl, buf, iters, smem);
                cudaEventRecord(e1, s);
                cudaError_t err = cudaStreamSynchronize(s);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("smem %6d iters %5d %-6s %-5s: %6.2f us/kernel  (%s)\n", smem, iters, pdl ? "pdl" : "plain",
                       graph ? "graph" : "eager", ms * 1e3 / n, cudaGetErrorString(err));
            }
        }
    }
    return 0;
}
