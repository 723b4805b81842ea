// xchg_probe.cu — cost of the split-K partial exchange of gemm_kernel on B200, by transport.
// A cluster of S = 4 CTAs each holds a 128 x TBN fp32 partial tile in shared memory (as after the mainloop); CTA s
// must end up with rows [32 s, 32 s + 32) summed over the 4 partials in the fixed order 0..3 and written to global.
//   0 none    : only the CTA's own partial (the floor: staging + stores)
//   1 dsmem   : ld.shared::cluster of the peers' rows after a cluster barrier (gemm_kernel today)
//   2 bulk    : each CTA pushes the rows a peer owns with cp.async.bulk shared::cta -> shared::cluster (the copy engine
//               of the SM, mbarrier complete_tx in the owner), the owner sums locally
//   3 l2      : each CTA st.global's the rows a peer owns into a workspace, cluster barrier, owner ld.global's them
// Reports per-variant the median / max over CTAs of the globaltimer span from "partial staged" to "rows stored", and
// the mean kernel time over 200 launches (events). Build:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/xchg_probe.cu -o tools/xchg_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int S = 4, ROWS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ float4 ld_cl(uint32_t a) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(smem_u32(b)),
        "r"(ph)
        : "memory");
}

template <int TBN>
__device__ __forceinline__ uint32_t part_off(int row, int chunk) {
    return (uint32_t)(row * (TBN * 4) + ((chunk ^ (row & (TBN / 4 - 1))) << 4));
}

template <int V, int TBN>
__global__ void __launch_bounds__(128, 1) xchg(float* out, float* ws, unsigned long long* span) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int CH = TBN / 4, RB = ROWS / S;                // float4 chunks per row, rows per owner
    constexpr int kPart = ROWS * TBN * 4, kBlk = RB * TBN * 4; // 64 KB / 16 KB at TBN 128
    uint8_t* recv = smem + kPart;                              // [S-1][RB][TBN] fp32 (bulk variant; slot of source s)
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kPart + (S - 1) * kBlk);
    const int tid = threadIdx.x, rank = (int)cluster_rank();
    const int cl = blockIdx.x / S;
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // stage: row = tid, the layout gemm_kernel writes
    for (int c = 0; c < CH; ++c)
        *reinterpret_cast<float4*>(smem + part_off<TBN>(tid, c)) =
            make_float4(rank + tid * 1e-3f, c, 1.f, 2.f);
    if (V == 2) {
        if (tid == 0) mbar_expect(bar, (S - 1) * kBlk);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const unsigned long long t0 = gt();
    const int r_lo = RB * rank;
    if (V == 3) {   // rows of peer p -> ws[cl][rank][p]
        const int p = tid / RB, r = tid % RB + RB * p;
        if (p != rank) {
            float4* dst = reinterpret_cast<float4*>(ws + (((size_t)cl * S + rank) * S + p) * RB * TBN) + (r - RB * p) * CH;
#pragma unroll 8
            for (int c = 0; c < CH; ++c) dst[c] = *reinterpret_cast<const float4*>(smem + part_off<TBN>(r, c));
        }
    }
    if (V != 0) cluster_sync();
    if (V == 2) {
        if (tid < S && tid != rank) {   // thread p pushes the rows owner p reduces into slot `rank` of p's recv
            const int p = tid;
            // the partial is stored swizzled per row; rows [RB p, RB p + RB) are contiguous (kBlk bytes)
            const uint32_t src = smem_u32(smem) + RB * p * TBN * 4;
            const uint32_t dst = mapa(smem_u32(recv) + (rank < p ? rank : rank - 1) * kBlk, p), mb = mapa(smem_u32(bar), p);
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "r"(src), "r"(kBlk), "r"(mb)
                : "memory");
        }
        mbar_wait(bar, 0);
    }
    const uint32_t base = smem_u32(smem);
    for (int idx = tid; idx < RB * CH; idx += 128) {
        const int r = r_lo + idx / CH, ch = idx % CH;
        float4 acc;
        if (V == 0) {
            acc = *reinterpret_cast<const float4*>(smem + part_off<TBN>(r, ch));
        } else {
            float4 p[S];
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) {
                if (V == 1) p[s2] = ld_cl(mapa(base + part_off<TBN>(r, ch), s2));
                else if (V == 2) p[s2] = s2 == rank ? *reinterpret_cast<const float4*>(smem + part_off<TBN>(r, ch))
                                                    : *reinterpret_cast<const float4*>(recv + (s2 < rank ? s2 : s2 - 1) * kBlk + part_off<TBN>(r, ch) - RB * rank * TBN * 4);
                else p[s2] = s2 == rank ? *reinterpret_cast<const float4*>(smem + part_off<TBN>(r, ch))
                                        : __ldcg(reinterpret_cast<const float4*>(ws + (((size_t)cl * S + s2) * S + rank) * RB * TBN) +
                                                 (r - r_lo) * CH + ch);
            }
            acc = p[0];
#pragma unroll
            for (int s2 = 1; s2 < S; ++s2) {
                acc.x += p[s2].x;
                acc.y += p[s2].y;
                acc.z += p[s2].z;
                acc.w += p[s2].w;
            }
        }
        reinterpret_cast<float4*>(out)[((size_t)blockIdx.x * RB + (r - r_lo)) * CH + ch] = acc;
    }
    if (V == 1) cluster_sync();
    __syncthreads();
    if (tid == 0) span[blockIdx.x] = gt() - t0;
}

template <int V, int TBN>
void run(int ctas, int smem, const char* name) {
    float *out, *ws;
    unsigned long long* span;
    cudaMalloc(&out, (size_t)ctas * ROWS * TBN * 4);
    cudaMalloc(&ws, (size_t)ctas * ROWS * TBN * 4 * 2);
    cudaMalloc(&span, ctas * 8);
    cudaFuncSetAttribute(xchg<V, TBN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(xchg<V, TBN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int i = 0; i < 5; ++i) cudaLaunchKernelEx(&cfg, xchg<V, TBN>, out, ws, span);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 200; ++i) cudaLaunchKernelEx(&cfg, xchg<V, TBN>, out, ws, span);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(ctas);
    cudaMemcpy(h.data(), span, ctas * 8, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    // check: owner of rows [32s, 32s+32) of cluster cl: sum over ranks of (rank + row*1e-3) in x
    std::vector<float> ho((size_t)ctas * ROWS / S * TBN);
    cudaMemcpy(ho.data(), out, ho.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    if (V != 0)
        for (int b = 0; b < ctas; ++b) {
            const int rank = b % S;
            for (int r = 0; r < ROWS / S; ++r) {
                const int row = rank * ROWS / S + r;
                const float want = (0 + row * 1e-3f) + (1 + row * 1e-3f) + (2 + row * 1e-3f) + (3 + row * 1e-3f);
                const float got = ho[((size_t)b * ROWS / S + r) * TBN];
                maxerr = std::max(maxerr, (double)std::abs(got - want));
            }
        }
    printf("{\"variant\": \"%s\", \"tbn\": %d, \"ctas\": %d, \"smem_kb\": %d, \"span_ns_median\": %llu, \"span_ns_max\": %llu, "
           "\"kernel_us\": %.2f, \"maxerr\": %.3g, \"err\": \"%s\"}\n",
           name, TBN, ctas, smem >> 10, h[ctas / 2], h[ctas - 1], ms * 1000 / 200, maxerr, cudaGetErrorString(err));
    cudaFree(out);
    cudaFree(ws);
    cudaFree(span);
}

int main() {
    // TBN 128: partial 64 KB + recv 48 KB + bar; 2 CTAs per SM at ~113 KB (QKV / FC1 at C2: 192 / 256 CTAs)
    const int sm2 = 113 * 1024, sm1 = 200 * 1024;
    for (int ctas : {192, 144}) {
        const int sm = ctas == 192 ? sm2 : sm1;
        run<0, 128>(ctas, sm, "none");
        run<1, 128>(ctas, sm, "dsmem");
        run<2, 128>(ctas, sm, "bulk");
        run<3, 128>(ctas, sm, "l2");
    }
    // TBN 64 (O / FC2 at C2: 128 CTAs, one per SM)
    run<0, 64>(128, sm1, "none");
    run<1, 64>(128, sm1, "dsmem");
    run<2, 64>(128, sm1, "bulk");
    run<3, 64>(128, sm1, "l2");
    return 0;
}
