// rownorm.cuh — the LayerNorm / RMSNorm row arithmetic shared by norm_kernel (simt.cu) and the norm items of the
// layer chain (chain.cu), so both produce identical bits.
//
// A row of d fp32 values is reduced by 256 virtual threads: virtual thread v sums elements v, v + 256, v + 512, ...
// in that order, each group of 32 virtual threads is reduced by an xor butterfly, and the 8 group sums by a
// second butterfly. Every operation is an explicit round-to-nearest intrinsic (no contraction the compiler
// could choose differently in the two kernels). Two-pass statistics: mean, then the mean of squared deviations.
#pragma once
#include <cuda_bf16.h>

namespace pb {
namespace rownorm {

constexpr int kVT = 256;   // virtual threads per row

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// Sum of the 8 group sums red[0..7] (every lane of the calling warp gets it).
__device__ __forceinline__ float combine8(const float* red, int lane) {
    return warp_sum(lane < 8 ? red[lane] : 0.f);
}
__device__ __forceinline__ float acc_sum(float s, float x) { return __fadd_rn(s, x); }
__device__ __forceinline__ float acc_sq(float q, float x, float mean) {
    const float t = __fsub_rn(x, mean);
    return __fmaf_rn(t, t, q);
}
__device__ __forceinline__ float mean_of(float total, int d) { return __fdiv_rn(total, (float)d); }
__device__ __forceinline__ float rstd_of(float sq_total, int d, float eps) {
    return rsqrtf(__fadd_rn(__fdiv_rn(sq_total, (float)d), eps));
}
__device__ __forceinline__ __nv_bfloat16 out_f(float x, float mean, float rstd, float g, float b, bool has_beta) {
    float y = __fmul_rn(__fmul_rn(__fsub_rn(x, mean), rstd), g);
    if (has_beta) y = __fadd_rn(y, b);
    return __float2bfloat16_rn(y);
}
__device__ __forceinline__ __nv_bfloat16 out(float x, float mean, float rstd, const __nv_bfloat16* gamma,
                                             const __nv_bfloat16* beta, int c) {
    return out_f(x, mean, rstd, __bfloat162float(gamma[c]), beta ? __bfloat162float(beta[c]) : 0.f, beta != nullptr);
}

}  // namespace rownorm
}  // namespace pb
