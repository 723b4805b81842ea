// driver.cpp — CUDA driver entry points (resolved through the runtime, no -lcuda):
// TMA tensor-map encoding and stream memory operations (cross-rank readiness waits).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>

#include "kernels.hpp"

namespace pb {

namespace {
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using WaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using GetErrorString = CUresult (*)(CUresult, const char**);

EncodeTiled g_encode = nullptr;
WaitValue32 g_wait32 = nullptr;
WriteValue32 g_write32 = nullptr;
GetErrorString g_errstr = nullptr;
std::once_flag g_once;
bool g_ok = false;
char g_err[256] = "";

void* entry(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return fn;
}
}  // namespace

bool driver_init(char* err, size_t errlen) {
    std::call_once(g_once, [] {
        g_encode = reinterpret_cast<EncodeTiled>(entry("cuTensorMapEncodeTiled"));
        g_wait32 = reinterpret_cast<WaitValue32>(entry("cuStreamWaitValue32"));
        g_write32 = reinterpret_cast<WriteValue32>(entry("cuStreamWriteValue32"));
        g_errstr = reinterpret_cast<GetErrorString>(entry("cuGetErrorString"));
        g_ok = g_encode && g_wait32 && g_write32;
        if (!g_ok) snprintf(g_err, sizeof g_err, "driver entry points unavailable (cuTensorMapEncodeTiled/cuStreamWaitValue32)");
    });
    if (!g_ok && err) snprintf(err, errlen, "%s", g_err);
    return g_ok;
}

bool make_map_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                   uint32_t box_rows, uint32_t box_cols, int swizzle_bytes, char* err, size_t errlen) {
    if (!driver_init(err, errlen)) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        const char* s = "?";
        if (g_errstr) g_errstr(r, &s);
        snprintf(err, errlen,
                 "cuTensorMapEncodeTiled failed (%d: %s) base=%p rows=%llu cols=%llu ld=%llu box=%ux%u sw=%d", (int)r,
                 s, base, (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)ld_elems, box_rows,
                 box_cols, swizzle_bytes);
        return false;
    }
    return true;
}

bool make_map_bf16_3d(CUtensorMap* map, const void* base, const uint64_t dims[3], const uint64_t strides_bytes[2],
                      const uint32_t box[3], int swizzle_bytes, char* err, size_t errlen) {
    if (!driver_init(err, errlen)) return false;
    cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
    cuuint64_t st[2] = {strides_bytes[0], strides_bytes[1]};
    cuuint32_t bx[3] = {box[0], box[1], box[2]};
    cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), d, st, bx, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        const char* s = "?";
        if (g_errstr) g_errstr(r, &s);
        snprintf(err, errlen, "cuTensorMapEncodeTiled (3-D) failed (%d: %s) base=%p dims=%llux%llux%llu", (int)r, s,
                 base, (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2]);
        return false;
    }
    return true;
}

cudaError_t stream_wait_geq(cudaStream_t s, const uint32_t* dev_addr, uint32_t value) {
    if (!g_wait32) return cudaErrorNotSupported;
    CUresult r = g_wait32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(dev_addr), value,
                          CU_STREAM_WAIT_VALUE_GEQ);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

cudaError_t stream_write(cudaStream_t s, uint32_t* dev_addr, uint32_t value) {
    if (!g_write32) return cudaErrorNotSupported;
    // default flags: a memory barrier orders every prior write of the stream before this one
    CUresult r = g_write32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(dev_addr), value,
                           CU_STREAM_WRITE_VALUE_DEFAULT);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

}  // namespace pb
