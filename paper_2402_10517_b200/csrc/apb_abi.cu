// apb_abi.cu -- version / status strings of the C ABI (include/anyprec_b200.h).
#include "../../include/anyprec_b200.h"

extern "C" int apb_version(void) { return 100; /* 0.1.0 */ }

extern "C" const char* apb_status_string(int status) {
    switch (status) {
        case APB_OK: return "ok";
        case APB_ERR_SHAPE: return "shape error";
        case APB_ERR_PARAM: return "parameter error";
        case APB_ERR_LAYOUT: return "layout error";
        case APB_ERR_CODE_RANGE: return "code range error";
        case APB_ERR_CUDA: return "CUDA error";
        case APB_ERR_NCCL: return "NCCL error";
        default: return "unknown status";
    }
}

#include <cuda_runtime.h>

// Host-path plumbing for bindings without their own CUDA runtime handle:
// an ordered async copy on the caller's stream (kind 0 H2D, 1 D2H, 2 D2D) and
// a stream synchronisation.
extern "C" int apb_memcpy_async(void* dst, const void* src, int64_t bytes, int kind, void* stream) {
    if (!dst || !src || bytes < 0 || kind < 0 || kind > 2) return APB_ERR_PARAM;
    const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                       : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
    return cudaMemcpyAsync(dst, src, (size_t)bytes, k, (cudaStream_t)stream) == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

extern "C" int apb_stream_sync(void* stream) {
    return cudaStreamSynchronize((cudaStream_t)stream) == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}
