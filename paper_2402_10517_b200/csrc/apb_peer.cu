// apb_peer.cu -- the completion half of the fused GEMV + all-gather
// and the CUDA IPC plumbing for its buffers.
//
// Each rank's row-sharded GEMV (apb_gemv_grouped_peers) stores every y value
// into its own output and into each peer's output over NVLink, then adds the
// number of values it wrote to every rank's arrival counter.  A rank's output
// is complete once its counter has grown by the full output size (rows x batch
// rows) since the previous step; apb_peer_wait waits for exactly that.  The
// target lives in device memory and advances inside the kernel, so the same
// launch replays correctly from a CUDA graph; counters wrap modulo 2^32.
// The spin is bounded: on timeout the kernel sets *status = 1 (and advances its
// target anyway) instead of hanging the stream; the host checks the status.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/anyprec_b200.h"

namespace {

__global__ void peer_wait_kernel(const uint32_t* arrivals, uint32_t* expected, uint32_t per_step, int* status,
                                 long long spin_limit) {
    asm volatile("griddepcontrol.launch_dependents;");
    // the local GEMV's own contribution arrives through the same counter, so no
    // griddepcontrol.wait is needed for correctness; waiting first keeps the
    // spinning CTA off the SMs while the GEMV runs
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t target = *expected + per_step;
    long long spins = 0;
    while (true) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(arrivals) : "memory");
        if ((int32_t)(v - target) >= 0) break;
        if (++spins > spin_limit) {
            *status = 1;
            break;
        }
        __nanosleep(64);
    }
    *expected = target;
}

}  // namespace

extern "C" int apb_peer_wait(const uint32_t* arrivals, uint32_t* expected, uint32_t per_step, int* status,
                             long long spin_limit, void* stream) {
    if (!arrivals || !expected || !status || spin_limit <= 0) return APB_ERR_PARAM;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(1);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, peer_wait_kernel, arrivals, expected, per_step, status, spin_limit) != cudaSuccess)
        return APB_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

extern "C" int apb_peer_alloc(int64_t bytes, void** ptr, void* handle) {
    if (bytes <= 0 || !ptr || !handle) return APB_ERR_PARAM;
    void* p = nullptr;
    if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) return APB_ERR_CUDA;
    if (cudaMemset(p, 0, (size_t)bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        cudaFree(p);
        return APB_ERR_CUDA;
    }
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        return APB_ERR_CUDA;
    }
    memcpy(handle, &h, sizeof(h));
    *ptr = p;
    return APB_OK;
}

extern "C" int apb_peer_open(const void* handle, void** ptr) {
    if (!handle || !ptr) return APB_ERR_PARAM;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

extern "C" int apb_peer_close(void* ptr) {
    return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

extern "C" int apb_peer_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? APB_OK : APB_ERR_CUDA; }

extern "C" int apb_peer_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }
