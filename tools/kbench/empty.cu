// Floor of a PDL-chained launch with the GEMV's launch shape: per-launch time of
// a CUDA graph of 50 launches of an (almost) empty kernel.
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)
__global__ void empty_kernel(int* p) {
    extern __shared__ int sm[];
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && p) p[blockIdx.x] = blockIdx.x;
}
int main() {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* buf;
    CK(cudaMalloc(&buf, 4096 * 4));
    CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    struct Cfg { int grid, threads, smem; } cfgs[] = {{1, 32, 0}, {296, 320, 113 * 1024}, {148, 448, 195 * 1024}};
    for (auto c : cfgs) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c.grid);
        cfg.blockDim = dim3(c.threads);
        cfg.dynamicSmemBytes = c.smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
        for (int i = 0; i < 50; ++i) CK(cudaLaunchKernelEx(&cfg, empty_kernel, buf));
        CK(cudaStreamEndCapture(s, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaGraphLaunch(ge, s));
        CK(cudaStreamSynchronize(s));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid %4d x %3d threads, %3d KB smem: %.2f us per launch\n", c.grid, c.threads, c.smem / 1024,
               ms * 1e3 / 500);
    }
    return 0;
}
