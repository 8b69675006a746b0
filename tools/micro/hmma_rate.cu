// Microbenchmark: legacy mma.sync HMMA.16816.F32 throughput per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
template <int CHAINS>
__global__ void k(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[CHAINS][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 1024 * 4 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    k<4><<<148, warps * 32>>>(o, 16); cudaDeviceSynchronize();
    cudaEventRecord(a); k<4><<<148, warps * 32>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double hmma = 148.0 * warps * iters * 4;
    printf("warps/SM %2d chains 4: %.3f ms  %.3f HMMA/clk/SM @1.9GHz  (%.1f TFLOPs)\n", warps, ms,
           hmma / 148 / (ms * 1e-3 * 1.9e9), hmma * 4096 / (ms * 1e-3) / 1e12);
  }
  for (int warps : {4, 16}) {
    k<1><<<148, warps * 32>>>(o, 16); cudaDeviceSynchronize();
    cudaEventRecord(a); k<1><<<148, warps * 32>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("warps/SM %2d chains 1: latency-bound %.1f cycles per dependent HMMA\n", warps, ms * 1e-3 * 1.9e9 / iters);
  }
  return 0;
}
