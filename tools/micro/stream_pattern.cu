// Microbenchmark: achievable HBM bandwidth for the GEMV's plane access pattern
// (16-row items, lanes (g,q) reading UB bytes of rows g and g+8 per plane,
// units strided over 15 warps, 2-deep register ring) vs a plain linear stream.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint2 ld8(const void* p) { uint2 r; asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p)); return r; }
__device__ __forceinline__ uint4 ld16(const void* p) { uint4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r; }

template <int K, int DEPTH>
__global__ void __launch_bounds__(512, 1) pattern(const uint8_t* planes, int64_t rows, int64_t row_bytes, int n_tiles, uint32_t* out, int spin) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int WC = 15; if (warp >= WC) return;
  const int64_t plane_stride = rows * row_bytes;
  const int n_items = (int)(rows / 16), upi = n_tiles * 4;  // UB = 8
  const int first = (int)((int64_t)n_items * blockIdx.x / gridDim.x), last = (int)((int64_t)n_items * (blockIdx.x + 1) / gridDim.x);
  const int64_t total = (int64_t)(last - first) * upi;
  uint32_t acc = 0;
  uint2 buf[DEPTH][2][K];
  auto load = [&](int64_t gidx, uint2 (&b)[2][K]) {
    if (gidx >= total) return;
    const int item = first + (int)(gidx / upi), u = (int)(gidx % upi);
    const int tile = u >> 2, s = u & 3;
    const uint8_t* p0 = planes + ((int64_t)item * 16 + g) * row_bytes + tile * 128 + s * 32 + q * 8;
#pragma unroll
    for (int p = 0; p < K; ++p) { b[0][p] = ld8(p0 + p * plane_stride); b[1][p] = ld8(p0 + 8 * row_bytes + p * plane_stride); }
  };
  int64_t gl = warp;
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) { load(gl, buf[d]); gl += WC; }
  int ring = 0;
  for (int64_t gi = warp; gi < total; gi += WC) {
    const int r = ring % DEPTH;
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) if (d == r) {
#pragma unroll
      for (int p = 0; p < K; ++p) acc ^= buf[d][0][p].x ^ buf[d][0][p].y ^ buf[d][1][p].x ^ buf[d][1][p].y;
      for (int i = 0; i < spin; ++i) acc = acc * 1664525u + 1013904223u;  // fake compute
      load(gl, buf[d]);
    }
    gl += WC; ++ring;
  }
  if (acc == 0x12345678) out[0] = acc;
}

__global__ void linear(const uint4* p, int64_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) { uint4 v = ld16(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const int64_t rows = 11008, cols = 4096, rb = cols / 8; const int n_tiles = cols / 1024;
  const int64_t bytes = 8 * rows * rb;  // 8 planes
  uint8_t* d; cudaMalloc(&d, bytes * 4); cudaMemset(d, 1, bytes * 4);
  uint32_t* o; cudaMalloc(&o, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); for (int c = 0; c < 4; ++c) linear<<<148 * 4, 512>>>((const uint4*)(d + c * bytes), bytes / 16, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("linear stream          : %.1f GB/s\n", 4 * bytes / (ms * 1e-3) / 1e9);
  }
  for (int spin : {0, 20, 60}) {
    cudaEventRecord(a); for (int c = 0; c < 4; ++c) pattern<8, 2><<<148, 512>>>(d + c * bytes, rows, rb, n_tiles, o, spin); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("pattern k=8 depth2 spin%2d: %.1f GB/s (%.1f us per layer)\n", spin, 4 * bytes / (ms * 1e-3) / 1e9, ms * 1e3 / 4);
    cudaEventRecord(a); for (int c = 0; c < 4; ++c) pattern<8, 4><<<148, 512>>>(d + c * bytes, rows, rb, n_tiles, o, spin); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("pattern k=8 depth4 spin%2d: %.1f GB/s\n", spin, 4 * bytes / (ms * 1e-3) / 1e9);
    cudaEventRecord(a); for (int c = 0; c < 4; ++c) pattern<3, 2><<<148, 512>>>(d + c * bytes, rows, rb, n_tiles, o, spin); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("pattern k=3 depth2 spin%2d: %.1f GB/s\n", spin, 4 * 3 * rows * rb / (ms * 1e-3) / 1e9);
  }
  return 0;
}
