// HBM bandwidth by access pattern (pure loads, 148 CTAs x 15 load warps, 2-deep ring).
// rows x 512 B planes (C = 4096), 8 planes, 4 layer copies (~360 MB).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint4 ld16(const void* p) { uint4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r; }
__device__ __forceinline__ uint2 ld8(const void* p) { uint2 r; asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p)); return r; }
// MODE 0: lanes (g,q): rows g,g+8; 8 B at q*8 + s*32 (current UB=8)
// MODE 1: lanes (g,q): rows g,g+8; 16 B at q*16 + h*64 (UB=16)
// MODE 2: lanes (r,c): 4 rows x 8 chunks of 16 B = full 128-B line per row (line-coalesced)
// MODE 3: each warp reads 512 contiguous bytes of one row (row-contiguous)
template <int MODE, int K>
__global__ void __launch_bounds__(512, 1) pat(const uint8_t* planes, int64_t rows, int64_t rb, uint32_t* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31; if (warp >= 15) return;
  const int64_t ps = rows * rb; const int n_items = (int)(rows / 16), n_tiles = (int)(rb / 128);
  const int first = (int)((int64_t)n_items * blockIdx.x / gridDim.x), last = (int)((int64_t)n_items * (blockIdx.x + 1) / gridDim.x);
  const int upi = MODE == 0 ? n_tiles * 4 : (MODE == 1 ? n_tiles * 2 : (MODE == 2 ? n_tiles * 4 : 16));
  const int64_t total = (int64_t)(last - first) * upi;
  uint32_t acc = 0;
  for (int64_t gi = warp; gi < total; gi += 15) {
    const int item = first + (int)(gi / upi), u = (int)(gi % upi);
    const uint8_t* base = planes + (int64_t)item * 16 * rb;
    uint4 v[K][2];
    if (MODE == 0) { const int g = lane >> 2, q = lane & 3, tile = u >> 2, s = u & 3;
      const uint8_t* p0 = base + g * rb + tile * 128 + s * 32 + q * 8;
#pragma unroll
      for (int p = 0; p < K; ++p) { uint2 a = ld8(p0 + p * ps), b = ld8(p0 + 8 * rb + p * ps); v[p][0] = make_uint4(a.x, a.y, b.x, b.y); v[p][1] = v[p][0]; }
    } else if (MODE == 1) { const int g = lane >> 2, q = lane & 3, tile = u >> 1, h = u & 1;
      const uint8_t* p0 = base + g * rb + tile * 128 + h * 64 + q * 16;
#pragma unroll
      for (int p = 0; p < K; ++p) { v[p][0] = ld16(p0 + p * ps); v[p][1] = ld16(p0 + 8 * rb + p * ps); }
    } else if (MODE == 2) { const int r = lane >> 3, c = lane & 7, tile = u >> 2, rq = u & 3;
      const uint8_t* p0 = base + (rq * 4 + r) * rb + tile * 128 + c * 16;
#pragma unroll
      for (int p = 0; p < K; ++p) { v[p][0] = ld16(p0 + p * ps); v[p][1] = v[p][0]; }
    } else { const uint8_t* p0 = base + u * rb + lane * 16;
#pragma unroll
      for (int p = 0; p < K; ++p) { v[p][0] = ld16(p0 + p * ps); v[p][1] = v[p][0]; }
    }
#pragma unroll
    for (int p = 0; p < K; ++p) acc ^= v[p][0].x ^ v[p][0].w ^ v[p][1].y;
  }
  if (acc == 0x12345678) out[0] = acc;
}
template <int MODE, int K> void run(const uint8_t* d, int64_t rows, int64_t rb, int64_t bytes, uint32_t* o, const char* name) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int c = 0; c < 4; ++c) pat<MODE, K><<<148, 512>>>(d + c * bytes, rows, rb, o);
  cudaEventRecord(a); for (int r = 0; r < 3; ++r) for (int c = 0; c < 4; ++c) pat<MODE, K><<<148, 512>>>(d + c * bytes, rows, rb, o);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  // bytes actually requested: K planes of rows x rb (MODE 3 reads all 16 rows per item too)
  printf("%-34s K=%d: %7.1f GB/s\n", name, K, 12.0 * K * rows * rb / (ms * 1e-3) / 1e9);
}
int main() {
  const int64_t rows = 11008 * 4, rb = 512, bytes = 8 * rows * rb;
  uint8_t* d; cudaMalloc(&d, bytes * 4); cudaMemset(d, 1, bytes * 4); uint32_t* o; cudaMalloc(&o, 64);
  run<0, 8>(d, rows, rb, bytes, o, "UB=8 lanes(g,q) 32B/row"); run<0, 3>(d, rows, rb, bytes, o, "UB=8 lanes(g,q) 32B/row");
  run<1, 8>(d, rows, rb, bytes, o, "UB=16 lanes(g,q) 64B/row"); run<1, 3>(d, rows, rb, bytes, o, "UB=16 lanes(g,q) 64B/row");
  run<2, 8>(d, rows, rb, bytes, o, "line: 4 rows x 128B"); run<2, 3>(d, rows, rb, bytes, o, "line: 4 rows x 128B");
  run<3, 8>(d, rows, rb, bytes, o, "row-contiguous 512B"); run<3, 3>(d, rows, rb, bytes, o, "row-contiguous 512B");
  return 0;
}
