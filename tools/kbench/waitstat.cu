// waitstat: fraction of compute-warp time spent waiting for plane stages (ring
// 'full' barrier) in one steady-state GEMV launch -- APB_TIMELINE build.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../include/anyprec_b200.h"
extern "C" int apb7_read_timeline(unsigned long long* host, int n);
extern "C" void apb7_timeline_reset(void);
__global__ void fill(uint8_t* p, size_t n, uint32_t s) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { uint32_t h = (uint32_t)i * 2654435761u ^ s; h ^= h >> 13; h *= 0x5bd1e995u; p[i] = (uint8_t)(h >> 8); } }
int main() {
    const int64_t shapes[][2] = {{28672, 8192}, {11008, 4096}, {4096, 4096}};
    for (auto& sh : shapes) {
        int64_t R = sh[0], C = sh[1], Cp = apb_pad_columns(C);
        uint8_t* planes; uint16_t *lut, *x; float* y;
        cudaMalloc(&planes, 8 * R * Cp / 8); cudaMalloc(&lut, R * 256 * 2); cudaMalloc(&x, C * 2); cudaMalloc(&y, R * 4);
        fill<<<512, 256>>>(planes, 8 * R * Cp / 8, 1); fill<<<512, 256>>>((uint8_t*)lut, R * 512, 2); cudaMemset(x, 0, C * 2);
        for (int k : {3, 5, 8}) {
            for (int it = 0; it < 3; ++it) apb_gemv(planes, 8, R, C, Cp, k, lut, x, 1, C, 0, y, APB_DTYPE_F32, R, 0, 0);
            cudaDeviceSynchronize();
            apb7_timeline_reset();
            apb_gemv(planes, 8, R, C, Cp, k, lut, x, 1, C, 0, y, APB_DTYPE_F32, R, 0, 0);
            cudaDeviceSynchronize();
            std::vector<unsigned long long> t(64 * 512 * 8);
            apb7_read_timeline(t.data(), 64 * 512 * 8);
            double fr = 0; int n = 0; double mx = 0, cyc = 0;
            for (int c = 0; c < 512; ++c) {
                unsigned long long v = t[(size_t)c * 8 + 7];
                if (!v) continue;
                double wait = (double)(v >> 32), tot = (double)(v & 0xFFFFFFFFull);
                if (tot > 0) { fr += wait / tot; ++n; mx = std::max(mx, wait / tot); cyc += tot; }
            }
            // in-loop rate: a CTA's weights over its loop cycles, x CTAs per SM (n / 148)
            const double wpc = n ? ((double)R * C / n) / (cyc / n) * ((double)n / 148) : 0;
            printf("%lldx%lld k=%d: warp-0 time waiting for plane stages: mean %.1f %% (max %.1f %%) over %d CTAs; "
                   "in-loop rate %.1f w/clk/SM (loop %.1f us avg)\n",
                   (long long)R, (long long)C, k, n ? 100 * fr / n : 0.0, 100 * mx, n, wpc, n ? cyc / n / 1965.0 : 0.0);
        }
        cudaFree(planes); cudaFree(lut); cudaFree(x); cudaFree(y);
    }
}
