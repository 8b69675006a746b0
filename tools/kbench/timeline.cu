// timeline: per-CTA phase stamps of one v7 GEMV launch (APB_TIMELINE build).
// stamps: 0 CTA start | 1 first table built | 2 x issued (after PDL wait)
//         3 first stage seen (warp 0) | 4 first item done (warp 0)
//         5 service done (last y stored) | 6 producer done issuing
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../include/anyprec_b200.h"
extern "C" int apb7_read_timeline(unsigned long long* host, int n);
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)
__global__ void fill(uint8_t* p, size_t n, uint32_t s) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { uint32_t h = (uint32_t)i * 2654435761u ^ s; h ^= h >> 13; h *= 0x5bd1e995u; p[i] = (uint8_t)(h >> 8); } }
int main() {
    cudaStream_t s; CK(cudaStreamCreate(&s));
    const int64_t shapes[][2] = {{4096, 4096}, {11008, 4096}};
    for (auto& sh : shapes) {
        int64_t R = sh[0], C = sh[1], Cp = apb_pad_columns(C);
        uint8_t *planes; uint16_t *lut, *x; float* y;
        CK(cudaMalloc(&planes, 8 * R * Cp / 8)); CK(cudaMalloc(&lut, R * 256 * 2)); CK(cudaMalloc(&x, C * 2)); CK(cudaMalloc(&y, R * 4));
        fill<<<512, 256>>>(planes, 8 * R * Cp / 8, 1); fill<<<512, 256>>>((uint8_t*)lut, R * 512, 2); CK(cudaMemset(x, 0, C * 2));
        for (int k : {3, 8}) {
            for (int it = 0; it < 3; ++it) apb_gemv(planes, 8, R, C, Cp, k, lut, x, 1, C, 0, y, APB_DTYPE_F32, R, 0, s);
            CK(cudaStreamSynchronize(s));
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a, s);
            apb_gemv(planes, 8, R, C, Cp, k, lut, x, 1, C, 0, y, APB_DTYPE_F32, R, 0, s);
            cudaEventRecord(b, s); CK(cudaStreamSynchronize(s));
            float ms; cudaEventElapsedTime(&ms, a, b);
            std::vector<unsigned long long> t(64 * 512 * 8);
            apb7_read_timeline(t.data(), 64 * 512 * 8);
            { // the timed launch is the newest: find the launch slot with the latest start
                int best = 0; unsigned long long bt = 0;
                for (int l = 0; l < 64; ++l) if (t[(size_t)l * 512 * 8] > bt) { bt = t[(size_t)l * 512 * 8]; best = l; }
                std::vector<unsigned long long> u(t.begin() + (size_t)best * 512 * 8, t.begin() + (size_t)(best + 1) * 512 * 8);
                t.swap(u);
            }
            unsigned long long t0 = ~0ull, tend = 0;
            for (int c = 0; c < 148; ++c) if (t[c * 8]) { t0 = std::min(t0, t[c * 8]); tend = std::max(tend, t[c * 8 + 5]); }
            printf("%lldx%lld k=%d event %.2f us, CTA span %.2f us\n", (long long)R, (long long)C, k, ms * 1e3, (tend - t0) / 1e3);
            const char* nm[] = {"start", "table0", "x_issue", "stage0", "item0", "svc_end", "prod_end"};
            for (int i = 0; i < 7; ++i) {
                std::vector<double> v;
                for (int c = 0; c < 148; ++c) if (t[c * 8] && t[c * 8 + i]) v.push_back((t[c * 8 + i] - t0) / 1e3);
                std::sort(v.begin(), v.end());
                if (v.empty()) continue;
                printf("   %-9s min %6.2f  med %6.2f  max %6.2f us\n", nm[i], v.front(), v[v.size() / 2], v.back());
            }
        }
        cudaFree(planes); cudaFree(lut); cudaFree(x); cudaFree(y);
    }
}
