// kbench: standalone timing + correctness harness for the GEMV C-ABI
// (no torch).  For each (shape, k): random permuted planes / fp16 LUT / fp16 x
// on the device, NCOPY weight copies (> L2) rotated per launch, launches
// captured in a CUDA graph (PDL chain), CUDA-event timing.  Correctness:
// a naive reference kernel (per-weight bit extraction, fp64 accumulate).
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <string>
#include <cmath>
#include "../../include/anyprec_b200.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void fill_rand(uint8_t* p, size_t n, uint32_t seed) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        p[i] = (uint8_t)h;
    }
}
__global__ void fill_half(__half* p, size_t n, uint32_t seed, float scale) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        p[i] = __float2half(((h & 0xFFFF) / 65536.0f - 0.5f) * scale);
    }
}
// planes permuted: byte (4t+j) of a 128-byte tile-plane-row holds bits of weights 256j+8t+i
__global__ void ref_gemv(const uint8_t* planes, int64_t R, int64_t C, int64_t Cp, int k,
                         const __half* lut, const __half* x, double* y) {
    int64_t r = blockIdx.x;
    x += blockIdx.y * ((C + 7) / 8 * 8);
    y += blockIdx.y * R;
    double acc = 0;
    const int64_t rb = Cp / 8;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
        int64_t tile = c / 1024, w = c % 1024;
        int j = w / 256, t = (w % 256) / 8, i = w % 8;
        int64_t byte = r * rb + tile * 128 + 4 * t + j;
        int code = 0;
        for (int p = 0; p < k; ++p) code = (code << 1) | ((planes[p * R * rb + byte] >> i) & 1);
        acc += (double)__half2float(lut[r * (1 << k) + code]) * (double)__half2float(x[c]);
    }
    __shared__ double s[256];
    s[threadIdx.x] = acc; __syncthreads();
    for (int o = 128; o; o >>= 1) { if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o]; __syncthreads(); }
    if (threadIdx.x == 0) y[r] = s[0];
}

struct Layer { int64_t R, C, Cp; std::vector<uint8_t*> planes; std::vector<__half*> lut; __half* x; float* y; };

static Layer make_layer(int64_t R, int64_t C, int ncopy, uint32_t seed, int M) {
    Layer L; L.R = R; L.C = C; L.Cp = apb_pad_columns(C);
    size_t pb = (size_t)8 * R * (L.Cp / 8);
    for (int c = 0; c < ncopy; ++c) {
        uint8_t* p; CK(cudaMalloc(&p, pb)); fill_rand<<<1024, 256>>>(p, pb, seed + 77 * c);
        __half* t; CK(cudaMalloc(&t, (size_t)R * 256 * 2 * 2));
        fill_half<<<1024, 256>>>(t, (size_t)R * 512, seed + 1000 + c, 2.0f);
        L.planes.push_back(p); L.lut.push_back(t);
    }
    int64_t ldx = (C + 7) / 8 * 8;
    CK(cudaMalloc(&L.x, M * ldx * 2)); fill_half<<<64, 256>>>(L.x, M * ldx, seed + 5, 2.0f);
    CK(cudaMalloc(&L.y, M * R * 4));
    return L;
}

// lut for bit width k lives at lut + lut_off(k) (tables for k=2..8 packed back to back)
static int64_t lut_off(int64_t R, int k) { int64_t o = 0; for (int b = 2; b < k; ++b) o += R << b; return o; }

int main(int argc, char** argv) {
    int ncopy = getenv("KB_NCOPY") ? atoi(getenv("KB_NCOPY")) : 4, reps = 20;  // KB_NCOPY=1: L2-resident weights
    std::string only = argc > 1 ? argv[1] : "";
    int konly = argc > 2 ? atoi(argv[2]) : 0;   // 0 = k 3..8
    if (argc > 3) reps = atoi(argv[3]);
    const int M = argc > 4 ? atoi(argv[4]) : 1;  // batch rows
    CK(cudaSetDevice(0));
    cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct Shape { const char* n; int64_t R, C; };
    std::vector<Shape> shapes = {{"4096x4096", 4096, 4096}, {"11008x4096", 11008, 4096}, {"4096x11008", 4096, 11008},
                                 {"28672x8192", 28672, 8192}};
    double* yref; CK(cudaMalloc(&yref, 8 * 28672 * 8));
    std::vector<double> h_ref(8 * 28672); std::vector<float> h_y(8 * 28672);
    for (auto& sh : shapes) {
        if (!only.empty() && only.find(sh.n) == std::string::npos && only != "all") continue;
        int nc = sh.R * sh.C > 100000000 && ncopy > 2 ? 2 : ncopy;
        Layer L = make_layer(sh.R, sh.C, nc, 1234, M);
        CK(cudaDeviceSynchronize());
        printf("%-11s", sh.n);
        for (int k = 3; k <= 8; ++k) {
            if (konly && k != konly) continue;
            int64_t ldx = (sh.C + 7) / 8 * 8;
            auto launch = [&](int c) {
                int rc = apb_gemv(L.planes[c], 8, sh.R, sh.C, L.Cp, k, (const uint16_t*)(L.lut[c] + lut_off(sh.R, k)),
                                  (const uint16_t*)L.x, M, ldx, 0, L.y, APB_DTYPE_F32, sh.R, APB_FLAG_PDL, s);
                if (rc) { fprintf(stderr, "apb_gemv rc=%d\n", rc); exit(1); }
            };
            // correctness vs naive reference (copy 0)
            launch(0); CK(cudaStreamSynchronize(s));
            ref_gemv<<<dim3(sh.R, M), 256, 0, s>>>(L.planes[0], sh.R, sh.C, L.Cp, k, L.lut[0] + lut_off(sh.R, k), L.x, yref);
            CK(cudaStreamSynchronize(s));
            CK(cudaMemcpy(h_y.data(), L.y, M * sh.R * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(h_ref.data(), yref, M * sh.R * 8, cudaMemcpyDeviceToHost));
            double num = 0, den = 0;
            for (int64_t r = 0; r < M * sh.R; ++r) { num += (h_y[r] - h_ref[r]) * (h_y[r] - h_ref[r]); den += h_ref[r] * h_ref[r]; }
            double err = sqrt(num / den);
            // timing: graph of reps*nc launches
            cudaGraph_t g; cudaGraphExec_t ge;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
            for (int i = 0; i < reps; ++i) for (int c = 0; c < nc; ++c) launch(c);
            CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
            CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            float best = 1e30f;
            for (int t = 0; t < 3; ++t) {
                cudaEventRecord(a, s); CK(cudaGraphLaunch(ge, s)); cudaEventRecord(b, s); CK(cudaStreamSynchronize(s));
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            double us = best * 1e3 / (reps * nc);
            double bytes = (double)sh.R * sh.C * k / 8 + sh.R * (1 << k) * 2 + M * (sh.C * 2 + sh.R * 2);
            printf(" | k%d %6.2fus %5.0fGB/s%s", k, us, bytes / us * 1e-3, err < 1e-3 ? "" : " ERR");
            if (err >= 1e-3) printf("(%.2e)", err);
            fflush(stdout);
            cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
        }
        printf("\n");
        for (int c = 0; c < nc; ++c) { cudaFree(L.planes[c]); cudaFree(L.lut[c]); }
        cudaFree(L.x); cudaFree(L.y);
    }
    return 0;
}
