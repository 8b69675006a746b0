// Host-side cost of one GEMV launch through the C ABI: apb_gemv (validate +
// build + encode + launch) vs a prepared plan (apb_gemv_plan_launch).
#include <chrono>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../../include/anyprec_b200.h"
int main() {
    const int64_t R = 4096, C = 4096, Cp = 4096;
    uint8_t* planes; uint16_t* lut; uint16_t* x; float* y;
    cudaMalloc(&planes, 8 * R * Cp / 8); cudaMemset(planes, 0x5a, 8 * R * Cp / 8);
    cudaMalloc(&lut, R * 256 * 2); cudaMemset(lut, 0, R * 256 * 2);
    cudaMalloc(&x, C * 2); cudaMemset(x, 0, C * 2);
    cudaMalloc(&y, R * 4);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto time_it = [&](const char* what, auto fn) {
        for (int i = 0; i < 50; ++i) fn();
        cudaStreamSynchronize(s);
        auto t0 = std::chrono::high_resolution_clock::now();
        for (int i = 0; i < 2000; ++i) fn();
        auto t1 = std::chrono::high_resolution_clock::now();
        cudaStreamSynchronize(s);
        printf("%-40s %.2f us/call (host)\n", what, std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000);
    };
    time_it("apb_gemv", [&] { apb_gemv(planes, 8, R, C, Cp, 3, lut, x, 1, C, 0, y, APB_DTYPE_F32, R, 0, s); });
    const uint8_t* pl[1] = {planes}; int nm[1] = {8}; int64_t rw[1] = {R}, cl[1] = {C}, pd[1] = {Cp};
    const uint16_t* lt[1] = {lut}; const uint16_t* xs[1] = {x}; int64_t lx[1] = {C}; void* ys[1] = {y};
    int64_t ly[1] = {R};
    void* plan = apb_gemv_plan_create(1, pl, nm, rw, cl, pd, 3, lt, xs, 1, lx, 0, ys, APB_DTYPE_F32, ly, 0);
    time_it("apb_gemv_plan_launch", [&] { apb_gemv_plan_launch(plan, nullptr, nullptr, s); });
    time_it("apb_gemv_plan_launch (new x/y)", [&] { apb_gemv_plan_launch(plan, xs, ys, s); });
    apb_gemv_plan_destroy(plan);
    return 0;
}
