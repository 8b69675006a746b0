// apb_dense.cu -- activation split for the dense (M > dense_threshold) path of
// engine.gemm (reference engine.py:343-354: dequantize + fp32 GEMM).  The
// dequantised weights are exact in fp16, so an fp32-accurate product runs on
// the tensor cores as ONE fp16 x fp16 -> fp32 GEMM over [hi; lo], where
// hi = fp16(x * s), lo = fp16(x * s - hi) and s is an exact power of two that
// brings the row's max magnitude into [2^14, 2^15) (no fp16 overflow; x*s - hi
// is exact in fp32, so hi + lo carries ~22 significant bits).  One CTA per row.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/anyprec_b200.h"

namespace {

constexpr int kThreads = 256;

// PAIRS = false: hi rows [0, m), lo rows [m, 2m) (dense GEMM operand).
// PAIRS = true : rows (2r, 2r+1) = (hi, lo), columns cols..ld-1 zeroed (the
//                quantized GEMV's x_split = 2 operand, see apb_split_x_scaled).
template <bool PAIRS>
__global__ void __launch_bounds__(kThreads) split_hilo_kernel(const float* __restrict__ x, int cols, int64_t ldx,
                                                              __half* __restrict__ out, int64_t ld, int m,
                                                              float* __restrict__ inv_scale) {
    __shared__ float red[kThreads / 32];
    const int row = blockIdx.x, t = threadIdx.x;
    const float* xr = x + (int64_t)row * ldx;
    float a = 0.f;
    for (int i = t; i < cols; i += kThreads) a = fmaxf(a, fabsf(xr[i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if ((t & 31) == 0) red[t >> 5] = a;
    __syncthreads();
    a = red[0];
#pragma unroll
    for (int w = 1; w < kThreads / 32; ++w) a = fmaxf(a, red[w]);
    float scale = 1.f;
    if (a > 0.f && isfinite(a)) {
        int e;
        frexpf(a, &e);                          // a = f * 2^e, f in [0.5, 1): floor(log2 a) = e - 1
        const int se = min(max(15 - e, -126), 126);
        scale = ldexpf(1.f, se);                // a * scale in [2^14, 2^15)
    }
    __half* hi = out + (int64_t)(PAIRS ? 2 * row : row) * ld;
    __half* lo = out + (int64_t)(PAIRS ? 2 * row + 1 : m + row) * ld;
    for (int i = t; i < (PAIRS ? (int)ld : cols); i += kThreads) {
        const float v = i < cols ? xr[i] * scale : 0.f;  // exact (power of two)
        const __half h = __float2half_rn(v);
        hi[i] = h;
        lo[i] = __float2half_rn(v - __half2float(h));
    }
    if (t == 0) inv_scale[row] = 1.f / scale;   // exact
}

}  // namespace

extern "C" int apb_split_hilo(const float* x, int64_t m, int64_t cols, int64_t ldx, uint16_t* out, int64_t ld,
                              float* inv_scale, void* stream) {
    if (!x || !out || !inv_scale) return APB_ERR_PARAM;
    if (m <= 0 || cols <= 0 || m > INT32_MAX || cols > INT32_MAX || ldx < cols || ld < cols) return APB_ERR_SHAPE;
    split_hilo_kernel<false><<<(unsigned)m, kThreads, 0, (cudaStream_t)stream>>>(x, (int)cols, ldx, (__half*)out,
                                                                                 ld, (int)m, inv_scale);
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

// Quantized-path operand of x_split = 2 (engine.py:270-281 _prep_x for fp32
// activations at fp32 accuracy): out [2m][ldx_out] (hi, lo) row pairs of x * s_r,
// then m float inverse scales 1 / s_r at element offset 2m * ldx_out.
extern "C" int apb_split_x_scaled(const float* x, int m, int64_t cols, int64_t ldx_in, uint16_t* out,
                                  int64_t ldx_out, void* stream) {
    if (!x || !out) return APB_ERR_PARAM;
    if (m <= 0 || cols <= 0 || cols > INT32_MAX || ldx_in < cols || ldx_out < cols || (ldx_out & 1))
        return APB_ERR_SHAPE;
    float* inv = reinterpret_cast<float*>(out + (int64_t)2 * m * ldx_out);
    split_hilo_kernel<true><<<(unsigned)m, kThreads, 0, (cudaStream_t)stream>>>(x, (int)cols, ldx_in, (__half*)out,
                                                                                ldx_out, m, inv);
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}
