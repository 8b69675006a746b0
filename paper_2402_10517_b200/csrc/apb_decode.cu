// apb_decode.cu -- fused glue of a decoder block around the quantized GEMVs
// (decode step of BASELINE config C5; not part of the reference's hot path,
// which is the GEMV).  One CTA per call: the vectors are one token wide.
//
//   apb_rms_residual : resid(f32) += add(f16, optional);  out(f16) = rmsnorm(resid) * w
//   apb_rope_cache   : q_out = rope(q); k_cache[pos] = rope(k); v_cache[pos] = v
//   apb_silu_mul     : out = silu(gate) * up   (f16 in / out, f32 math)
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/anyprec_b200.h"

namespace {

__device__ __forceinline__ float block_sum(float v, float* sh) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.f;
    if (w == 0)
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;  // valid in warp 0
}

__global__ void __launch_bounds__(1024) rms_residual_kernel(float* resid, const __half* add, const __half* w,
                                                            __half* out, int n, float eps) {
    __shared__ float sh[32];
    __shared__ float scale;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float ss = 0.f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        float r = resid[i];
        if (add) {
            r += __half2float(add[i]);
            resid[i] = r;
        }
        ss += r * r;
    }
    ss = block_sum(ss, sh);
    if (threadIdx.x == 0) scale = rsqrtf(ss / n + eps);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = __float2half(resid[i] * scale * __half2float(w[i]));
}

__global__ void __launch_bounds__(1024) rope_cache_kernel(const __half* q, const __half* k, const __half* v,
                                                          const float* cosv, const float* sinv, __half* q_out,
                                                          __half* k_cache, __half* v_cache, int heads, int hd,
                                                          int64_t cache_head_stride) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int h2 = hd / 2;
    for (int i = threadIdx.x; i < heads * h2; i += blockDim.x) {
        const int h = i / h2, j = i - h * h2;
        const float c = cosv[j], s = sinv[j];
        const float qa = __half2float(q[h * hd + j]), qb = __half2float(q[h * hd + j + h2]);
        const float ka = __half2float(k[h * hd + j]), kb = __half2float(k[h * hd + j + h2]);
        q_out[h * hd + j] = __float2half(qa * c - qb * s);
        q_out[h * hd + j + h2] = __float2half(qb * c + qa * s);
        __half* kc = k_cache + h * cache_head_stride;
        __half* vc = v_cache + h * cache_head_stride;
        kc[j] = __float2half(ka * c - kb * s);
        kc[j + h2] = __float2half(kb * c + ka * s);
        vc[j] = v[h * hd + j];
        vc[j + h2] = v[h * hd + j + h2];
    }
}

__global__ void __launch_bounds__(1024) silu_mul_kernel(const __half* gate, const __half* up, __half* out, int n) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const float g = __half2float(gate[i]);
        out[i] = __float2half(g / (1.f + __expf(-g)) * __half2float(up[i]));
    }
}

int finish() { return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA; }

}  // namespace

extern "C" int apb_rms_residual(float* resid, const uint16_t* add, const uint16_t* w, uint16_t* out, int64_t n,
                                float eps, void* stream) {
    if (n <= 0 || !resid || !w || !out) return APB_ERR_PARAM;
    rms_residual_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(resid, (const __half*)add, (const __half*)w,
                                                              (__half*)out, (int)n, eps);
    return finish();
}

extern "C" int apb_rope_cache(const uint16_t* q, const uint16_t* k, const uint16_t* v, const float* cosv,
                              const float* sinv, uint16_t* q_out, uint16_t* k_cache, uint16_t* v_cache,
                              int heads, int head_dim, int64_t cache_head_stride, void* stream) {
    if (heads <= 0 || head_dim <= 0 || (head_dim & 1)) return APB_ERR_PARAM;
    rope_cache_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
        (const __half*)q, (const __half*)k, (const __half*)v, cosv, sinv, (__half*)q_out, (__half*)k_cache,
        (__half*)v_cache, heads, head_dim, cache_head_stride);
    return finish();
}

extern "C" int apb_silu_mul(const uint16_t* gate, const uint16_t* up, uint16_t* out, int64_t n, void* stream) {
    if (n <= 0) return APB_ERR_PARAM;
    silu_mul_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>((const __half*)gate, (const __half*)up, (__half*)out,
                                                          (int)n);
    return finish();
}
