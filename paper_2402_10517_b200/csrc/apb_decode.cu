// apb_decode.cu -- fused glue of a decoder block around the quantized GEMVs
// (decode step of BASELINE config C5; not part of the reference's hot path,
// which is the GEMV).  One CTA per call: the vectors are one token wide.
//
//   apb_rms_residual : resid(f32) += add(f16, optional);  out(f16) = rmsnorm(resid) * w
//   apb_rope_cache   : q_out = rope(q); k_cache[pos] = rope(k); v_cache[pos] = v
//   apb_silu_mul     : out = silu(gate) * up   (f16 in / out, f32 math)
//   apb_attention_decode : RoPE(q, k) + KV-cache append + single-query
//                      attention over the cache, split over key chunks (below)
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

// All three: launched with programmatic stream serialisation; they let the next
// kernel (a GEMV, which prefetches its weights and builds its tables before its
// own griddepcontrol.wait) launch at once, and wait for the previous kernel
// before touching its outputs.
// vec (n % 4 == 0, n <= 4 * 4 * 1024, aligned buffers): one vectorised round trip, values kept in
// registers between the sum of squares and the scaled store.
constexpr int kRmsVec = 4;
__global__ void __launch_bounds__(1024) rms_residual_kernel(float* __restrict__ resid, const __half* __restrict__ add,
                                                            const __half* __restrict__ w, __half* __restrict__ out,
                                                            int n, float eps, int vec) {
    __shared__ float sh[32];
    __shared__ float scale;
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float ss = 0.f;
    if (vec) {
        float4 r[kRmsVec];
        const int n4 = n >> 2;
#pragma unroll
        for (int c = 0; c < kRmsVec; ++c) {
            const int i = threadIdx.x + c * blockDim.x;
            if (i < n4) {
                r[c] = reinterpret_cast<const float4*>(resid)[i];
                if (add) {
                    const uint2 a = reinterpret_cast<const uint2*>(add)[i];
                    const float2 a0 = __half22float2(*reinterpret_cast<const __half2*>(&a.x));
                    const float2 a1 = __half22float2(*reinterpret_cast<const __half2*>(&a.y));
                    r[c].x += a0.x;
                    r[c].y += a0.y;
                    r[c].z += a1.x;
                    r[c].w += a1.y;
                    reinterpret_cast<float4*>(resid)[i] = r[c];
                }
                ss += r[c].x * r[c].x + r[c].y * r[c].y + r[c].z * r[c].z + r[c].w * r[c].w;
            }
        }
        ss = block_sum(ss, sh);
        if (threadIdx.x == 0) scale = rsqrtf(ss / n + eps);
        __syncthreads();
        const float sc = scale;
#pragma unroll
        for (int c = 0; c < kRmsVec; ++c) {
            const int i = threadIdx.x + c * blockDim.x;
            if (i < n4) {
                const uint2 wv = reinterpret_cast<const uint2*>(w)[i];
                const float2 w0 = __half22float2(*reinterpret_cast<const __half2*>(&wv.x));
                const float2 w1 = __half22float2(*reinterpret_cast<const __half2*>(&wv.y));
                __half2 o0 = __floats2half2_rn(r[c].x * sc * w0.x, r[c].y * sc * w0.y);
                __half2 o1 = __floats2half2_rn(r[c].z * sc * w1.x, r[c].w * sc * w1.y);
                uint2 ov;
                ov.x = *reinterpret_cast<uint32_t*>(&o0);
                ov.y = *reinterpret_cast<uint32_t*>(&o1);
                reinterpret_cast<uint2*>(out)[i] = ov;
            }
        }
        return;
    }
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
    asm volatile("griddepcontrol.launch_dependents;");
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

constexpr int kSiluThreads = 256;
__global__ void __launch_bounds__(kSiluThreads) silu_mul_kernel(const __half* __restrict__ gate,
                                                                const __half* __restrict__ up,
                                                                __half* __restrict__ out, int n) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // 2 elements per thread
    if (2 * i + 1 < n) {
        const float2 g = __half22float2(reinterpret_cast<const __half2*>(gate)[i]);
        const float2 u = __half22float2(reinterpret_cast<const __half2*>(up)[i]);
        reinterpret_cast<__half2*>(out)[i] =
            __floats2half2_rn(g.x / (1.f + __expf(-g.x)) * u.x, g.y / (1.f + __expf(-g.y)) * u.y);
    } else if (2 * i < n) {
        const float g = __half2float(gate[2 * i]);
        out[2 * i] = __float2half(g / (1.f + __expf(-g)) * __half2float(up[2 * i]));
    }
}

// ---- single-query attention (flash-decoding split over 64-key chunks) -------
// grid (chunks, heads), 128 threads.  K/V rows older than `pos` are loaded
// into registers BEFORE griddepcontrol.wait (they were written by earlier
// steps), so the KV stream overlaps the tail of the qkv GEMV; after the wait the
// CTA rotates q (and, in the chunk holding `pos`, the new k, writing k/v to the
// cache), scores its 64 keys (half-warp per key, 16-byte row slices), and writes
// (max, sum, unnormalised out[128]) to the workspace.  The last CTA of a head
// (atomic ticket) merges the chunks and writes out[h] in fp16 -- straight into
// the o-projection's activation buffer.  Scores are kept in the log2 domain.
constexpr int kAttnHd = 128, kAttnChunk = 64, kAttnThreads = 128;
constexpr int kAttnMaxChunks = 8 * kAttnHd / 2;  // merge staging fits the reduction buffer: 32K keys

__device__ __forceinline__ uint4 ld16(const __half* p) { return *reinterpret_cast<const uint4*>(p); }

__device__ __forceinline__ void h8_to_f(const uint4& u, float* f) {
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 t = __half22float2(h[e]);
        f[2 * e] = t.x;
        f[2 * e + 1] = t.y;
    }
}

__global__ void __launch_bounds__(kAttnThreads) attention_decode_kernel(
    const __half* q, const __half* k, const __half* v, const float* cosv, const float* sinv, __half* k_cache,
    __half* v_cache, int64_t head_stride, int pos, float scale_log2, float* ws, int* tickets, __half* out,
    const __half* next_k, const __half* next_v) {
    __shared__ float qs[kAttnHd];
    __shared__ __align__(16) __half knew[kAttnHd], vnew[kAttnHd];
    __shared__ float sc[kAttnChunk];
    __shared__ float red[8][kAttnHd];
    __shared__ float m_sh, l_sh;
    __shared__ int last;
    asm volatile("griddepcontrol.launch_dependents;");
    const int h = blockIdx.y, chunk = blockIdx.x, chunks = gridDim.x, base = chunk * kAttnChunk;
    const int t = threadIdx.x, w = t >> 5, l = t & 31, hl = l & 15, kk = l >> 4;
    const int vg = t & 15, kg = t >> 4;
    __half* kc = k_cache + h * head_stride;
    __half* vc = v_cache + h * head_stride;
    const bool has_new = pos >= base && pos < base + kAttnChunk;
    if (next_k && t == 0) {
        // the same slice of the next block's cache -> L2, read by its attention
        // after ~4 weight-streaming GEMVs (whose plane loads are evict-first)
        const int nk = min(kAttnChunk, pos + 1 - base);
        const uint32_t bytes = (uint32_t)nk * kAttnHd * 2;
        const int64_t off = h * head_stride + (int64_t)base * kAttnHd;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(next_k + off), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(next_v + off), "r"(bytes) : "memory");
    }
    // score phase: warp w, step i -> key base + 16w + 2i + kk, dims 8hl..8hl+7
    // value phase: thread t -> keys base + 8kg + i, dims 8vg..8vg+7
    uint4 kr[8], vr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int kkey = base + 16 * w + 2 * i + kk, vkey = base + 8 * kg + i;
        kr[i] = kkey < pos ? ld16(kc + (int64_t)kkey * kAttnHd + 8 * hl) : make_uint4(0, 0, 0, 0);
        vr[i] = vkey < pos ? ld16(vc + (int64_t)vkey * kAttnHd + 8 * vg) : make_uint4(0, 0, 0, 0);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (t < kAttnHd / 2) {
        const int j = t;
        const float c = cosv[j], sn = sinv[j];
        const float qa = __half2float(q[h * kAttnHd + j]), qb = __half2float(q[h * kAttnHd + j + 64]);
        qs[j] = (qa * c - qb * sn) * scale_log2;
        qs[j + 64] = (qb * c + qa * sn) * scale_log2;
        if (has_new) {
            const float ka = __half2float(k[h * kAttnHd + j]), kb = __half2float(k[h * kAttnHd + j + 64]);
            const __half ra = __float2half(ka * c - kb * sn), rb = __float2half(kb * c + ka * sn);
            knew[j] = ra;
            knew[j + 64] = rb;
            kc[(int64_t)pos * kAttnHd + j] = ra;
            kc[(int64_t)pos * kAttnHd + j + 64] = rb;
            const __half va = v[h * kAttnHd + j], vb = v[h * kAttnHd + j + 64];
            vnew[j] = va;
            vnew[j + 64] = vb;
            vc[(int64_t)pos * kAttnHd + j] = va;
            vc[(int64_t)pos * kAttnHd + j + 64] = vb;
        }
    }
    __syncthreads();
    if (has_new) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (base + 16 * w + 2 * i + kk == pos) kr[i] = *reinterpret_cast<const uint4*>(knew + 8 * hl);
            if (base + 8 * kg + i == pos) vr[i] = *reinterpret_cast<const uint4*>(vnew + 8 * vg);
        }
    }
    float qf[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) qf[e] = qs[8 * hl + e];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float kf[8];
        h8_to_f(kr[i], kf);
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) d = fmaf(qf[e], kf[e], d);
#pragma unroll
        for (int o = 8; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        const int key = base + 16 * w + 2 * i + kk;
        if (hl == 0) sc[16 * w + 2 * i + kk] = key <= pos ? d : -INFINITY;
    }
    __syncthreads();
    // chunk max (every warp, redundantly) and sum (warp 0)
    float m = fmaxf(sc[l], sc[l + 32]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (w == 0) {
        float ls = exp2f(sc[l] - m) + exp2f(sc[l + 32] - m);
#pragma unroll
        for (int o = 16; o; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
        if (l == 0) {
            m_sh = m;
            l_sh = ls;
        }
    }
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float p = exp2f(sc[8 * kg + i] - m);
        float vf[8];
        h8_to_f(vr[i], vf);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = fmaf(p, vf[e], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) red[kg][8 * vg + e] = acc[e];
    __syncthreads();
    float o = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) o += red[g][t];
    float* wso = ws + ((int64_t)h * chunks + chunk) * (kAttnHd + 2);
    wso[t] = o;
    if (t == 0) {
        wso[kAttnHd] = m_sh;
        wso[kAttnHd + 1] = l_sh;
    }
    __threadfence();
    __syncthreads();
    if (t == 0) last = atomicAdd(&tickets[h], 1) == chunks - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // merge: (max, sum) of every chunk staged in shared memory in parallel, then
    // each thread sums its dim over the chunks with 8 loads in flight
    const float* wsh = ws + (int64_t)h * chunks * (kAttnHd + 2);
    float* cm = &red[0][0];                      // reuse: kAttnMaxChunks maxima
    float* cl = &red[0][0] + kAttnMaxChunks;     // and sums
    for (int c = t; c < chunks; c += kAttnThreads) {
        cm[c] = __ldcg(wsh + c * (kAttnHd + 2) + kAttnHd);
        cl[c] = __ldcg(wsh + c * (kAttnHd + 2) + kAttnHd + 1);
    }
    __syncthreads();
    float M = -INFINITY;
    for (int c = 0; c < chunks; ++c) M = fmaxf(M, cm[c]);
    float L = 0.f, O = 0.f;
    int c = 0;
    for (; c + 8 <= chunks; c += 8) {
        float ov[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) ov[u] = __ldcg(wsh + (c + u) * (kAttnHd + 2) + t);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float f = exp2f(cm[c + u] - M);
            L = fmaf(f, cl[c + u], L);
            O = fmaf(f, ov[u], O);
        }
    }
    for (; c < chunks; ++c) {
        const float f = exp2f(cm[c] - M);
        L = fmaf(f, cl[c], L);
        O = fmaf(f, __ldcg(wsh + c * (kAttnHd + 2) + t), O);
    }
    out[h * kAttnHd + t] = __float2half(O / L);
    if (t == 0) tickets[h] = 0;
}

int finish() { return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA; }

template <typename... KArgs, typename... Args>
int launch_pdl_grid(dim3 grid, dim3 block, void (*kern)(KArgs...), cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, args...) != cudaSuccess) return APB_ERR_CUDA;
    return finish();
}

template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), cudaStream_t s, Args... args) {
    return launch_pdl_grid(dim3(1), dim3(1024), kern, s, args...);
}

}  // namespace

extern "C" int apb_rms_residual(float* resid, const uint16_t* add, const uint16_t* w, uint16_t* out, int64_t n,
                                float eps, void* stream) {
    if (n <= 0 || n > INT32_MAX || !resid || !w || !out) return APB_ERR_PARAM;
    const bool aligned = !(((uintptr_t)resid & 15) | ((uintptr_t)add & 7) | ((uintptr_t)w & 7) | ((uintptr_t)out & 7));
    const int vec = aligned && (n & 3) == 0 && n <= kRmsVec * 4 * 1024;
    return launch_pdl(rms_residual_kernel, (cudaStream_t)stream, resid, (const __half*)add, (const __half*)w,
                      (__half*)out, (int)n, eps, vec);
}

extern "C" int apb_rope_cache(const uint16_t* q, const uint16_t* k, const uint16_t* v, const float* cosv,
                              const float* sinv, uint16_t* q_out, uint16_t* k_cache, uint16_t* v_cache,
                              int heads, int head_dim, int64_t cache_head_stride, void* stream) {
    if (heads <= 0 || head_dim <= 0 || (head_dim & 1)) return APB_ERR_PARAM;
    return launch_pdl(rope_cache_kernel, (cudaStream_t)stream, (const __half*)q, (const __half*)k, (const __half*)v,
                      cosv, sinv, (__half*)q_out, (__half*)k_cache, (__half*)v_cache, heads, head_dim,
                      cache_head_stride);
}

extern "C" int apb_silu_mul(const uint16_t* gate, const uint16_t* up, uint16_t* out, int64_t n, void* stream) {
    if (n <= 0 || n > INT32_MAX || (((uintptr_t)gate | (uintptr_t)up | (uintptr_t)out) & 3)) return APB_ERR_PARAM;
    const int blocks = (int)((n + 2 * kSiluThreads - 1) / (2 * kSiluThreads));
    return launch_pdl_grid(dim3(blocks), dim3(kSiluThreads), silu_mul_kernel, (cudaStream_t)stream,
                           (const __half*)gate, (const __half*)up, (__half*)out, (int)n);
}

extern "C" int64_t apb_attention_decode_workspace(int heads, int head_dim, int64_t max_keys) {
    if (heads <= 0 || head_dim != kAttnHd || max_keys <= 0) return -1;
    const int64_t chunks = (max_keys + kAttnChunk - 1) / kAttnChunk;
    return (int64_t)heads * chunks * (kAttnHd + 2) * 4 + (int64_t)heads * 4;
}

extern "C" int apb_attention_decode(const uint16_t* q, const uint16_t* k, const uint16_t* v, const float* cosv,
                                    const float* sinv, uint16_t* k_cache, uint16_t* v_cache, int heads,
                                    int head_dim, int64_t cache_head_stride, int pos, float scale, void* workspace,
                                    int64_t workspace_bytes, uint16_t* out, const uint16_t* next_k_cache,
                                    const uint16_t* next_v_cache, void* stream) {
    if (!q || !k || !v || !cosv || !sinv || !k_cache || !v_cache || !workspace || !out) return APB_ERR_PARAM;
    if (!next_k_cache != !next_v_cache || (((uintptr_t)next_k_cache | (uintptr_t)next_v_cache) & 15) ||
        (cache_head_stride & 7))
        return APB_ERR_PARAM;
    if (heads <= 0 || head_dim != kAttnHd || pos < 0 || pos >= kAttnMaxChunks * kAttnChunk ||
        cache_head_stride < (int64_t)(pos + 1) * head_dim)
        return APB_ERR_PARAM;
    const int64_t need = apb_attention_decode_workspace(heads, head_dim, (int64_t)pos + 1);
    if (workspace_bytes < need) return APB_ERR_PARAM;
    const int chunks = (pos + 1 + kAttnChunk - 1) / kAttnChunk;
    float* ws = (float*)workspace;
    // tickets live at the END of the workspace so any chunk count below the
    // allocation's maximum finds them at the same place
    int* tickets = (int*)((char*)workspace + workspace_bytes) - heads;
    if ((uintptr_t)tickets & 3) return APB_ERR_PARAM;
    const float scale_log2 = scale * 1.4426950408889634f;
    return launch_pdl_grid(dim3(chunks, heads), dim3(kAttnThreads), attention_decode_kernel, (cudaStream_t)stream,
                           (const __half*)q, (const __half*)k, (const __half*)v, cosv, sinv, (__half*)k_cache,
                           (__half*)v_cache, cache_head_stride, pos, scale_log2, ws, tickets, (__half*)out,
                           (const __half*)next_k_cache, (const __half*)next_v_cache);
}

// ---- decode-step ends: embedding row -> residual + first RMSNorm; argmax ----
namespace {

__global__ void __launch_bounds__(1024) embed_rms_kernel(const __half* __restrict__ embed,
                                                         const int64_t* __restrict__ token, int n,
                                                         float* __restrict__ resid, const __half* __restrict__ w,
                                                         __half* __restrict__ out, float eps) {
    __shared__ float sh[32];
    __shared__ float scale;
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const __half* row = embed + token[0] * (int64_t)n;
    float ss = 0.f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const float r = __half2float(row[i]);
        resid[i] = r;
        ss += r * r;
    }
    ss = block_sum(ss, sh);
    if (threadIdx.x == 0) scale = rsqrtf(ss / n + eps);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        out[i] = __float2half(__half2float(row[i]) * scale * __half2float(w[i]));
}

// index of the largest value (first one on ties; NaN never wins)
__global__ void __launch_bounds__(1024) argmax_kernel(const __half* __restrict__ x, int n, int64_t* __restrict__ out) {
    __shared__ float sv[32];
    __shared__ int si[32];
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float bv = -INFINITY;
    int bi = INT32_MAX;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const float v = __half2float(x[i]);
        if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float v = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i = __shfl_xor_sync(0xffffffffu, bi, o);
        if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sv[w] = bv;
        si[w] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int j = 1; j < (int)(blockDim.x >> 5); ++j)
            if (sv[j] > bv || (sv[j] == bv && si[j] < bi)) {
                bv = sv[j];
                bi = si[j];
            }
        out[0] = bi == INT32_MAX ? 0 : bi;
    }
}

}  // namespace

extern "C" int apb_embed_rms(const uint16_t* embed, const int64_t* token, int64_t n, float* resid,
                             const uint16_t* w, uint16_t* out, float eps, void* stream) {
    if (!embed || !token || !resid || !w || !out || n <= 0 || n > INT32_MAX) return APB_ERR_PARAM;
    return launch_pdl(embed_rms_kernel, (cudaStream_t)stream, (const __half*)embed, token, (int)n, resid,
                      (const __half*)w, (__half*)out, eps);
}

extern "C" int apb_argmax_f16(const uint16_t* x, int64_t n, int64_t* out, void* stream) {
    if (!x || !out || n <= 0 || n > INT32_MAX) return APB_ERR_PARAM;
    return launch_pdl(argmax_kernel, (cudaStream_t)stream, (const __half*)x, (int)n, out);
}
