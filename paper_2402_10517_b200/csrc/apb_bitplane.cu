// apb_bitplane.cu -- layout kernels: packer, permutation, prefix unpack,
// SWAR word transpose, dequantisation and the activation split helper.
//
// Work unit for pack / unpack / dequant: one thread per (row, tile, lane t)
// -- one 32-bit lane word per plane, 32 weights.  A warp covers one
// 128-byte tile-plane row, so every plane access is a coalesced 128 B line in
// the permuted layout, and code/weight rows are read/written as 4 runs of
// 8 contiguous bytes (256 B apart) per thread, i.e. 256 contiguous bytes per
// warp per run.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/anyprec_b200.h"
#include "apb_common.cuh"

namespace apb {

struct TileGeom {
    int64_t rows, cols, row_bytes, plane_stride, n_tiles;
};

__device__ __forceinline__ bool decode_thread(const TileGeom& g, int64_t& row, int64_t& tile,
                                              int& t) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    t = (int)(gid & 31);
    const int64_t rt = gid >> 5;
    row = rt / g.n_tiles;
    tile = rt - row * g.n_tiles;
    return row < g.rows;
}

// Load 8 consecutive bytes (columns col..col+7 of a code row), zero beyond cols.
__device__ __forceinline__ uint2 load_codes8(const uint8_t* rowp, int64_t col, int64_t cols,
                                             bool vec_ok) {
    if (vec_ok && col + 8 <= cols) return *reinterpret_cast<const uint2*>(rowp + col);
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t v = (col + i < cols) ? (uint32_t)rowp[col + i] : 0u;
        if (i < 4) lo |= v << (8 * i);
        else hi |= v << (8 * (i - 4));
    }
    return make_uint2(lo, hi);
}

// ---------------------------------------------------------------------------
// pack_bitplanes (+ permute_layout): bitplane.py:76-100, 121-130.
// W[o] byte p = code of column 256p + 8t + o; the byte->plane transpose is
// to_bytes<8> applied to W (the network is an involution up to role swap).
template <int NMAX, bool PERMUTED>
__global__ void __launch_bounds__(256) pack_kernel(const uint8_t* __restrict__ codes, int64_t ld,
                                                   bool vec_ok, TileGeom g,
                                                   uint8_t* __restrict__ planes,
                                                   uint32_t* code_or) {
    int64_t row, tile;
    int t;
    const bool live = decode_thread(g, row, tile, t);
    uint32_t orv = 0;
    if (live) {
        const uint8_t* rowp = codes + row * ld;
        uint32_t lo[4], hi[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const uint2 v = load_codes8(rowp, tile * kTileWeights + 256 * p + 8 * t, g.cols, vec_ok);
            lo[p] = v.x;
            hi[p] = v.y;
            orv |= v.x | v.y;
        }
        uint32_t W[8];
        byte_transpose4(lo, W);
        byte_transpose4(hi, W + 4);
        uint32_t Q[8];
        to_bytes<8>(W, Q);  // Q[b] bit (8p + i) = code bit b of column 256p + 8t + i
#pragma unroll
        for (int p = 0; p < NMAX; ++p) {
            const uint32_t word = Q[NMAX - 1 - p];  // plane p holds code bit NMAX-1-p
            uint8_t* dst = planes + p * g.plane_stride + row * g.row_bytes + tile * kTileBytes;
            if (PERMUTED) {
                reinterpret_cast<uint32_t*>(dst)[t] = word;
            } else {
                // linear byte 32j + t holds columns 256j + 8t .. +7
#pragma unroll
                for (int j = 0; j < 4; ++j) dst[32 * j + t] = (uint8_t)(word >> (8 * j));
            }
        }
    }
    if (code_or != nullptr) {
        orv |= (orv >> 16);
        orv |= (orv >> 8);
        orv &= 0xFFu;
        orv = __reduce_or_sync(0xFFFFFFFFu, orv);
        // only bits not yet recorded go to the (single, shared) word: after the
        // first few warps every code bit is usually set and no atomic is issued
        // (one atomicOr per warp serialised ~230K atomics on one address for a
        // 28672x8192 matrix)
        if ((threadIdx.x & 31) == 0 && (orv & ~__ldcg(code_or))) atomicOr(code_or, orv);
    }
}

// ---------------------------------------------------------------------------
// permute_layout / inverse_permute_layout: bitplane.py:121-136.
// One thread per output (or input) lane word t of a tile row: permuted word t
// is linear bytes {32j + t : j = 0..3}.
__global__ void __launch_bounds__(256) permute_kernel(const uint8_t* __restrict__ in,
                                                      uint8_t* __restrict__ out, int64_t n_words,
                                                      int inverse) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n_words) return;
    const int t = (int)(gid & 31);
    const int64_t base = (gid >> 5) * kTileBytes;
    if (!inverse) {
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) w |= (uint32_t)in[base + 32 * j + t] << (8 * j);
        reinterpret_cast<uint32_t*>(out + base)[t] = w;
    } else {
        const uint32_t w = reinterpret_cast<const uint32_t*>(in + base)[t];
#pragma unroll
        for (int j = 0; j < 4; ++j) out[base + 32 * j + t] = (uint8_t)(w >> (8 * j));
    }
}

// Load the k lane words (MSB plane first in memory) as Q[i] = plane k-1-i.
template <int K, bool PERMUTED>
__device__ __forceinline__ void load_lane_words(const uint8_t* __restrict__ planes, const TileGeom& g,
                                                int64_t row, int64_t tile, int t, uint32_t* Q) {
#pragma unroll
    for (int p = 0; p < K; ++p) {
        const uint8_t* src = planes + p * g.plane_stride + row * g.row_bytes + tile * kTileBytes;
        uint32_t w;
        if (PERMUTED) {
            w = ldg_stream4(src + 4 * t);
        } else {
            w = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) w |= (uint32_t)src[32 * j + t] << (8 * j);
        }
        Q[K - 1 - p] = w;
    }
}

// ---------------------------------------------------------------------------
// unpack_codes: bitplane.py:103-118.  Reads planes[0..K-1] only.
template <int K, bool PERMUTED>
__global__ void __launch_bounds__(256) unpack_kernel(const uint8_t* __restrict__ planes, TileGeom g,
                                                     uint8_t* __restrict__ codes, int64_t ld,
                                                     bool vec_ok) {
    int64_t row, tile;
    int t;
    if (!decode_thread(g, row, tile, t)) return;
    uint32_t Q[8];
    load_lane_words<K, PERMUTED>(planes, g, row, tile, t, Q);
    uint32_t W[8];
    to_bytes<K>(Q, W);  // W[b] byte p = code of column 256p + 8t + b
    uint32_t lo[4], hi[4];
    byte_transpose4(W, lo);  // lo[p] byte b = code of column 256p + 8t + b, b < 4
    byte_transpose4(W + 4, hi);
    uint8_t* rowp = codes + row * ld;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int64_t col = tile * kTileWeights + 256 * p + 8 * t;
        if (col >= g.cols) continue;
        if (vec_ok && col + 8 <= g.cols) {
            *reinterpret_cast<uint2*>(rowp + col) = make_uint2(lo[p], hi[p]);
        } else {
            for (int i = 0; i < 8 && col + i < g.cols; ++i)
                rowp[col + i] = (uint8_t)((i < 4 ? lo[p] >> (8 * i) : hi[p] >> (8 * (i - 4))) & 0xFFu);
        }
    }
}

// ---------------------------------------------------------------------------
// dequantize: engine.py:357-362 (= take_along_axis(table_k, codes_at(k))).
template <int K, bool PERMUTED, bool F16OUT>
__global__ void __launch_bounds__(256) dequant_kernel(const uint8_t* __restrict__ planes, TileGeom g,
                                                      const uint16_t* __restrict__ lut,
                                                      void* __restrict__ w, int64_t ldw) {
    int64_t row, tile;
    int t;
    if (!decode_thread(g, row, tile, t)) return;
    uint32_t Q[8];
    load_lane_words<K, PERMUTED>(planes, g, row, tile, t, Q);
    uint32_t W[8];
    to_bytes<K>(Q, W);
    const uint16_t* lrow = lut + row * (1 << K);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int64_t col = tile * kTileWeights + 256 * p + 8 * t;
        if (col >= g.cols) continue;
        uint16_t v[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) v[b] = __ldg(lrow + ((W[b] >> (8 * p)) & 0xFFu));
        const bool full = col + 8 <= g.cols && (ldw % 8) == 0;
        if (F16OUT) {
            uint16_t* dst = reinterpret_cast<uint16_t*>(w) + row * ldw + col;
            if (full) {
                uint4 o;
                o.x = v[0] | ((uint32_t)v[1] << 16);
                o.y = v[2] | ((uint32_t)v[3] << 16);
                o.z = v[4] | ((uint32_t)v[5] << 16);
                o.w = v[6] | ((uint32_t)v[7] << 16);
                *reinterpret_cast<uint4*>(dst) = o;
            } else {
                for (int b = 0; b < 8 && col + b < g.cols; ++b) dst[b] = v[b];
            }
        } else {
            float* dst = reinterpret_cast<float*>(w) + row * ldw + col;
            float f[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) f[b] = __half2float(__ushort_as_half(v[b]));
            if (full) {
                reinterpret_cast<float4*>(dst)[0] = make_float4(f[0], f[1], f[2], f[3]);
                reinterpret_cast<float4*>(dst)[1] = make_float4(f[4], f[5], f[6], f[7]);
            } else {
                for (int b = 0; b < 8 && col + b < g.cols; ++b) dst[b] = f[b];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// transpose_any_width: engine.py:48-92 restated literally (masked delta swaps,
// LSB plane first, zero-extended to B words).
template <int K>
__global__ void __launch_bounds__(256) transpose_words_kernel(const uint32_t* __restrict__ pw,
                                                              int64_t n, uint32_t* __restrict__ out) {
    constexpr int B = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t w[B];
#pragma unroll
    for (int b = 0; b < B; ++b) w[b] = b < K ? pw[(int64_t)(K - 1 - b) * n + i] : 0u;
#pragma unroll
    for (int d = 1; d < B; d <<= 1) {
        const uint32_t mask = d == 1 ? 0x55555555u : (d == 2 ? 0x33333333u : 0x0F0F0F0Fu);
#pragma unroll
        for (int r = 0; r < B; ++r) {
            if (r & d) continue;
            const uint32_t tt = ((w[r] >> d) ^ w[r + d]) & mask;
            w[r] ^= tt << d;
            w[r + d] ^= tt;
        }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) out[(int64_t)b * n + i] = w[b];
}

// ---------------------------------------------------------------------------
// fp32 activations -> fp16 (hi, lo) pairs (or fp16 rounding only).
__global__ void __launch_bounds__(256) split_x_kernel(const float* __restrict__ x, int m, int64_t cols,
                                                      int64_t ldx_in, uint16_t* __restrict__ out,
                                                      int64_t ldx_out, int round_only) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)m * ldx_out;
    if (gid >= total) return;
    const int64_t r = gid / ldx_out, c = gid - r * ldx_out;
    const float v = c < cols ? x[r * ldx_in + c] : 0.0f;
    const __half hi = __float2half_rn(v);
    if (round_only) {
        out[r * ldx_out + c] = __half_as_ushort(hi);
    } else {
        const __half lo = __float2half_rn(v - __half2float(hi));
        out[(2 * r) * ldx_out + c] = __half_as_ushort(hi);
        out[(2 * r + 1) * ldx_out + c] = __half_as_ushort(lo);
    }
}

}  // namespace apb

// ===========================================================================
// C ABI
using namespace apb;

static int launch_status() {
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

static TileGeom make_geom(int64_t rows, int64_t cols, int64_t padded) {
    TileGeom g;
    g.rows = rows;
    g.cols = cols;
    g.row_bytes = padded / 8;
    g.plane_stride = rows * (padded / 8);
    g.n_tiles = padded / kTileWeights;
    return g;
}

static unsigned grid_for(int64_t threads) { return (unsigned)((threads + 255) / 256); }

extern "C" int64_t apb_pad_columns(int64_t cols) {
    return ((cols + kTileWeights - 1) / kTileWeights) * kTileWeights;
}

template <bool P>
static void launch_pack(int n_max, unsigned grid, cudaStream_t s, const uint8_t* codes, int64_t ld,
                        bool vec_ok, TileGeom g, uint8_t* planes, uint32_t* code_or) {
    switch (n_max) {
#define APB_PACK_CASE(N) \
    case N: pack_kernel<N, P><<<grid, 256, 0, s>>>(codes, ld, vec_ok, g, planes, code_or); break;
        APB_PACK_CASE(1) APB_PACK_CASE(2) APB_PACK_CASE(3) APB_PACK_CASE(4)
        APB_PACK_CASE(5) APB_PACK_CASE(6) APB_PACK_CASE(7) APB_PACK_CASE(8)
#undef APB_PACK_CASE
    }
}

extern "C" int apb_pack(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ld_codes,
                        int n_max, int permuted, uint8_t* planes, uint32_t* d_code_or,
                        void* stream) {
    if (rows <= 0 || cols <= 0 || ld_codes < cols) return APB_ERR_SHAPE;
    if (n_max < 1 || n_max > 8) return APB_ERR_PARAM;
    if (!codes || !planes) return APB_ERR_PARAM;
    const TileGeom g = make_geom(rows, cols, apb_pad_columns(cols));
    const bool vec_ok = (ld_codes % 8 == 0) && (((uintptr_t)codes & 7) == 0);
    const unsigned grid = grid_for(rows * g.n_tiles * 32);
    cudaStream_t s = (cudaStream_t)stream;
    if (permuted) launch_pack<true>(n_max, grid, s, codes, ld_codes, vec_ok, g, planes, d_code_or);
    else launch_pack<false>(n_max, grid, s, codes, ld_codes, vec_ok, g, planes, d_code_or);
    return launch_status();
}

extern "C" int apb_permute(const uint8_t* in, uint8_t* out, int n_planes, int64_t rows,
                           int64_t padded_cols, int inverse, void* stream) {
    if (n_planes < 1 || rows <= 0 || padded_cols <= 0 || padded_cols % kTileWeights) return APB_ERR_SHAPE;
    if (!in || !out || in == out) return APB_ERR_PARAM;
    const int64_t n_words = (int64_t)n_planes * rows * (padded_cols / kTileWeights) * 32;
    permute_kernel<<<grid_for(n_words), 256, 0, (cudaStream_t)stream>>>(in, out, n_words, inverse);
    return launch_status();
}

template <bool P>
static void launch_unpack(int k, unsigned grid, cudaStream_t s, const uint8_t* planes, TileGeom g,
                          uint8_t* codes, int64_t ld, bool vec_ok) {
    switch (k) {
#define APB_UNPACK_CASE(N) \
    case N: unpack_kernel<N, P><<<grid, 256, 0, s>>>(planes, g, codes, ld, vec_ok); break;
        APB_UNPACK_CASE(1) APB_UNPACK_CASE(2) APB_UNPACK_CASE(3) APB_UNPACK_CASE(4)
        APB_UNPACK_CASE(5) APB_UNPACK_CASE(6) APB_UNPACK_CASE(7) APB_UNPACK_CASE(8)
#undef APB_UNPACK_CASE
    }
}

extern "C" int apb_unpack(const uint8_t* planes, int n_max, int64_t rows, int64_t cols,
                          int64_t padded_cols, int permuted, int k, uint8_t* codes,
                          int64_t ld_codes, void* stream) {
    if (rows <= 0 || cols <= 0 || ld_codes < cols) return APB_ERR_SHAPE;
    if (padded_cols != apb_pad_columns(cols)) return APB_ERR_SHAPE;
    if (n_max < 1 || n_max > 8 || k < 1 || k > n_max) return APB_ERR_PARAM;
    const TileGeom g = make_geom(rows, cols, padded_cols);
    const bool vec_ok = (ld_codes % 8 == 0) && (((uintptr_t)codes & 7) == 0);
    const unsigned grid = grid_for(rows * g.n_tiles * 32);
    cudaStream_t s = (cudaStream_t)stream;
    if (permuted) launch_unpack<true>(k, grid, s, planes, g, codes, ld_codes, vec_ok);
    else launch_unpack<false>(k, grid, s, planes, g, codes, ld_codes, vec_ok);
    return launch_status();
}

extern "C" int apb_transpose_words(const uint32_t* plane_words, int k, int64_t n, uint32_t* out,
                                   void* stream) {
    if (k < 2 || k > 8) return APB_ERR_PARAM;
    if (n <= 0) return APB_ERR_SHAPE;
    const unsigned grid = grid_for(n);
    cudaStream_t s = (cudaStream_t)stream;
    switch (k) {
#define APB_TW_CASE(N) \
    case N: transpose_words_kernel<N><<<grid, 256, 0, s>>>(plane_words, n, out); break;
        APB_TW_CASE(2) APB_TW_CASE(3) APB_TW_CASE(4) APB_TW_CASE(5)
        APB_TW_CASE(6) APB_TW_CASE(7) APB_TW_CASE(8)
#undef APB_TW_CASE
    }
    return launch_status();
}

template <bool P, bool H>
static void launch_dequant(int k, unsigned grid, cudaStream_t s, const uint8_t* planes, TileGeom g,
                           const uint16_t* lut, void* w, int64_t ldw) {
    switch (k) {
#define APB_DQ_CASE(N) \
    case N: dequant_kernel<N, P, H><<<grid, 256, 0, s>>>(planes, g, lut, w, ldw); break;
        APB_DQ_CASE(1) APB_DQ_CASE(2) APB_DQ_CASE(3) APB_DQ_CASE(4)
        APB_DQ_CASE(5) APB_DQ_CASE(6) APB_DQ_CASE(7) APB_DQ_CASE(8)
#undef APB_DQ_CASE
    }
}

extern "C" int apb_dequant(const uint8_t* planes, int n_max, int64_t rows, int64_t cols,
                           int64_t padded_cols, int permuted, int k, const uint16_t* lut, void* w,
                           int w_dtype, int64_t ldw, void* stream) {
    if (rows <= 0 || cols <= 0 || ldw < cols) return APB_ERR_SHAPE;
    if (padded_cols != apb_pad_columns(cols)) return APB_ERR_SHAPE;
    if (n_max < 1 || n_max > 8 || k < 1 || k > n_max) return APB_ERR_PARAM;
    if (w_dtype != APB_DTYPE_F32 && w_dtype != APB_DTYPE_F16) return APB_ERR_PARAM;
    const TileGeom g = make_geom(rows, cols, padded_cols);
    const unsigned grid = grid_for(rows * g.n_tiles * 32);
    cudaStream_t s = (cudaStream_t)stream;
    if (permuted) {
        if (w_dtype == APB_DTYPE_F16) launch_dequant<true, true>(k, grid, s, planes, g, lut, w, ldw);
        else launch_dequant<true, false>(k, grid, s, planes, g, lut, w, ldw);
    } else {
        if (w_dtype == APB_DTYPE_F16) launch_dequant<false, true>(k, grid, s, planes, g, lut, w, ldw);
        else launch_dequant<false, false>(k, grid, s, planes, g, lut, w, ldw);
    }
    return launch_status();
}

extern "C" int apb_split_x(const float* x, int m, int64_t cols, int64_t ldx_in, uint16_t* out,
                           int64_t ldx_out, int round_only, void* stream) {
    if (m < 1 || cols <= 0 || ldx_in < cols || ldx_out < cols) return APB_ERR_SHAPE;
    const int64_t total = (int64_t)m * ldx_out;
    split_x_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(x, m, cols, ldx_in, out,
                                                                      ldx_out, round_only);
    return launch_status();
}
