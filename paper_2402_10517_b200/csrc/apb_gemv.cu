// apb_gemv.cu -- bitplane any-precision GEMV / small-batch GEMM for sm_100a.
//
// Replaces engine.py:284-309 (gemv) and engine.py:312-341 (gemm, quantized
// path) of the reference.  Same maths: y[m][r] = sum_c LUT_k[r][code_k(r,c)] *
// x[m][c], reading ONLY planes 0..k-1 and the k-bit table.
//
// CTA  = 16 output rows x all K columns; W warps split the K dimension into
//        "units" (one 16- or 8-byte slice of a 128-byte tile-plane row per
//        lane).  Deterministic: every output is reduced in a fixed order
//        (mma k-order, then warps 0..W-1 through shared memory).
// Lane = (g, q) = (lane>>2, lane&3): lane owns rows g and g+8 of the CTA and a
//        fixed set of columns; it loads k plane words per row with 128-bit
//        (or 64-bit) streaming loads (ld.global.nc.L1::no_allocate).
// Decode: bit networks of apb_common.cuh (no per-weight shift/mask):
//        k <= 4: to_pairs -> one PRMT + one LDS per PAIR of weights from a
//                4^k-entry pair table (paper's merged lookup)
//        k >= 5: to_bytes -> one PRMT + one LDS per weight, pairs packed into
//                fp16x2 with one IMAD (FMA pipe).
//        Shared-memory tables are replicated per lane slot ([entry][row-half]
//        [lane]) so every lookup is bank-conflict free (bank == lane), and the
//        PRMT builds the full byte address [lane*4 | row-half*128 | idx<<8]
//        in one instruction; the table base folds into the LDS immediate.
// MAC:   the decoded fp16x2 weights ARE the A fragment of
//        mma.sync.m16n8k16 (rows g, g+8; k-slots 2q.., 2q+8..), the
//        activations are the B fragment (batch columns n = g), accumulation is
//        fp32 in the tensor core.  This offloads the multiply-add (1 HMMA per
//        256 weights instead of 128 FFMA) from the ALU/FMA pipes, which the
//        decode saturates on B200, and makes batch 1..8 (or 1..4 with fp32
//        hi/lo activations) cost the same instructions as batch 1.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/anyprec_b200.h"
#include "apb_common.cuh"

namespace apb {

constexpr int kMaxGroup = 16;
constexpr int kRowsPerCta = 16;

struct GemvProblem {
    const uint8_t* planes;  // permuted planes, plane 0 (MSB) first
    const uint16_t* lut;    // fp16 [rows][1<<K]
    const uint16_t* x;      // fp16 [m_x][ldx]
    void* y;                // [m_out][ldy]
    int64_t rows, cols, row_bytes, plane_stride, ldx, ldy;
    int n_tiles;
    int block_begin;
};

struct GemvLaunch {
    GemvProblem prob[kMaxGroup];
    int n_prob;
    int m_x;
    int x_split;
    int y_f16;
};

template <int UB>
struct UnitVec;
template <>
struct UnitVec<16> {
    using T = uint4;
    static __device__ __forceinline__ T load(const void* p) { return ldg_stream16(p); }
    static __device__ __forceinline__ T zero() { return make_uint4(0, 0, 0, 0); }
    static __device__ __forceinline__ uint32_t word(const T& v, int i) {
        return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
    }
};
template <>
struct UnitVec<8> {
    using T = uint2;
    static __device__ __forceinline__ T load(const void* p) { return ldg_stream8(p); }
    static __device__ __forceinline__ T zero() { return make_uint2(0, 0); }
    static __device__ __forceinline__ uint32_t word(const T& v, int i) { return i == 0 ? v.x : v.y; }
};

__device__ __forceinline__ uint32_t lds32(const uint8_t* base, uint32_t off) {
    return *reinterpret_cast<const uint32_t*>(base + off);
}

__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 8 fp16 activations at columns col..col+7, zero beyond cols (tail tile only).
__device__ __noinline__ uint4 load_x8_tail(const uint16_t* xrow, int64_t col, int64_t cols) {
    if (col + 8 <= cols) return __ldg(reinterpret_cast<const uint4*>(xrow + col));
    uint32_t h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = (col + i < cols) ? (uint32_t)__ldg(xrow + col + i) : 0u;
    return make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16),
                      h[6] | (h[7] << 16));
}

__device__ __forceinline__ uint32_t u4_word(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

template <int K>
struct TableGeom {
    static constexpr bool kPair = K <= 4;
    static constexpr int kEntries = kPair ? (1 << (2 * K)) : (1 << K);
    static constexpr int kBytes = kEntries * 256;  // [entry][row-half 2][lane 32] x u32
};

// Decode one lane word of one row into 16 fp16x2 values:
// out[p*4 + j] = weights of columns (256p + 8t + 2j, +1) of this row.
template <int K>
__device__ __forceinline__ void decode_word(const uint32_t* Q, const uint8_t* table, uint32_t off,
                                            uint32_t* out) {
    if constexpr (TableGeom<K>::kPair) {
        uint32_t U[4];
        to_pairs<K>(Q, U);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p)
                out[p * 4 + j] = lds32(table, prmt(U[j], off, 0x5504u | (uint32_t)(p << 4)));
    } else {
        uint32_t Wb[8];
        to_bytes<K>(Q, Wb);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const uint32_t sel = 0x5504u | (uint32_t)(p << 4);
                const uint32_t e = lds32(table, prmt(Wb[2 * j], off, sel));
                const uint32_t o = lds32(table, prmt(Wb[2 * j + 1], off, sel));
                out[p * 4 + j] = e + (o << 16);  // IMAD: o * 65536 + e (e < 65536)
            }
    }
}

template <int NG>
struct GemvBounds {
    // NG == 1: up to 12 warps (<= 168 registers); wider batches: 8 warps (<= 255).
    static constexpr int kThreads = NG == 1 ? 384 : 256;
};

template <int K, int NG, int UB>
__global__ void __launch_bounds__(GemvBounds<NG>::kThreads) gemv_kernel(const __grid_constant__ GemvLaunch L) {
    using V = UnitVec<UB>;
    using VT = typename V::T;
    constexpr int WPU = UB / 4;             // lane words per unit per row
    constexpr int UPT = 128 / (4 * UB);     // units per tile
    constexpr int TB = TableGeom<K>::kBytes;

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* table = smem;
    uint8_t* scratch = smem + TB;

    int pi = 0;
#pragma unroll 1
    for (int i = 1; i < L.n_prob; ++i)
        if ((int)blockIdx.x >= L.prob[i].block_begin) pi = i;
    // problem fields -> registers once (avoid indexed constant-bank reloads in the loop)
    const uint8_t* const planes = L.prob[pi].planes;
    const uint16_t* const lut = L.prob[pi].lut;
    const uint16_t* const xg = L.prob[pi].x;
    void* const yg = L.prob[pi].y;
    const int64_t rows = L.prob[pi].rows, cols = L.prob[pi].cols;
    const int64_t row_bytes = L.prob[pi].row_bytes, plane_stride = L.prob[pi].plane_stride;
    const int64_t ldx = L.prob[pi].ldx, ldy = L.prob[pi].ldy;
    const int n_tiles = L.prob[pi].n_tiles;
    const int64_t rb = (int64_t)blockIdx.x - L.prob[pi].block_begin;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3;
    const int nwarps = blockDim.x >> 5;
    const int64_t row0 = rb * kRowsPerCta + g, row1 = row0 + 8;
    const bool ok0 = row0 < rows, ok1 = row1 < rows;
    const int n_units = n_tiles * UPT;

    auto load_unit = [&](int u, VT (&dst)[2][K]) {
        const int tile = u / UPT, s = u - tile * UPT;
        const int64_t off = (int64_t)tile * kTileBytes + s * 4 * UB + q * UB;
        const uint8_t* b0 = planes + row0 * row_bytes + off;
        const uint8_t* b1 = planes + row1 * row_bytes + off;
#pragma unroll
        for (int p = 0; p < K; ++p) {
            dst[0][K - 1 - p] = ok0 ? V::load(b0 + p * plane_stride) : V::zero();
            dst[1][K - 1 - p] = ok1 ? V::load(b1 + p * plane_stride) : V::zero();
        }
    };

    VT bufA[2][K], bufB[2][K];
    int u = warp;
    if (u < n_units) load_unit(u, bufA);

    // ---- centroid tables -> replicated shared-memory lookup tables ----------
    {
        uint16_t* lut_s = reinterpret_cast<uint16_t*>(scratch);
        constexpr int NL = kRowsPerCta << K;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(lut + rb * kRowsPerCta * (1 << K));
        const int64_t valid = (rows - rb * kRowsPerCta) << K;  // halves available
        for (int i = tid; i < NL / 2; i += blockDim.x)
            reinterpret_cast<uint32_t*>(lut_s)[i] = (2 * i < valid) ? __ldg(src + i) : 0u;
        __syncthreads();
        constexpr int NE = TableGeom<K>::kEntries;
        for (int i = tid; i < NE * kRowsPerCta; i += blockDim.x) {
            const int idx = i >> 4, rl = i & 15;
            const uint16_t* lr = lut_s + (rl << K);
            uint32_t v;
            if constexpr (TableGeom<K>::kPair) {
                uint32_t ce, co;
                pair_codes<K>((uint32_t)idx, ce, co);
                v = (uint32_t)lr[ce] | ((uint32_t)lr[co] << 16);
            } else {
                v = lr[idx];
            }
            *reinterpret_cast<uint4*>(table + idx * 256 + rl * 16) = make_uint4(v, v, v, v);
        }
        __syncthreads();
    }

    const uint32_t off0 = (uint32_t)lane * 4u, off1 = 128u + (uint32_t)lane * 4u;
    const uint16_t* xrow[NG];
#pragma unroll
    for (int ng = 0; ng < NG; ++ng) {
        const int m = min(g + 8 * ng, L.m_x - 1);
        xrow[ng] = xg + (int64_t)m * ldx;
    }
    float acc[NG][4];
#pragma unroll
    for (int ng = 0; ng < NG; ++ng) acc[ng][0] = acc[ng][1] = acc[ng][2] = acc[ng][3] = 0.f;

    auto compute_unit = [&](int uu, const VT (&buf)[2][K]) {
        const int tile = uu / UPT, s = uu - tile * UPT;
        const bool full_tile = (int64_t)(tile + 1) * kTileWeights <= cols;
#pragma unroll
        for (int w = 0; w < WPU; ++w) {
            const int t = s * UB + q * WPU + w;  // lane word within the tile
            const int64_t colbase = (int64_t)tile * kTileWeights + 8 * t;
            uint4 xv[NG][4];
            if (full_tile) {
#pragma unroll
                for (int ng = 0; ng < NG; ++ng)
#pragma unroll
                    for (int p = 0; p < 4; ++p)
                        xv[ng][p] = __ldg(reinterpret_cast<const uint4*>(xrow[ng] + colbase + 256 * p));
            } else {
#pragma unroll
                for (int ng = 0; ng < NG; ++ng)
#pragma unroll
                    for (int p = 0; p < 4; ++p)
                        xv[ng][p] = load_x8_tail(xrow[ng], colbase + 256 * p, cols);
            }
            uint32_t Q0[K], Q1[K];
#pragma unroll
            for (int i = 0; i < K; ++i) {
                Q0[i] = V::word(buf[0][i], w);
                Q1[i] = V::word(buf[1][i], w);
            }
            uint32_t a0[16], a1[16];
            decode_word<K>(Q0, table, off0, a0);
            decode_word<K>(Q1, table, off1, a1);
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                    for (int ng = 0; ng < NG; ++ng)
                        mma16816(acc[ng], a0[p * 4 + 2 * jj], a1[p * 4 + 2 * jj],
                                 a0[p * 4 + 2 * jj + 1], a1[p * 4 + 2 * jj + 1],
                                 u4_word(xv[ng][p], 2 * jj), u4_word(xv[ng][p], 2 * jj + 1));
        }
    };

    // ---- main loop: double-buffered unit stream ------------------------------
#pragma unroll 1
    while (u < n_units) {
        int un = u + nwarps;
        if (un < n_units) load_unit(un, bufB);
        compute_unit(u, bufA);
        u = un;
        if (u >= n_units) break;
        un = u + nwarps;
        if (un < n_units) load_unit(un, bufA);
        compute_unit(u, bufB);
        u = un;
    }

    // ---- fixed-order CTA reduction + store ---------------------------------
    float* red = reinterpret_cast<float*>(scratch);  // [warp][16 rows][8*NG cols]
    constexpr int RC = 8 * NG;
#pragma unroll
    for (int ng = 0; ng < NG; ++ng) {
        float* r0p = red + (warp * kRowsPerCta + g) * RC + ng * 8 + 2 * q;
        float* r1p = red + (warp * kRowsPerCta + g + 8) * RC + ng * 8 + 2 * q;
        r0p[0] = acc[ng][0];
        r0p[1] = acc[ng][1];
        r1p[0] = acc[ng][2];
        r1p[1] = acc[ng][3];
    }
    __syncthreads();
    const int m_out = L.x_split ? (L.m_x >> 1) : L.m_x;
    for (int i = tid; i < kRowsPerCta * m_out; i += blockDim.x) {
        const int rl = i & 15, m = i >> 4;
        const int64_t row = rb * kRowsPerCta + rl;
        if (row >= rows) continue;
        float s;
        if (L.x_split) {
            float hi = 0.f, lo = 0.f;
            for (int w = 0; w < nwarps; ++w) hi += red[(w * kRowsPerCta + rl) * RC + 2 * m];
            for (int w = 0; w < nwarps; ++w) lo += red[(w * kRowsPerCta + rl) * RC + 2 * m + 1];
            s = hi + lo;
        } else {
            s = 0.f;
            for (int w = 0; w < nwarps; ++w) s += red[(w * kRowsPerCta + rl) * RC + m];
        }
        if (L.y_f16)
            reinterpret_cast<__half*>(yg)[(int64_t)m * ldy + row] = __float2half_rn(s);
        else
            reinterpret_cast<float*>(yg)[(int64_t)m * ldy + row] = s;
    }
}

template <int K, int NG, int UB>
static size_t smem_bytes(int nwarps) {
    const size_t lut_stage = (size_t)kRowsPerCta * (1u << K) * 2;
    const size_t red = (size_t)nwarps * kRowsPerCta * 8 * NG * 4;
    return TableGeom<K>::kBytes + (lut_stage > red ? lut_stage : red);
}

template <int K, int NG, int UB>
static int launch_variant(const GemvLaunch& L, int n_blocks, int nwarps, cudaStream_t s) {
    static std::atomic<int> configured{0};
    const size_t smem = smem_bytes<K, NG, UB>(GemvBounds<NG>::kThreads / 32);
    if (!configured.load(std::memory_order_acquire)) {
        if (cudaFuncSetAttribute(gemv_kernel<K, NG, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return APB_ERR_CUDA;
        configured.store(1, std::memory_order_release);
    }
    gemv_kernel<K, NG, UB><<<n_blocks, nwarps * 32, smem_bytes<K, NG, UB>(nwarps), s>>>(L);
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

template <int K, int NG>
static int dispatch_ub(const GemvLaunch& L, int n_blocks, int nwarps, cudaStream_t s) {
    if constexpr (K <= 5) return launch_variant<K, NG, 16>(L, n_blocks, nwarps, s);
    else return launch_variant<K, NG, 8>(L, n_blocks, nwarps, s);
}

template <int K>
static int dispatch_ng(int ng, const GemvLaunch& L, int n_blocks, int nwarps, cudaStream_t s) {
    switch (ng) {
        case 1: return dispatch_ub<K, 1>(L, n_blocks, nwarps, s);
        case 2: return dispatch_ub<K, 2>(L, n_blocks, nwarps, s);
        default: return dispatch_ub<K, 4>(L, n_blocks, nwarps, s);
    }
}

static int units_per_tile(int k) { return k <= 5 ? 2 : 4; }

// Warps per CTA: a divisor of the unit count in [4, 12] when one exists
// (balanced K split), otherwise 8.
static int pick_warps(int n_units, int max_warps) {
    for (int w = 8; w >= 4; --w)
        if (n_units % w == 0) return w;
    for (int w = 9; w <= max_warps; ++w)
        if (n_units % w == 0) return w;
    return n_units < 8 ? (n_units < 1 ? 1 : n_units) : 8;
}

}  // namespace apb

using namespace apb;

static int gemv_launch_chunk(int n, const uint8_t* const* planes, const int* n_max,
                             const int64_t* rows, const int64_t* cols, const int64_t* padded, int k,
                             const uint16_t* const* lut, const uint16_t* const* x, int m_x,
                             const int64_t* ldx, int64_t x_off, int x_split, void* const* y,
                             int y_dtype, const int64_t* ldy, int64_t y_off, cudaStream_t s) {
    GemvLaunch L;
    L.n_prob = n;
    L.m_x = m_x;
    L.x_split = x_split;
    L.y_f16 = y_dtype == APB_DTYPE_F16;
    int blocks = 0, max_units = 0;
    const int esz = y_dtype == APB_DTYPE_F16 ? 2 : 4;
    for (int i = 0; i < n; ++i) {
        GemvProblem& P = L.prob[i];
        P.planes = planes[i];
        P.lut = lut[i];
        P.x = x[i] + x_off * ldx[i];
        P.y = reinterpret_cast<uint8_t*>(y[i]) + y_off * ldy[i] * esz;
        P.rows = rows[i];
        P.cols = cols[i];
        P.row_bytes = padded[i] / 8;
        P.plane_stride = rows[i] * (padded[i] / 8);
        P.ldx = ldx[i];
        P.ldy = ldy[i];
        P.n_tiles = (int)(padded[i] / kTileWeights);
        P.block_begin = blocks;
        blocks += (int)((rows[i] + kRowsPerCta - 1) / kRowsPerCta);
        const int nu = P.n_tiles * units_per_tile(k);
        if (nu > max_units) max_units = nu;
    }
    const int ng = m_x <= 8 ? 1 : (m_x <= 16 ? 2 : 4);
    const int nwarps = pick_warps(max_units, ng == 1 ? 12 : 8);
    switch (k) {
        case 2: return dispatch_ng<2>(ng, L, blocks, nwarps, s);
        case 3: return dispatch_ng<3>(ng, L, blocks, nwarps, s);
        case 4: return dispatch_ng<4>(ng, L, blocks, nwarps, s);
        case 5: return dispatch_ng<5>(ng, L, blocks, nwarps, s);
        case 6: return dispatch_ng<6>(ng, L, blocks, nwarps, s);
        case 7: return dispatch_ng<7>(ng, L, blocks, nwarps, s);
        case 8: return dispatch_ng<8>(ng, L, blocks, nwarps, s);
    }
    return APB_ERR_PARAM;
}

extern "C" int apb_gemv_grouped(int n_problems, const uint8_t* const* planes, const int* n_max,
                                const int64_t* rows, const int64_t* cols,
                                const int64_t* padded_cols, int k, const uint16_t* const* lut,
                                const uint16_t* const* x, int m_x, const int64_t* ldx, int x_split,
                                void* const* y, int y_dtype, const int64_t* ldy, void* stream) {
    if (n_problems < 1) return APB_ERR_SHAPE;
    if (k < 2 || k > 8) return APB_ERR_PARAM;
    if (y_dtype != APB_DTYPE_F32 && y_dtype != APB_DTYPE_F16) return APB_ERR_PARAM;
    if (m_x < 1 || (x_split && (m_x & 1))) return APB_ERR_SHAPE;
    const int m_out = x_split ? m_x / 2 : m_x;
    for (int i = 0; i < n_problems; ++i) {
        if (rows[i] <= 0 || cols[i] <= 0) return APB_ERR_SHAPE;
        if (padded_cols[i] != apb_pad_columns(cols[i])) return APB_ERR_SHAPE;
        if (k > n_max[i] || n_max[i] > 8) return APB_ERR_PARAM;
        if (ldx[i] < cols[i] || (ldx[i] % 8) != 0) return APB_ERR_PARAM;
        if (((uintptr_t)x[i] & 15) != 0 || ((uintptr_t)planes[i] & 15) != 0) return APB_ERR_PARAM;
        if (((uintptr_t)lut[i] & 3) != 0) return APB_ERR_PARAM;
        if (ldy[i] < rows[i]) return APB_ERR_SHAPE;
        if (!planes[i] || !lut[i] || !x[i] || !y[i]) return APB_ERR_PARAM;
    }
    cudaStream_t s = (cudaStream_t)stream;
    // batch columns per launch: 32 fp16 activation rows (4 mma column groups)
    const int chunk = 32;
    for (int p0 = 0; p0 < n_problems; p0 += kMaxGroup) {
        const int n = n_problems - p0 < kMaxGroup ? n_problems - p0 : kMaxGroup;
        for (int m0 = 0; m0 < m_x; m0 += chunk) {
            const int mc = m_x - m0 < chunk ? m_x - m0 : chunk;
            const int rc = gemv_launch_chunk(n, planes + p0, n_max + p0, rows + p0, cols + p0,
                                             padded_cols + p0, k, lut + p0, x + p0, mc, ldx + p0,
                                             m0, x_split, y + p0, y_dtype, ldy + p0,
                                             x_split ? m0 / 2 : m0, s);
            if (rc != APB_OK) return rc;
        }
    }
    (void)m_out;
    return APB_OK;
}

extern "C" int apb_gemv(const uint8_t* planes, int n_max, int64_t rows, int64_t cols,
                        int64_t padded_cols, int k, const uint16_t* lut, const uint16_t* x, int m_x,
                        int64_t ldx, int x_split, void* y, int y_dtype, int64_t ldy, void* stream) {
    return apb_gemv_grouped(1, &planes, &n_max, &rows, &cols, &padded_cols, k, &lut, &x, m_x, &ldx,
                            x_split, &y, y_dtype, &ldy, stream);
}
