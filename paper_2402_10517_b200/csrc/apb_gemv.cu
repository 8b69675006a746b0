// apb_gemv.cu -- bitplane any-precision GEMV / small-batch GEMM for sm_100a.
//
// Replaces engine.py:284-309 (gemv) and engine.py:312-341 (gemm, quantized
// path) of the reference.  Same maths: y[m][r] = sum_c LUT_k[r][code_k(r,c)] *
// x[m][c], reading ONLY planes 0..k-1 and the k-bit table.
//
// Work item = one 16-row block of one problem (layer) x all K columns.
// Persistent grid: each CTA owns a contiguous, cost-balanced range of items
// (possibly spanning several layers of a grouped launch) and streams them:
// while a row block is being computed, the planes of the next units (which
// may belong to the next row block) are already in flight in registers and
// the next block's centroid rows are being copied into shared memory by
// cp.async, so the per-block prologue (DRAM latency + table build) is hidden.
//
// Inside an item, W warps split the K dimension into "units" (one 16- or
// 8-byte slice of a 128-byte tile-plane row per lane).  Lane (g, q) =
// (lane>>2, lane&3) owns rows g and g+8 of the block.
// Decode: bit networks of apb_common.cuh (no per-weight shift/mask):
//   k <= 4: to_pairs -> one PRMT + one LDS per PAIR of weights from a 4^k
//           entry pair table (the paper's merged lookup);
//   k >= 5: to_bytes -> one PRMT + one LDS per weight, pairs packed into
//           fp16x2 with one IMAD (FMA pipe).
//   Tables are replicated per lane slot ([entry][row-half][lane]) so every
//   lookup is bank-conflict free (bank == lane); one PRMT builds the byte
//   address [lane*4 | row-half*128 | idx<<8], the table base folds into the
//   LDS immediate.
// MAC: the decoded fp16x2 weights ARE the A fragment of mma.sync.m16n8k16
//   (rows g, g+8; k-slots 2q.., 2q+8..), the activations the B fragment
//   (batch columns n = g), accumulation fp32 in the tensor core: 1 HMMA per
//   256 weights instead of 128 FFMA, and batch 1..8 costs the same as batch 1.
// Deterministic: fixed mma k-order, fixed chain split, warps reduced 0..W-1.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>

#include "../../include/anyprec_b200.h"
#include "apb_common.cuh"

namespace apb {

constexpr int kMaxGroup = 16;
constexpr int kRowsPerCta = 16;

#ifdef APB_TIMELINE
// Debug builds (tools/timeline): per-CTA phase timestamps (globaltimer, ns).
__device__ unsigned long long* g_timeline = nullptr;
#define APB_TS(i)                                                          \
    do {                                                                   \
        if (threadIdx.x == 0 && g_timeline) {                              \
            unsigned long long t_;                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));         \
            g_timeline[(size_t)blockIdx.x * 8 + (i)] = t_;                 \
        }                                                                  \
    } while (0)
// per-warp cycle accounting: [prologue, in-unit, total, units]
__device__ unsigned long long* g_warpstat = nullptr;
#define APB_CLK(v) long long v = clock64()
#else
#define APB_TS(i) \
    do {          \
    } while (0)
#define APB_CLK(v)
#endif

struct GemvProblem {
    const uint8_t* planes;  // permuted planes, plane 0 (MSB) first
    const uint16_t* lut;    // fp16 [rows][1<<K]
    const uint16_t* x;      // fp16 [m_x][ldx]
    void* y;                // [m_out][ldy]
    int64_t rows, cols, row_bytes, plane_stride, ldx, ldy;
    int n_tiles;
    int item_begin;         // first global item (row block) of this problem
    int64_t cost_begin;     // prefix cost (tiles) of the items before this problem
    const float* xinv;      // x_split == 2: per output row inverse activation scale (else null)
};

struct GemvLaunch {
    GemvProblem prob[kMaxGroup];
    int n_prob;
    int n_items;
    int64_t total_cost;
    int m_x;
    int x_split;
    int y_f16;
    int64_t xs_bytes;  // > 0: activations staged in shared memory ([m_x][padded] fp16)
    int flags;         // APB_FLAG_*
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

// Shared-window address of the dynamic shared memory (the lookup table sits at
// its start).  sm_100 reserves the first 1 KB of the window, so the table is at
// 0x400; the kernel verifies this at entry (and traps otherwise) so the table
// lookup can be a single LDS [R + imm] with the PRMT-built byte offset --
// without it ptxas keeps the base in a general register and spends one IADD
// per lookup.
#define APB_SMEM_BASE 1024
__device__ __forceinline__ uint32_t lds_table(uint32_t off) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+1024];" : "=r"(v) : "r"(off));
    return v;
}
__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }
// 16-byte shared load executed only where pred != 0; elsewhere the outputs are
// don't-care values (used for MMA B-fragment columns that are never read).
__device__ __forceinline__ void lds128_pred(uint4& v, uint32_t saddr, uint32_t pred) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t"
        "@p ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
        : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
        : "r"(saddr), "r"(pred));
}

__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// cp.async 16 bytes, zero-filling beyond src_bytes (0..16).
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 8 fp16 activations at columns col..col+7, zero beyond cols (tail tile, global path).
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
    static constexpr int kStageBytes = kRowsPerCta * (1 << K) * 2;  // 16 centroid rows
};

// Decode one lane word of one row into 16 fp16x2 values:
// out[p*4 + j] = weights of columns (256p + 8t + 2j, +1) of this row.
template <int K>
__device__ __forceinline__ void decode_word(const uint32_t* Q, uint32_t off, uint32_t* out) {
    if constexpr (TableGeom<K>::kPair) {
        uint32_t U[4];
        to_pairs<K>(Q, U);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p)
                out[p * 4 + j] = lds_table(prmt(U[j], off, 0x7604u | (uint32_t)(p << 4)));
    } else {
        uint32_t Wb[8];
        to_bytes<K>(Q, Wb);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const uint32_t sel = 0x7604u | (uint32_t)(p << 4);
                const uint32_t e = lds_table(prmt(Wb[2 * j], off, sel));
                const uint32_t o = lds_table(prmt(Wb[2 * j + 1], off, sel));
                out[p * 4 + j] = e + (o << 16);  // IMAD: o * 65536 + e (e < 65536)
            }
    }
}

// ---- warp-specialised persistent kernel --------------------------------------
// One CTA per SM.  Compute warps stream units (decode + MMA) continuously
// across row blocks; service warps (1 or 2, by table size) build each block's
// lookup table into one of two table slots, stage activations, and reduce +
// store each block's outputs.  Compute and service warps hand off through
// mbarriers (table_ready[slot], item_done[slot]); there is no CTA-wide barrier
// in the steady state, so a slow warp never stalls the others.
template <int K, int NG>
struct WsGeom {
    static constexpr int kTotalWarps = NG == 1 ? 16 : 8;
    static constexpr int kServiceWarps = TableGeom<K>::kEntries >= 256 ? 2 : 1;
    static constexpr int kComputeWarps = kTotalWarps - kServiceWarps;
    static constexpr int kThreads = kTotalWarps * 32;
    // table slot 1 sits 64 KB after slot 0, so the slot index is address byte 2
    // and the lookup address stays one PRMT (see decode_word / lds_table)
    static constexpr int kSlotStride = 64 * 1024;
    static constexpr int kRedBytes = kComputeWarps * kRowsPerCta * 8 * NG * 4;  // one slot
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ int problem_of(const GemvLaunch& L, int item) {
    int pi = 0;
#pragma unroll 1
    for (int i = 1; i < L.n_prob; ++i)
        if (item >= L.prob[i].item_begin) pi = i;
    return pi;
}
__device__ __forceinline__ int problem_end(const GemvLaunch& L, int pi) {
    return pi + 1 < L.n_prob ? L.prob[pi + 1].item_begin : L.n_items;
}

// First item whose cumulative cost start is >= target (items are cost-uniform
// within a problem, cost = n_tiles).  Every CTA gets a contiguous,
// cost-balanced item range.
__device__ __forceinline__ int item_at_cost(const GemvLaunch& L, int64_t target) {
    if (target >= L.total_cost) return L.n_items;
#pragma unroll 1
    for (int i = 0; i < L.n_prob; ++i) {
        const GemvProblem& P = L.prob[i];
        const int n = problem_end(L, i) - P.item_begin;
        const int64_t end = P.cost_begin + (int64_t)n * P.n_tiles;
        if (target < end) {
            const int64_t d = target - P.cost_begin;
            return P.item_begin + (int)((d + P.n_tiles - 1) / P.n_tiles);
        }
    }
    return L.n_items;
}

// smem layout: [table slot 0][.. slot 1 at +64K][red x2][xs x2][mbarriers]
template <int K, int NG>
struct WsLayout {
    static constexpr int kTable1 = WsGeom<K, NG>::kSlotStride;
    static constexpr int kRed = kTable1 + TableGeom<K>::kBytes;
    static constexpr int kXs = kRed + 2 * WsGeom<K, NG>::kRedBytes;
    __host__ __device__ static size_t bars(int64_t xs_bytes) { return (size_t)kXs + 2 * (size_t)((xs_bytes + 127) / 128 * 128); }
    __host__ __device__ static size_t total(int64_t xs_bytes) { return bars(xs_bytes) + 64; }
};

// Service role (1-2 warps): for every item of the CTA's range, build its lookup
// table into table slot (j & 1), stage the layer's activations (XS) on a layer
// change, and -- two items later, once every compute warp has arrived on
// item_done -- reduce the per-warp partials and store y.  Shared by the v5 and
// v6 kernels.
template <int K, int NSW, int WC, int RC, bool XS, int XUB = 0, int NSLOT = 2, int KPF = 0>
__device__ __forceinline__ void service_role(const GemvLaunch& L, int first, int last, uint8_t* smem,
                                             uint32_t bar, float* red, uint8_t* xs, int64_t xs_slot,
                                             int st, int slot_stride) {
    using TG = TableGeom<K>;
    const int n_local = last - first;
    {
        // =============================== service warps =========================
        const int nst = NSW * 32;
        const int lane = st & 31;
        // centroid rows of the next block, prefetched into registers
        constexpr int kItems = TG::kPair ? (kRowsPerCta << K) : (kRowsPerCta * (1 << K) / 8);
        constexpr int kPer = (kItems + NSW * 32 - 1) / (NSW * 32);
        constexpr int kRowVecs = TG::kPair ? ((1 << K) + 7) / 8 : 1;
        uint4 src[kPer][kRowVecs];
        auto load_lut = [&](int item, int pi) {
            const GemvProblem& P = L.prob[pi];
            const int64_t rb = item - P.item_begin;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int it = st + i * nst;
                const int rl = it & 15;
                const int64_t row = rb * kRowsPerCta + rl;
#pragma unroll
                for (int v = 0; v < kRowVecs; ++v) src[i][v] = make_uint4(0, 0, 0, 0);
                if (it < kItems && row < P.rows) {
                    const uint16_t* lr = P.lut + row * (1 << K);
                    if constexpr (TG::kPair) {
                        if constexpr ((1 << K) >= 8) {
#pragma unroll
                            for (int v = 0; v < kRowVecs; ++v)
                                src[i][v] = __ldg(reinterpret_cast<const uint4*>(lr) + v);
                        } else {
                            const uint2 h = __ldg(reinterpret_cast<const uint2*>(lr));
                            src[i][0] = make_uint4(h.x, h.y, 0, 0);
                        }
                    } else {
                        src[i][0] = __ldg(reinterpret_cast<const uint4*>(lr) + (it >> 4));
                    }
                }
            }
        };
        auto half_at = [&](const uint4(&rv)[kRowVecs], int i) -> uint32_t {
            const uint32_t w = u4_word(rv[i >> 3], (i >> 1) & 3);
            return (i & 1) ? (w >> 16) : (w & 0xFFFFu);
        };
        auto build = [&](int slot) {
            uint8_t* const tbase = smem + slot * slot_stride;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int it = st + i * nst;
                if (it >= kItems) continue;
                const int rl = it & 15;
                uint8_t* dst = tbase + rl * 16;
                if constexpr (TG::kPair) {
                    const int ce = it >> 4;  // its 2^K entries are (L[ce], L[co]) for every co
                    uint32_t lce = 0;
#pragma unroll
                    for (int c = 0; c < (1 << K); ++c)
                        if (c == ce) lce = half_at(src[i], c);
                    uint32_t sce = 0;  // code bit b -> pair-index bit 2b
#pragma unroll
                    for (int b = 0; b < K; ++b) sce |= (((uint32_t)ce >> b) & 1u) << (2 * b);
#pragma unroll
                    for (int co = 0; co < (1 << K); ++co) {
                        uint32_t sco = 0;
#pragma unroll
                        for (int b = 0; b < K; ++b) sco |= ((uint32_t)(co >> b) & 1u) << (2 * b + 1);
                        const uint32_t v = lce | (half_at(src[i], co) << 16);
                        *reinterpret_cast<uint4*>(dst + (sce | sco) * 256) = make_uint4(v, v, v, v);
                    }
                } else {
                    const int e8 = it >> 4;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const uint32_t v = half_at(src[i], jj);
                        *reinterpret_cast<uint4*>(dst + (e8 * 8 + jj) * 256) = make_uint4(v, v, v, v);
                    }
                }
            }
        };
        auto stage_x = [&](int pi, int xb) {
            const GemvProblem& P = L.prob[pi];
            if constexpr (XUB > 0) {
                // v6 layout: [unit u][m][p][wi][q] 16-byte chunks, m stride XMSTR
                // (= 64 mod 128: batch rows of one chunk group hit disjoint banks)
                constexpr int WPU = XUB / 4, UPT = 128 / (4 * XUB), XMSTR = 4 * WPU * 64 + 64;
                const int per_u = L.m_x * 4 * WPU * 4;  // chunks per unit
                const int chunks = P.n_tiles * UPT * per_u;
                for (int c = st; c < chunks; c += nst) {
                    const int u = c / per_u, r = c - u * per_u;
                    const int m = r / (4 * WPU * 4), r2 = r - m * (4 * WPU * 4);
                    const int pw = r2 >> 2, qq = r2 & 3;  // pw = p*WPU + wi
                    const int pp = pw / WPU, wi = pw - pp * WPU;
                    const int tile = u / UPT, sl = u - tile * UPT;
                    const int t = sl * XUB + qq * WPU + wi;
                    const int64_t col = (int64_t)tile * kTileWeights + 256 * pp + 8 * t;
                    const int64_t nb = (P.cols - col) * 2;
                    const uint16_t* srow = P.x + (int64_t)m * P.ldx;
                    uint8_t* dst = xs + xb * xs_slot + ((int64_t)u * L.m_x + m) * XMSTR + r2 * 16;
                    cp_async16(dst, nb > 0 ? (const void*)(srow + col) : (const void*)srow,
                               nb >= 16 ? 16 : (nb > 0 ? (int)nb : 0));
                }
                cp_async_commit();
                cp_async_wait_all();
                return;
            }
            const int64_t padded = (int64_t)P.n_tiles * kTileWeights;
            const int chunks = (int)(padded / 8);
            for (int m = 0; m < L.m_x; ++m) {
                const uint16_t* srow = P.x + (int64_t)m * P.ldx;
                uint8_t* drow = xs + xb * xs_slot + (int64_t)m * padded * 2;
                for (int c = st; c < chunks; c += nst) {
                    const int64_t col = (int64_t)c * 8;
                    const int64_t nb = (P.cols - col) * 2;
                    cp_async16(drow + col * 2, nb > 0 ? (const void*)(srow + col) : (const void*)srow,
                               nb >= 16 ? 16 : (nb > 0 ? (int)nb : 0));
                }
            }
            cp_async_commit();
            cp_async_wait_all();
        };
        auto reduce = [&](int item, int pi, int slot) {
            const GemvProblem& P = L.prob[pi];
            const int64_t rb = item - P.item_begin;
            const int m_out = L.x_split ? (L.m_x >> 1) : L.m_x;
            const float* r = red + slot * (WC * kRowsPerCta * RC);
            for (int i = st; i < kRowsPerCta * m_out; i += nst) {
                const int rl = i & 15, m = i >> 4;
                const int64_t row = rb * kRowsPerCta + rl;
                if (row >= P.rows) continue;
                float sum;
                if (L.x_split) {
                    float hi = 0.f, lo = 0.f;
#pragma unroll
                    for (int w = 0; w < WC; ++w) hi += r[(w * kRowsPerCta + rl) * RC + 2 * m];
#pragma unroll
                    for (int w = 0; w < WC; ++w) lo += r[(w * kRowsPerCta + rl) * RC + 2 * m + 1];
                    sum = hi + lo;
                    if (L.x_split == 2) sum *= P.xinv[m];  // scaled pairs: undo the power-of-two scale
                } else {
                    sum = 0.f;
#pragma unroll
                    for (int w = 0; w < WC; ++w) sum += r[(w * kRowsPerCta + rl) * RC + m];
                }
                if (L.y_f16)
                    reinterpret_cast<__half*>(P.y)[(int64_t)m * P.ldy + row] = __float2half_rn(sum);
                else
                    reinterpret_cast<float*>(P.y)[(int64_t)m * P.ldy + row] = sum;
            }
        };

        // L2 prefetch (bulk, one instruction per plane) of the top-KPF planes of
        // an upcoming item, so the compute warps' plane loads hit L2
        auto prefetch_item = [&](int item) {
            if constexpr (KPF > 0) {
                if (st != 0 || item >= last) return;
                const GemvProblem& P = L.prob[problem_of(L, item)];
                const int64_t r0 = (int64_t)(item - P.item_begin) * kRowsPerCta;
                const int64_t nr = P.rows - r0 < kRowsPerCta ? P.rows - r0 : kRowsPerCta;
                const uint8_t* a = P.planes + r0 * P.row_bytes;
                const uint32_t bytes = (uint32_t)(nr * P.row_bytes);
#pragma unroll 1
                for (int pl = 0; pl < KPF; ++pl)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + (int64_t)pl * P.plane_stride),
                                 "r"(bytes)
                                 : "memory");
            }
        };
        prefetch_item(first + 1);
        prefetch_item(first + 2);
        // activations / outputs may belong to the previous kernel in the stream
        asm volatile("griddepcontrol.wait;" ::: "memory");
        int pi = problem_of(L, first), pend = problem_end(L, pi);
        int xb = 0, pi_hist[NSLOT];
#pragma unroll
        for (int i = 0; i < NSLOT; ++i) pi_hist[i] = pi;
        load_lut(first, pi);
#pragma unroll 1
        for (int jl = 0; jl < n_local + NSLOT; ++jl) {
            const int sl = jl % NSLOT;
            if (jl >= NSLOT) {  // item jl-NSLOT finished by every compute warp: reduce it, free its slot
                mbar_wait(bar + 8 * NSLOT + 8 * sl, ((jl - NSLOT) / NSLOT) & 1);
                reduce(first + jl - NSLOT, pi_hist[sl], sl);
            }
            if (jl < n_local) {
                prefetch_item(first + jl + 3);
                const int item = first + jl;
                if (item >= pend) {  // next layer of a grouped launch
                    pi = problem_of(L, item);
                    pend = problem_end(L, pi);
                    xb ^= 1;
                    if constexpr (XS) stage_x(pi, xb);
                } else if (jl == 0) {
                    if constexpr (XS) stage_x(pi, xb);
                }
                pi_hist[sl] = pi;
                build(sl);
                // prefetch the next block's centroid rows while this one is consumed
                if (item + 1 < last) {
                    const int npi = item + 1 >= pend ? problem_of(L, item + 1) : pi;
                    load_lut(item + 1, npi);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bar + 8 * sl);
            }
        }
    }
}

template <int K, int NG, int UB, bool XS>
__global__ void __launch_bounds__(WsGeom<K, NG>::kThreads, 1)
    gemv_kernel(const __grid_constant__ GemvLaunch L) {
    using V = UnitVec<UB>;
    using VT = typename V::T;
    using TG = TableGeom<K>;
    using G = WsGeom<K, NG>;
    using LY = WsLayout<K, NG>;
    constexpr int WC = G::kComputeWarps;
    constexpr int WPU = UB / 4;          // lane words per unit per row
    constexpr int UPT = 128 / (4 * UB);  // units per tile
    constexpr int RC = 8 * NG;           // reduction columns

    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3;
    if (smem_addr(smem) != APB_SMEM_BASE) __trap();  // see lds_table

    const int first = item_at_cost(L, L.total_cost * (int64_t)blockIdx.x / gridDim.x);
    const int last = item_at_cost(L, L.total_cost * (int64_t)(blockIdx.x + 1) / gridDim.x);
    asm volatile("griddepcontrol.launch_dependents;");
    if (first >= last) return;
    const int n_local = last - first;

    float* const red = reinterpret_cast<float*>(smem + LY::kRed);  // [2][WC][16][RC]
    const int64_t xs_slot = (L.xs_bytes + 127) / 128 * 128;
    uint8_t* const xs = smem + LY::kXs;                              // [2][xs_slot]
    const uint32_t bar = smem_addr(smem + LY::bars(L.xs_bytes));
    // bar + 0 / 8: table_ready[slot] (count = service warps)
    // bar + 16 / 24: item_done[slot] (count = compute warps)
    if (tid == 0) {
        mbar_init(bar + 0, G::kServiceWarps);
        mbar_init(bar + 8, G::kServiceWarps);
        mbar_init(bar + 16, WC);
        mbar_init(bar + 24, WC);
    }
    __syncthreads();

    if (warp >= WC) {
        service_role<K, G::kServiceWarps, WC, RC, XS>(L, first, last, smem, bar, red, xs, xs_slot,
                                                      tid - WC * 32, G::kSlotStride);
        return;
    }

    // =============================== compute warps =============================
#ifdef APB_TIMELINE
    long long clk_start = clock64(), clk_units = 0, clk_ldwait = 0, clk_tblwait = 0, n_done = 0;
#endif
    if constexpr (!XS) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int w = warp;
    // plane-load iterator over this warp's global unit sequence w, w+WC, ...
    int li_j = 0, li_pi = problem_of(L, first), li_pend = problem_end(L, li_pi);
    int64_t li_base = 0;
    int li_units = 0;
    int64_t li_rows = 0, li_rbytes = 0, li_row0 = 0, li_pstride = 0;
    const uint8_t* li_b0 = nullptr;
    int64_t li_g = w;
    auto li_fields = [&](int item) {
        const GemvProblem& P = L.prob[li_pi];
        li_units = P.n_tiles * UPT;
        li_rows = P.rows;
        li_rbytes = P.row_bytes;
        li_pstride = P.plane_stride;
        li_row0 = (int64_t)(item - P.item_begin) * kRowsPerCta + g;
        li_b0 = P.planes + li_row0 * P.row_bytes + q * UB;
    };
    li_fields(first);
    auto li_load = [&](VT(&dst)[2][K]) {
        while (li_j < n_local && li_g >= li_base + li_units) {  // advance to the unit's block
            li_base += li_units;
            ++li_j;
            if (li_j >= n_local) break;
            const int item = first + li_j;
            if (item >= li_pend) {
                ++li_pi;
                while (item >= problem_end(L, li_pi)) ++li_pi;
                li_pend = problem_end(L, li_pi);
                li_fields(item);
            } else {
                li_row0 += kRowsPerCta;
                li_b0 += kRowsPerCta * li_rbytes;
            }
        }
        if (li_j >= n_local) return;
        const int u = (int)(li_g - li_base);
        const int tile = u / UPT, s = u - tile * UPT;
        const uint8_t* p0 = li_b0 + (int64_t)tile * kTileBytes + s * 4 * UB;
        const uint8_t* p1 = p0 + 8 * li_rbytes;
        const bool ok0 = li_row0 < li_rows, ok1 = li_row0 + 8 < li_rows;
#pragma unroll
        for (int p = 0; p < K; ++p) {
            dst[0][K - 1 - p] = ok0 ? V::load(p0 + p * li_pstride) : V::zero();
            dst[1][K - 1 - p] = ok1 ? V::load(p1 + p * li_pstride) : V::zero();
        }
        li_g += WC;
    };

    VT bufA[2][K], bufB[2][K];
    li_load(bufA);
    li_load(bufB);

    int xm[NG];
#pragma unroll
    for (int ng = 0; ng < NG; ++ng) xm[ng] = min(g + 8 * ng, L.m_x - 1);
    int cpi = problem_of(L, first), cpend = problem_end(L, cpi), xb = 0;
    int64_t base = 0, gu = w;
    int ring = 0;
#pragma unroll 1
    for (int jl = 0; jl < n_local; ++jl) {
        const int item = first + jl;
        if (item >= cpend) {
            cpi = problem_of(L, item);
            cpend = problem_end(L, cpi);
            xb ^= 1;
        }
        const GemvProblem& P = L.prob[cpi];
        const int units = P.n_tiles * UPT;
        const int64_t cols = P.cols;
        const int64_t padded = (int64_t)P.n_tiles * kTileWeights;
        const uint8_t* const xsb = xs + xb * xs_slot;
        const uint32_t slot_bits = (uint32_t)(jl & 1) << 16;
        const uint32_t off0 = slot_bits | ((uint32_t)lane * 4u), off1 = off0 + 128u;
        float acc[NG][2][4];
#pragma unroll
        for (int ng = 0; ng < NG; ++ng)
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) acc[ng][c2][0] = acc[ng][c2][1] = acc[ng][c2][2] = acc[ng][c2][3] = 0.f;

        auto compute_unit = [&](int uu, const VT(&buf)[2][K]) {
#ifdef APB_TIMELINE
            {  // diagnostics: force the wait for this unit's plane data here
                long long t0 = clock64();
                uint32_t dep = 0;
#pragma unroll
                for (int i = 0; i < K; ++i) dep ^= V::word(buf[0][i], 0) ^ V::word(buf[1][i], WPU - 1);
                asm volatile("" ::"r"(dep));
                if (dep == 0x9e3779b9u) clk_units += 1;  // keep dep live
                clk_ldwait += clock64() - t0;
            }
#endif
            const int tile = uu / UPT, s = uu - tile * UPT;
            const bool full_tile = XS || (int64_t)(tile + 1) * kTileWeights <= cols;
#pragma unroll
            for (int wi = 0; wi < WPU; ++wi) {
                const int t = s * UB + q * WPU + wi;  // lane word within the tile
                const int64_t colbase = (int64_t)tile * kTileWeights + 8 * t;
                uint4 xv[NG][4];
#pragma unroll
                for (int ng = 0; ng < NG; ++ng)
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        // only lanes holding a real batch column load x (B columns
                        // n >= m_x are never read back)
                        if (g + 8 * ng >= L.m_x) {
                            xv[ng][p] = make_uint4(0, 0, 0, 0);
                        } else if constexpr (XS) {
                            xv[ng][p] = lds128(xsb + (xm[ng] * padded + colbase + 256 * p) * 2);
                        } else {
                            const uint16_t* xr = P.x + (int64_t)xm[ng] * P.ldx;
                            xv[ng][p] = full_tile ? __ldg(reinterpret_cast<const uint4*>(xr + colbase + 256 * p))
                                                  : load_x8_tail(xr, colbase + 256 * p, cols);
                        }
                    }
                uint32_t Q0[K], Q1[K];
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    Q0[i] = V::word(buf[0][i], wi);
                    Q1[i] = V::word(buf[1][i], wi);
                }
                uint32_t a0[16], a1[16];
                decode_word<K>(Q0, off0, a0);
                decode_word<K>(Q1, off1, a1);
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                        for (int ng = 0; ng < NG; ++ng)
                            mma16816(acc[ng][p & 1], a0[p * 4 + 2 * jj], a1[p * 4 + 2 * jj],
                                     a0[p * 4 + 2 * jj + 1], a1[p * 4 + 2 * jj + 1],
                                     u4_word(xv[ng][p], 2 * jj), u4_word(xv[ng][p], 2 * jj + 1));
            }
        };

#ifdef APB_TIMELINE
        long long tw0 = clock64();
#endif
        mbar_wait(bar + 8 * (jl & 1), (jl >> 1) & 1);  // this block's table (and x) ready
#ifdef APB_TIMELINE
        clk_tblwait += clock64() - tw0;
        long long tu0 = clock64();
#endif
#pragma unroll 1
        for (; gu < base + units; gu += WC) {
            const int u = (int)(gu - base);
            if (ring & 1) {
                compute_unit(u, bufB);
                li_load(bufB);
            } else {
                compute_unit(u, bufA);
                li_load(bufA);
            }
            ++ring;
#ifdef APB_TIMELINE
            ++n_done;
#endif
        }
#ifdef APB_TIMELINE
        clk_units += clock64() - tu0;
#endif
        float* r = red + (jl & 1) * (WC * kRowsPerCta * RC);
#pragma unroll
        for (int ng = 0; ng < NG; ++ng) {
            float* r0p = r + (w * kRowsPerCta + g) * RC + ng * 8 + 2 * q;
            float* r1p = r + (w * kRowsPerCta + g + 8) * RC + ng * 8 + 2 * q;
            r0p[0] = acc[ng][0][0] + acc[ng][1][0];
            r0p[1] = acc[ng][0][1] + acc[ng][1][1];
            r1p[0] = acc[ng][0][2] + acc[ng][1][2];
            r1p[1] = acc[ng][0][3] + acc[ng][1][3];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar + 16 + 8 * (jl & 1));
        base += units;
    }
#ifdef APB_TIMELINE
    if (lane == 0 && g_warpstat) {  // [total, in-unit loop, load wait, table wait, units]
        unsigned long long* st = g_warpstat + ((size_t)blockIdx.x * 16 + warp) * 8;
        st[0] = clock64() - clk_start;
        st[1] = clk_units;
        st[2] = clk_ldwait;
        st[3] = clk_tblwait;
        st[4] = n_done;
    }
#endif
}

// ---- v6: lean batch <= 8 kernel ---------------------------------------------
// Same roles, tables, hand-offs and arithmetic (bit-identical results) as the
// v5 kernel above, with a compute loop stripped to the essential instruction
// stream per lane word: k plane words -> bit network -> PRMT + LDS per lookup
// -> HMMA.  Differences: activations always come from shared memory and every
// lane loads its B fragment (columns n >= m_x are never read back, so no
// zeroing); rows past the layer end are clamped onto its last row instead of
// predicated (their outputs are never stored); the plane walker keeps one
// 64-bit pointer plus 32-bit offsets.
template <int K, int UB>
struct G6 {
    static constexpr int kTotalWarps = K >= 7 ? 12 : 16;
    static constexpr int kServiceWarps = 2;
    static constexpr int kWC = kTotalWarps - kServiceWarps;
    static constexpr int kThreads = kTotalWarps * 32;
    static constexpr int kUPT = 128 / (4 * UB);  // units per tile
    static constexpr int kLgUPT = kUPT == 2 ? 1 : (kUPT == 4 ? 2 : 3);
    static constexpr int kWPU = UB / 4;          // lane words per unit per row
    static constexpr int kSlotStride = 64 * 1024;
    // table slots: 3 where they fit next to the rest (more slack between a
    // table's build and its first use), else 2
#ifndef APB_SLOTS3_MAXB
#define APB_SLOTS3_MAXB (32 * 1024)
#endif
    static constexpr int kSlots = TableGeom<K>::kBytes <= APB_SLOTS3_MAXB ? 3 : 2;
    static constexpr int kRedBytes = kWC * kRowsPerCta * 8 * 4;  // one slot
    static constexpr int kRed = (kSlots - 1) * kSlotStride + TableGeom<K>::kBytes;
    static constexpr int kXs = kRed + kSlots * kRedBytes;
    static constexpr int kXmStride = 4 * kWPU * 64 + 64;  // x bytes per (unit, batch row)
    __host__ __device__ static int64_t xs_bytes(int64_t padded, int m_x) {
        return padded / (4 * UB * 8) * m_x * kXmStride;
    }
    __host__ __device__ static size_t bars(int64_t xs_bytes) { return (size_t)kXs + 2 * (size_t)((xs_bytes + 127) / 128 * 128); }
    __host__ __device__ static size_t total(int64_t xs_bytes) { return bars(xs_bytes) + 16 * kSlots; }
};

template <int K, int UB>
__global__ void __launch_bounds__(G6<K, UB>::kThreads, 1) gemv6_kernel(const __grid_constant__ GemvLaunch L) {
    using V = UnitVec<UB>;
    using VT = typename V::T;
    using G = G6<K, UB>;
    constexpr int WC = G::kWC, UPT = G::kUPT, LG = G::kLgUPT, WPU = G::kWPU;

    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3;
    if (smem_addr(smem) != APB_SMEM_BASE) __trap();  // see lds_table

    const int first = item_at_cost(L, L.total_cost * (int64_t)blockIdx.x / gridDim.x);
    const int last = item_at_cost(L, L.total_cost * (int64_t)(blockIdx.x + 1) / gridDim.x);
    asm volatile("griddepcontrol.launch_dependents;");
    if (first >= last) return;
    const int n_local = last - first;

    float* const red = reinterpret_cast<float*>(smem + G::kRed);  // [2][WC][16][8]
    const int64_t xs_slot = (L.xs_bytes + 127) / 128 * 128;
    uint8_t* const xs = smem + G::kXs;
    const uint32_t bar = smem_addr(smem + G::bars(L.xs_bytes));
    constexpr int NS = G::kSlots;
    // bar + 8s: table_ready[s] (count = service warps); bar + 8(NS + s): item_done[s]
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            mbar_init(bar + 8 * i, G::kServiceWarps);
            mbar_init(bar + 8 * (NS + i), WC);
        }
    }
    __syncthreads();

    if (warp >= WC) {
#ifndef APB_PF
#define APB_PF 1
#endif
        service_role<K, G::kServiceWarps, WC, 8, true, UB, NS, APB_PF ? K : 0>(L, first, last, smem, bar, red, xs, xs_slot,
                                                                  tid - WC * 32, G::kSlotStride);
        return;
    }

    // ---- plane walker: next unit (item lj, unit lv) this warp loads ----
    int lj = 0, lv = warp, lpi = problem_of(L, first), lpend = problem_end(L, lpi), lU = 0;
    uint32_t lps = 0;
    int32_t ld1 = 0;
    const uint8_t* lb0 = nullptr;
    auto lset = [&](int item) {
        const GemvProblem& P = L.prob[lpi];
        lU = P.n_tiles * UPT;
        lps = (uint32_t)P.plane_stride;
        const int64_t r0 = (int64_t)(item - P.item_begin) * kRowsPerCta + g;
        const int64_t ra = r0 < P.rows ? r0 : P.rows - 1;
        const int64_t rb = r0 + 8 < P.rows ? r0 + 8 : P.rows - 1;
        lb0 = P.planes + ra * P.row_bytes + q * UB;
        ld1 = (int32_t)((rb - ra) * P.row_bytes);
    };
    lset(first);
    bool ldone = false;
    auto lnorm = [&]() {
#pragma unroll 1
        while (lv >= lU) {
            lv -= lU;
            if (++lj >= n_local) {
                ldone = true;
                return;
            }
            const int item = first + lj;
            if (item >= lpend) {
                ++lpi;
#pragma unroll 1
                while (item >= problem_end(L, lpi)) ++lpi;
                lpend = problem_end(L, lpi);
            }
            lset(item);
        }
    };
    lnorm();
    auto lload = [&](VT(&dst)[2][K]) {
        if (ldone) return;
        const uint8_t* p0 = lb0 + (((uint32_t)lv >> LG) * (uint32_t)kTileBytes + ((uint32_t)lv & (UPT - 1)) * (4u * UB));
        const uint8_t* p1 = p0 + ld1;
#pragma unroll
        for (int p = 0; p < K; ++p) {
            dst[0][K - 1 - p] = V::load(p0);
            dst[1][K - 1 - p] = V::load(p1);
            p0 += lps;
            p1 += lps;
        }
        lv += WC;
        lnorm();
    };

    VT bufA[2][K], bufB[2][K];
    lload(bufA);
    lload(bufB);

    // B fragment: only lanes whose batch column n = g is real load x; the
    // others keep don't-care registers (MMA columns are independent and
    // columns n >= m_x are never read back)
    const uint32_t xlive = g < L.m_x ? 1u : 0u;
    int cpi = problem_of(L, first), cpend = problem_end(L, cpi), xb = 0;
    int U = L.prob[cpi].n_tiles * UPT;
    int gu = warp, ring = 0;
#pragma unroll 1
    for (int jl = 0; jl < n_local; ++jl) {
        const int item = first + jl;
        if (item >= cpend) {
            cpi = problem_of(L, item);
            cpend = problem_end(L, cpi);
            xb ^= 1;
            U = L.prob[cpi].n_tiles * UPT;
        }
        const uint32_t xrow = smem_addr(xs + xb * xs_slot) + (uint32_t)g * G::kXmStride + (uint32_t)q * 16u;
        const uint32_t xustride = (uint32_t)L.m_x * G::kXmStride;
        const int sl = jl % NS;
        const uint32_t off0 = ((uint32_t)sl << 16) | ((uint32_t)lane * 4u), off1 = off0 + 128u;
        float acc[2][4];
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) acc[c2][0] = acc[c2][1] = acc[c2][2] = acc[c2][3] = 0.f;

        auto unit = [&](int u, const VT(&buf)[2][K]) {
            // lane word t = s*UB + q*WPU + wi of tile `tile`; x columns 256p + 8t + 0..7
            const uint32_t xa = xrow + (uint32_t)u * xustride;
#pragma unroll
            for (int wi = 0; wi < WPU; ++wi) {
                uint4 xv[4];
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    xv[p] = make_uint4(0, 0, 0, 0);
                    lds128_pred(xv[p], xa + (p * WPU + wi) * 64, xlive);
                }
                uint32_t Q0[K], Q1[K];
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    Q0[i] = V::word(buf[0][i], wi);
                    Q1[i] = V::word(buf[1][i], wi);
                }
                uint32_t a0[16], a1[16];
                decode_word<K>(Q0, off0, a0);
                decode_word<K>(Q1, off1, a1);
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj)
                        mma16816(acc[p & 1], a0[p * 4 + 2 * jj], a1[p * 4 + 2 * jj], a0[p * 4 + 2 * jj + 1],
                                 a1[p * 4 + 2 * jj + 1], u4_word(xv[p], 2 * jj), u4_word(xv[p], 2 * jj + 1));
            }
        };

        mbar_wait(bar + 8 * sl, (jl / NS) & 1);  // this item's table (and x) ready
#pragma unroll 1
        for (; gu < U; gu += WC) {
            if (ring) {
                unit(gu, bufB);
                lload(bufB);
            } else {
                unit(gu, bufA);
                lload(bufA);
            }
            ring ^= 1;
        }
        gu -= U;
        float* r = red + sl * (WC * kRowsPerCta * 8) + (warp * kRowsPerCta + g) * 8 + 2 * q;
        r[0] = acc[0][0] + acc[1][0];
        r[1] = acc[0][1] + acc[1][1];
        r[8 * 8] = acc[0][2] + acc[1][2];
        r[8 * 8 + 1] = acc[0][3] + acc[1][3];
        __syncwarp();
        if (lane == 0) mbar_arrive(bar + 8 * (NS + sl));
    }
}

template <int K, int UB>
static int launch6(const GemvLaunch& L, cudaStream_t s);

constexpr int64_t kMaxXsBytes = 48 * 1024;
constexpr size_t kSmemLimitBytes = 227 * 1024;

static int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cached[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cached[dev] = n;
    }
    return cached[dev];
}

template <int K, int NG, int UB, bool XS>
static int launch_variant(const GemvLaunch& L, cudaStream_t s) {
    using LY = WsLayout<K, NG>;
    auto kern = gemv_kernel<K, NG, UB, XS>;
    static std::atomic<unsigned long long> configured{0};
    {
        size_t max_smem = LY::total(XS ? kMaxXsBytes : 0);
        if (max_smem > kSmemLimitBytes) max_smem = kSmemLimitBytes;
        if (!apb::ensure_smem_optin(kern, (int)max_smem, configured)) return APB_ERR_CUDA;
    }
    const size_t smem = LY::total(XS ? L.xs_bytes : 0);
    if (smem > kSmemLimitBytes) return APB_ERR_PARAM;
    int grid = sm_count();
    if (grid > L.n_items) grid = L.n_items;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)WsGeom<K, NG>::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (L.flags & APB_FLAG_PDL) ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, kern, L) != cudaSuccess) return APB_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

template <int K>
constexpr int unit_bytes() {
    return K <= 3 ? 16 : 8;
}

constexpr size_t kSmemLimit = 227 * 1024;

template <int K, int UB>
static int launch6(const GemvLaunch& L, cudaStream_t s) {
    using G = G6<K, UB>;
    auto kern = gemv6_kernel<K, UB>;
    static std::atomic<unsigned long long> configured{0};
    if (!apb::ensure_smem_optin(kern, (int)kSmemLimitBytes, configured)) return APB_ERR_CUDA;
    const size_t smem = G::total(L.xs_bytes);
    int grid = sm_count();
    if (grid > L.n_items) grid = L.n_items;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)G::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (L.flags & APB_FLAG_PDL) ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, kern, L) != cudaSuccess) return APB_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

template <int K, int NG>
static int dispatch_xs(GemvLaunch& L, cudaStream_t s) {
    if constexpr (NG == 1) {
        if (L.m_x <= 8) {  // the lean v6 kernel; v5 serves the 16-row chunks of larger batches
            using G = G6<K, unit_bytes<K>()>;
            GemvLaunch L6 = L;
            int64_t mp = 0;
            for (int i = 0; i < L.n_prob; ++i)
                mp = L.prob[i].n_tiles > mp ? L.prob[i].n_tiles : mp;
            L6.xs_bytes = G::xs_bytes(mp * kTileWeights, L.m_x);
            if (G::total(L6.xs_bytes) <= kSmemLimit) return launch6<K, unit_bytes<K>()>(L6, s);
        }
        // activations in shared memory when both buffers fit next to the tables
        if (L.xs_bytes > 0 && L.xs_bytes <= kMaxXsBytes && WsLayout<K, NG>::total(L.xs_bytes) <= kSmemLimit)
            return launch_variant<K, NG, unit_bytes<K>(), true>(L, s);
    }
    L.xs_bytes = 0;
    return launch_variant<K, NG, unit_bytes<K>(), false>(L, s);
}

template <int K>
static int dispatch_ng(int ng, GemvLaunch& L, cudaStream_t s) {
    switch (ng) {
        case 1: return dispatch_xs<K, 1>(L, s);
        case 2: return dispatch_xs<K, 2>(L, s);
        default: return dispatch_xs<K, 4>(L, s);
    }
}

}  // namespace apb

using namespace apb;

static int gemv_launch_chunk(int n, const uint8_t* const* planes, const int64_t* rows,
                             const int64_t* cols, const int64_t* padded, int k,
                             const uint16_t* const* lut, const uint16_t* const* x, int m_x,
                             const int64_t* ldx, int64_t x_off, int x_split, void* const* y,
                             int y_dtype, const int64_t* ldy, int64_t y_off, int flags,
                             cudaStream_t s, int m_x_total) {
    GemvLaunch L;
    L.flags = flags;
    L.n_prob = n;
    L.m_x = m_x;
    L.x_split = x_split;
    L.y_f16 = y_dtype == APB_DTYPE_F16;
    int items = 0;
    int64_t cost = 0, max_padded = 0;
    const int esz = y_dtype == APB_DTYPE_F16 ? 2 : 4;
    for (int i = 0; i < n; ++i) {
        GemvProblem& P = L.prob[i];
        P.planes = planes[i];
        P.lut = lut[i];
        P.x = x[i] + x_off * ldx[i];
        // scaled pairs: the inverse scales follow the whole [m_x_total][ldx] block
        P.xinv = x_split == 2 ? reinterpret_cast<const float*>(x[i] + (int64_t)m_x_total * ldx[i]) + x_off / 2 : nullptr;
        P.y = reinterpret_cast<uint8_t*>(y[i]) + y_off * ldy[i] * esz;
        P.rows = rows[i];
        P.cols = cols[i];
        P.row_bytes = padded[i] / 8;
        P.plane_stride = rows[i] * (padded[i] / 8);
        P.ldx = ldx[i];
        P.ldy = ldy[i];
        P.n_tiles = (int)(padded[i] / kTileWeights);
        P.item_begin = items;
        P.cost_begin = cost;
        const int n_items = (int)((rows[i] + kRowsPerCta - 1) / kRowsPerCta);
        items += n_items;
        cost += (int64_t)n_items * P.n_tiles;
        if (padded[i] > max_padded) max_padded = padded[i];
    }
    L.n_items = items;
    L.total_cost = cost;
    const int ng = m_x <= 8 ? 1 : (m_x <= 16 ? 2 : 4);
    L.xs_bytes = (int64_t)m_x * max_padded * 2;  // per buffer; dispatch decides if it fits
    switch (k) {
        case 2: return dispatch_ng<2>(ng, L, s);
        case 3: return dispatch_ng<3>(ng, L, s);
        case 4: return dispatch_ng<4>(ng, L, s);
        case 5: return dispatch_ng<5>(ng, L, s);
        case 6: return dispatch_ng<6>(ng, L, s);
        case 7: return dispatch_ng<7>(ng, L, s);
        case 8: return dispatch_ng<8>(ng, L, s);
    }
    return APB_ERR_PARAM;
}

extern "C" int apb7_try_gemv(int n, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
                             const int64_t* cols, const int64_t* padded, int k, const uint16_t* const* lut,
                             const uint16_t* const* x, int m_x, const int64_t* ldx, int64_t x_off, int x_split,
                             void* const* y, int y_dtype, const int64_t* ldy, int64_t y_off, int flags, void* stream, int n_peers,
                             void* const* y_peers, uint32_t* const* peer_flags,
                             const apb_norm_epilogue* norm);

extern "C" int apb_gemv_grouped(int n_problems, const uint8_t* const* planes, const int* n_max,
                                const int64_t* rows, const int64_t* cols,
                                const int64_t* padded_cols, int k, const uint16_t* const* lut,
                                const uint16_t* const* x, int m_x, const int64_t* ldx, int x_split,
                                void* const* y, int y_dtype, const int64_t* ldy, int flags,
                                void* stream) {
    if (n_problems < 1) return APB_ERR_SHAPE;
    if (k < 2 || k > 8) return APB_ERR_PARAM;
    if (y_dtype != APB_DTYPE_F32 && y_dtype != APB_DTYPE_F16) return APB_ERR_PARAM;
    if (x_split < 0 || x_split > 2) return APB_ERR_PARAM;
    if (m_x < 1 || (x_split && (m_x & 1))) return APB_ERR_SHAPE;
    const bool glu = (flags & APB_FLAG_GLU) != 0;
    for (int i = 0; i < n_problems; ++i) {
        if (rows[i] <= 0 || cols[i] <= 0 || (glu && (rows[i] & 1))) return APB_ERR_SHAPE;
        if (padded_cols[i] != apb_pad_columns(cols[i])) return APB_ERR_SHAPE;
        if (k > n_max[i] || n_max[i] > 8) return APB_ERR_PARAM;
        if (ldx[i] < cols[i] || (ldx[i] % 8) != 0) return APB_ERR_PARAM;
        if (!planes[i] || !lut[i] || !x[i] || !y[i]) return APB_ERR_PARAM;
        if (((uintptr_t)x[i] & 15) != 0 || ((uintptr_t)planes[i] & 15) != 0) return APB_ERR_PARAM;
        if (((uintptr_t)lut[i] & 15) != 0) return APB_ERR_PARAM;
        if (ldy[i] < (glu ? rows[i] / 2 : rows[i])) return APB_ERR_SHAPE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (m_x <= 16 && n_problems <= 16) {  // TMA-fed kernel (apb_gemv7.cu)
        const int rc = apb7_try_gemv(n_problems, planes, n_max, rows, cols, padded_cols, k, lut, x, m_x, ldx, 0,
                                     x_split, y, y_dtype, ldy, 0, flags, stream, 0, nullptr, nullptr, nullptr);
        if (rc != -1) return rc;
    }
    if (glu) return APB_ERR_PARAM;  // the gate/up epilogue exists on the TMA kernel only
    // batch columns per launch: 32 fp16 activation rows (4 mma column groups)
    const int chunk = 32;
    for (int p0 = 0; p0 < n_problems; p0 += kMaxGroup) {
        const int n = n_problems - p0 < kMaxGroup ? n_problems - p0 : kMaxGroup;
        for (int m0 = 0; m0 < m_x; m0 += chunk) {
            const int mc = m_x - m0 < chunk ? m_x - m0 : chunk;
            const int rc = gemv_launch_chunk(n, planes + p0, rows + p0, cols + p0, padded_cols + p0, k,
                                             lut + p0, x + p0, mc, ldx + p0, m0, x_split, y + p0,
                                             y_dtype, ldy + p0, x_split ? m0 / 2 : m0, flags, s, m_x);
            if (rc != APB_OK) return rc;
        }
    }
    return APB_OK;
}

extern "C" void* apb7_plan_create(int n, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
                                  const int64_t* cols, const int64_t* padded, int k, const uint16_t* const* lut,
                                  const uint16_t* const* x, int m_x, const int64_t* ldx, int x_split, void* const* y,
                                  int y_dtype, const int64_t* ldy, int flags);

// Caller-owned launch plan (apb_gemv_plan_create / _launch / _destroy): the
// arguments of apb_gemv_grouped validated and prepared once; NULL when the call
// is not served by the TMA kernel (use apb_gemv_grouped then).
extern "C" void* apb_gemv_plan_create(int n_problems, const uint8_t* const* planes, const int* n_max,
                                      const int64_t* rows, const int64_t* cols, const int64_t* padded_cols, int k,
                                      const uint16_t* const* lut, const uint16_t* const* x, int m_x,
                                      const int64_t* ldx, int x_split, void* const* y, int y_dtype,
                                      const int64_t* ldy, int flags) {
    if (n_problems < 1 || n_problems > 16 || k < 3 || k > 8) return nullptr;
    if (y_dtype != APB_DTYPE_F32 && y_dtype != APB_DTYPE_F16) return nullptr;
    if (x_split < 0 || x_split > 2 || m_x < 1 || m_x > 16 || (x_split && (m_x & 1))) return nullptr;
    const bool glu = (flags & APB_FLAG_GLU) != 0;
    for (int i = 0; i < n_problems; ++i) {
        if (rows[i] <= 0 || cols[i] <= 0 || (glu && (rows[i] & 1))) return nullptr;
        if (padded_cols[i] != apb_pad_columns(cols[i])) return nullptr;
        if (k > n_max[i] || n_max[i] > 8) return nullptr;
        if (ldx[i] < cols[i] || (ldx[i] % 8) != 0) return nullptr;
        if (!planes[i] || !lut[i] || !x[i] || !y[i]) return nullptr;
        if (((uintptr_t)x[i] & 15) != 0 || ((uintptr_t)planes[i] & 15) != 0 || ((uintptr_t)lut[i] & 15) != 0)
            return nullptr;
        if (ldy[i] < (glu ? rows[i] / 2 : rows[i])) return nullptr;
    }
    return apb7_plan_create(n_problems, planes, n_max, rows, cols, padded_cols, k, lut, x, m_x, ldx, x_split, y,
                            y_dtype, ldy, flags);
}

// Row-sharded GEMV with the all-gather fused into the epilogue:
// the grouped GEMV of this rank's row slab, every y value also stored into the
// same place of each peer's output (y_peers[i * n_peers + j]: problem i's y as
// mapped from peer j, e.g. through CUDA IPC), and each CTA adding the number of
// values it wrote to every rank's arrival counter (peer_flags[0..n_peers-1] the
// peers', peer_flags[n_peers] this rank's own).  apb_peer_wait completes it.
extern "C" int apb_gemv_grouped_peers(int n_problems, const uint8_t* const* planes, const int* n_max,
                                      const int64_t* rows, const int64_t* cols, const int64_t* padded_cols, int k,
                                      const uint16_t* const* lut, const uint16_t* const* x, int m_x,
                                      const int64_t* ldx, int x_split, void* const* y, int y_dtype,
                                      const int64_t* ldy, int n_peers, void* const* y_peers,
                                      uint32_t* const* peer_flags, int flags, void* stream) {
    if (n_problems < 1) return APB_ERR_SHAPE;
    if (k < 3 || k > 8) return APB_ERR_PARAM;  // the TMA kernel's range
    if (y_dtype != APB_DTYPE_F32 && y_dtype != APB_DTYPE_F16) return APB_ERR_PARAM;
    if (x_split < 0 || x_split > 2) return APB_ERR_PARAM;
    if (m_x < 1 || m_x > 16 || n_problems > 16 || (x_split && (m_x & 1))) return APB_ERR_SHAPE;
    if (n_peers < 0 || n_peers > 7 || (n_peers > 0 && !y_peers) || !peer_flags) return APB_ERR_PARAM;
    for (int j = 0; j <= n_peers; ++j)
        if (!peer_flags[j] || ((uintptr_t)peer_flags[j] & 3)) return APB_ERR_PARAM;
    for (int i = 0; i < n_problems; ++i) {
        if (rows[i] <= 0 || cols[i] <= 0) return APB_ERR_SHAPE;
        if (padded_cols[i] != apb_pad_columns(cols[i])) return APB_ERR_SHAPE;
        if (k > n_max[i] || n_max[i] > 8) return APB_ERR_PARAM;
        if (ldx[i] < cols[i] || (ldx[i] % 8) != 0) return APB_ERR_PARAM;
        if (!planes[i] || !lut[i] || !x[i] || !y[i]) return APB_ERR_PARAM;
        if (((uintptr_t)x[i] & 15) != 0 || ((uintptr_t)planes[i] & 15) != 0) return APB_ERR_PARAM;
        if (((uintptr_t)lut[i] & 15) != 0) return APB_ERR_PARAM;
        if ((flags & APB_FLAG_GLU) && (rows[i] & 1)) return APB_ERR_SHAPE;
        if (ldy[i] < ((flags & APB_FLAG_GLU) ? rows[i] / 2 : rows[i])) return APB_ERR_SHAPE;
        for (int j = 0; j < n_peers; ++j)
            if (!y_peers[(size_t)i * n_peers + j]) return APB_ERR_PARAM;
    }
    const int rc = apb7_try_gemv(n_problems, planes, n_max, rows, cols, padded_cols, k, lut, x, m_x, ldx, 0,
                                 x_split, y, y_dtype, ldy, 0, flags, stream, n_peers, y_peers, peer_flags,
                                 nullptr);
    return rc == -1 ? APB_ERR_PARAM : rc;  // e.g. more than 64K columns: not on the fused path
}

// Decode-step RMSNorm folded into the GEMV epilogues (see apb_norm_epilogue).
extern "C" int apb_gemv_grouped_norm(int n_problems, const uint8_t* const* planes, const int* n_max,
                                     const int64_t* rows, const int64_t* cols, const int64_t* padded_cols, int k,
                                     const uint16_t* const* lut, const uint16_t* const* x, int m_x,
                                     const int64_t* ldx, void* const* y, int y_dtype, const int64_t* ldy,
                                     const apb_norm_epilogue* norm, int flags, void* stream) {
    if (!norm || norm->mode < 0 || norm->mode > 2) return APB_ERR_PARAM;
    if (n_problems < 1 || n_problems > 16) return APB_ERR_SHAPE;
    if (k < 3 || k > 8 || (y_dtype != APB_DTYPE_F16 && y_dtype != APB_DTYPE_F32)) return APB_ERR_PARAM;
    if (m_x < 1 || m_x > 16) return APB_ERR_SHAPE;
    const bool glu = (flags & APB_FLAG_GLU) != 0;
    if (norm->mode == 1) {  // producer: one batch row, one problem, fp16 normalised output
        if (m_x != 1 || n_problems != 1 || glu || y_dtype != APB_DTYPE_F16) return APB_ERR_PARAM;
        if (!norm->resid || !norm->norm_w || !norm->partials) return APB_ERR_PARAM;
        if (norm->n_partials < 1) return APB_ERR_PARAM;  // checked against the launch grid later
    }
    if (norm->mode == 2 && (!norm->partials || norm->n_partials <= 0 || norm->norm_size <= 0))
        return APB_ERR_PARAM;
    for (int i = 0; i < n_problems; ++i) {
        if (rows[i] <= 0 || cols[i] <= 0 || (glu && (rows[i] & 1))) return APB_ERR_SHAPE;
        if (padded_cols[i] != apb_pad_columns(cols[i])) return APB_ERR_SHAPE;
        if (k > n_max[i] || n_max[i] > 8) return APB_ERR_PARAM;
        if (ldx[i] < cols[i] || (ldx[i] % 8) != 0) return APB_ERR_PARAM;
        if (!planes[i] || !lut[i] || !x[i] || !y[i]) return APB_ERR_PARAM;
        if (((uintptr_t)x[i] & 15) != 0 || ((uintptr_t)planes[i] & 15) != 0) return APB_ERR_PARAM;
        if (((uintptr_t)lut[i] & 15) != 0) return APB_ERR_PARAM;
        if (ldy[i] < (glu ? rows[i] / 2 : rows[i])) return APB_ERR_SHAPE;
    }
    const int rc = apb7_try_gemv(n_problems, planes, n_max, rows, cols, padded_cols, k, lut, x, m_x, ldx, 0, 0, y,
                                 y_dtype, ldy, 0, flags, stream, 0, nullptr, nullptr, norm);
    return rc == -1 ? APB_ERR_PARAM : rc;
}

#ifdef APB_TIMELINE
extern "C" int apb_debug_set_timeline(unsigned long long* p) {
    return cudaMemcpyToSymbol(g_timeline, &p, sizeof(p)) == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}
extern "C" int apb_debug_set_warpstat(unsigned long long* p) {
    return cudaMemcpyToSymbol(g_warpstat, &p, sizeof(p)) == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}
#endif

extern "C" int apb_gemv(const uint8_t* planes, int n_max, int64_t rows, int64_t cols,
                        int64_t padded_cols, int k, const uint16_t* lut, const uint16_t* x, int m_x,
                        int64_t ldx, int x_split, void* y, int y_dtype, int64_t ldy, int flags,
                        void* stream) {
    return apb_gemv_grouped(1, &planes, &n_max, &rows, &cols, &padded_cols, k, &lut, &x, m_x, &ldx,
                            x_split, &y, y_dtype, &ldy, flags, stream);
}

// SURVEY 8(b) names.  Small-batch GEMM (engine.py:312-341, M <= dense
// threshold): the quantized kernel over M activation rows.
extern "C" int apb_gemm_small(const uint8_t* planes, int n_max, int64_t rows, int64_t cols, int64_t padded_cols,
                              int k, const uint16_t* lut, int m, const uint16_t* X, int64_t ldx, void* Y,
                              int y_dtype, int64_t ldy, void* stream) {
    return apb_gemv(planes, n_max, rows, cols, padded_cols, k, lut, X, m, ldx, 0, Y, y_dtype, ldy, 0, stream);
}

// Row-sharded GEMV + all-gather of one layer: this rank's slab
// [row_offset, row_offset + rows) of a [m][ldy] output, written into every
// rank's output (y_ranks[r]: rank r's output as mapped here) with the arrival
// counters flag_ranks[r]; complete it with apb_peer_wait on flag_ranks[rank].
extern "C" int apb_gemv_allgather(const uint8_t* planes, int n_max, int64_t rows, int64_t cols,
                                  int64_t padded_cols, int k, const uint16_t* lut, const uint16_t* x, int m_x,
                                  int64_t ldx, int rank, int world, void* const* y_ranks, int64_t row_offset,
                                  int y_dtype, int64_t ldy, uint32_t* const* flag_ranks, int flags, void* stream) {
    if (world < 1 || world > 8 || rank < 0 || rank >= world || !y_ranks || !flag_ranks || row_offset < 0)
        return APB_ERR_PARAM;
    const int64_t esz = y_dtype == APB_DTYPE_F16 ? 2 : 4;
    void* own = static_cast<uint8_t*>(y_ranks[rank]) + row_offset * esz;
    void* peers[8];
    uint32_t* fl[9];
    int np = 0;
    for (int r = 0; r < world; ++r)
        if (r != rank) {
            if (!y_ranks[r]) return APB_ERR_PARAM;
            peers[np] = static_cast<uint8_t*>(y_ranks[r]) + row_offset * esz;
            fl[np++] = flag_ranks[r];
        }
    fl[np] = flag_ranks[rank];
    return apb_gemv_grouped_peers(1, &planes, &n_max, &rows, &cols, &padded_cols, k, &lut, &x, m_x, &ldx, 0, &own,
                                  y_dtype, &ldy, np, peers, fl, flags, stream);
}
