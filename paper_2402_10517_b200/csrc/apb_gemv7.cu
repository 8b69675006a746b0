// apb_gemv7.cu -- TMA-fed bitplane GEMV for batch <= 2 (sm_100a).
//
// Replaces engine.py:284-309 (gemv) and the M <= 2 case of engine.py:312-341
// (gemm, quantized path) of the reference: y[m][r] = sum_c LUT_k[r][code_k(r,c)]
// * x[m][c], reading ONLY planes 0..k-1 and the k-bit centroid table.
//
// Why a second kernel: the register-streaming kernels (apb_gemv.cu) load the
// planes with warp-wide LDGs that touch 8 rows x 32 B each, which keeps the
// L1 tag stage ~70 % busy at ~40 % of HBM bandwidth.  Here the planes never
// pass through the LSU: a producer thread streams them with TMA
// (cp.async.bulk.tensor, 3-D map {row bytes, rows, planes}, 128-B swizzle)
// into a ring of shared-memory stages, one stage = one 1024-column tile x 16
// rows x k planes, and the compute warps read them back with conflict-free
// LDS.128.  The centroid rows of each item are brought in the same way.
//
// Lane mapping ("row copies"): lane (g, q) of a compute warp owns row
// 2g + (q >> 1) of the 16-row item, copy q & 1.  Rows 2g / 2g+1 share one MMA
// row (g for columns set A, g + 8 for set B); the B operand is block-sparse:
// column 0 holds x on the k-slots of lanes q = 0,1 (row 2g, set A), column 1
// on those of q = 2,3 (row 2g+1), columns 2/3 likewise for set B, columns 4..7
// the same for the second batch row.  So every lane looks up ITS row only and
// a table needs 2 copies per row (one per lane) instead of 4 -- half the
// table bytes and build work of the 16-row mapping, with every lookup still
// bank-conflict free (bank = lane).
//
// Numerics are those of the other kernels: fp16 table entries, fp16
// activations, fp32 MMA accumulation, a fixed reduction order (per-warp
// partials summed in warp order) -> bit-reproducible.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/anyprec_b200.h"
#include "apb_common.cuh"

namespace apb7 {
using apb::kTileBytes;
using apb::kTileWeights;
using apb::prmt;

constexpr int kRows = 16;      // rows per item
constexpr int kMaxProb = 16;   // problems per grouped launch
constexpr int kMaxPeers = 8;   // fused all-gather: ranks of one NVSwitch node
constexpr int kMaxPartials = 320;  // RMSNorm epilogue: >= the largest grid (2 CTAs x 148 SMs)
constexpr int kSmemBase = 1024;  // sm_100 reserves the first 1 KB of the shared window
constexpr int kMaxCols = 64 * 1024;  // padded columns per layer on this path

// Zero activations: B-fragment lanes that must hold zeros read from here, so
// every lane issues the same unpredicated load (no divergence).
__device__ __align__(16) uint16_t g_zero_x[kMaxCols];

#ifdef APB_TIMELINE
// Debug builds (tools/kbench timeline / chain): per-launch, per-CTA globaltimer
// stamps (ns) at [launch % 64][block][8]; the launch index is a host-side
// counter carried in Launch7::tl_launch.
__device__ unsigned long long g_tl7[64 * 512 * 8];
#define tl_stamp(i)                                                                              \
    do {                                                                                         \
        unsigned long long t_;                                                                   \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
        g_tl7[((size_t)(L.tl_launch % 64) * 512 + blockIdx.x) * 8 + (i)] = t_;                  \
    } while (0)
#define APB_TL(i) tl_stamp(i)
#else
#define APB_TL(i) \
    do {          \
    } while (0)
#endif

struct Prob7 {
    const uint16_t* x;  // fp16 [m_x][ldx]
    void* y;            // [m_out][ldy]
    int64_t rows, cols, ldx, ldy;
    int n_tiles;
    int item_begin;
    int64_t cost_begin;
    int xid;  // problems with equal xid read the same activations (staged once)
    const float* xinv;  // x_split == 2: inverse activation scale per output batch row
};

struct alignas(64) Launch7 {
    CUtensorMap tm_planes[kMaxProb];  // 3-D {row_bytes, rows, n_max} u8, box {128, 16, 1}, 128B swizzle
    CUtensorMap tm_lut[kMaxProb];     // 2-D {2^k, rows} f16, box {min(2^k, 64), 16}
    Prob7 prob[kMaxProb];
    int n_prob, n_items;
    int64_t total_cost;
    int m_x, x_split, y_f16;
    int glu;           // APB_FLAG_GLU: interleaved (gate, up) rows -> silu(gate) * up
    // RMSNorm folded into the epilogues (apb_gemv_grouped_norm): 1 = producer
    // (resid += y; y_out = fp16(resid * norm_w); partials[cta] = sum resid^2),
    // 2 = consumer (row sums scaled by rsqrt(sum(partials) / norm_size + eps))
    int norm_mode, n_partials, norm_size;
    float norm_eps;
    float* resid;
    const __half* norm_w;
    float* partials;
    int n_stages;      // ring depth
    int64_t xs_bytes;  // one activation buffer
    int x_bufs;        // 1 when every problem shares one x, else 2
    int tl_launch;     // APB_TIMELINE builds: launch index
    // fused all-gather of row-sharded outputs: every y value is also stored at
    // the same offset of each peer's output (P2P over NVLink), and each CTA then
    // adds the number of y values it wrote to every peer's arrival counter
    int n_peers;
    uint8_t* y_peer[kMaxProb][kMaxPeers];
    uint32_t* peer_flag[kMaxPeers + 1];  // the n_peers others, then this rank's own
};

template <int K, int NB = 1, int CPS = 1>
struct Geo {
    static constexpr bool kPair = K <= 4;
    static constexpr int kEntries = kPair ? (1 << (2 * K)) : (1 << K);
    // NB == 4: "batch-in-N" mapping (lane owns rows g and g+8, 4 copies per row,
    // up to 8 batch rows in the MMA N dimension); its table is
    // [slot (64 KB stride)][entry][row-half 2][lane 32] u32.  Otherwise the
    // row-copy mapping: [entry][slot 2][lane 32] u32.
    static constexpr bool kMapN = NB >= 4;  // NB == 8: 16 batch rows, two MMAs per A fragment
    static constexpr int kTableBytes = kMapN ? 65536 + kEntries * 256 : kEntries * 256;
    static constexpr int kLutHalves = 1 << K;
    static constexpr int kLutBox = kLutHalves < 64 ? kLutHalves : 64;  // halves per box row
    static constexpr int kLutBoxes = kLutHalves / kLutBox;
    static constexpr int kLutBytes = kRows * kLutHalves * 2;
    static constexpr int kLutSlot = (kLutBytes + 1023) / 1024 * 1024;
    static constexpr int kStageBytes = K * 2048;  // 16 rows x 128 B x K planes
#ifdef APB7_WC
    static constexpr int kWC = APB7_WC;
#else
    // compute warps, groups of 4 (measured best per k; 8 for 4 batch pairs: registers;
    // 8 when two CTAs share an SM)
    static constexpr int kWC = NB == 8 ? 8 : (NB == 4 ? 12 : (CPS == 2 ? 8 : (K == 8 ? 12 : 16)));
#endif
    static constexpr int kNG = kWC / 4;
    static constexpr int kThreads = (kWC + 2) * 32;
    static constexpr int kRedBytes = 2 * kWC * 2 * NB * kRows * 4;  // [slot][warp][m][row] f32
    // layout: tables | lut x2 | ring | xs x2 | red | barriers
    static constexpr int kLut = (kTableBytes + 1023) / 1024 * 1024;
    static constexpr int kRing = kLut + 2 * kLutSlot;
    static size_t total(int n_stages, int64_t xs_total) {
        return (size_t)kRing + (size_t)n_stages * kStageBytes + (size_t)xs_total + kRedBytes + 16 * n_stages + 96;
    }
};

// ---- PTX helpers ---------------------------------------------------------------
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.shared::cta.b64 s, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;\n\t}" ::"r"(a),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(a),
        "r"(parity), "r"(1000000)
        : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in the barrier unit
// instead of spinning through issue slots other warps could use.
__device__ __forceinline__ void mbar_sleep(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra S_%=;\n\t}" ::"r"(a),
        "r"(parity), "r"(1000000)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds64_keep(uint32_t& v0, uint32_t& v1, uint32_t a, uint32_t pred) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t"
        "@p ld.shared.v2.u32 {%0,%1}, [%2];\n\t}"
        : "+r"(v0), "+r"(v1)
        : "r"(a), "r"(pred));
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
// Plane tiles are read exactly once per call: evict-first keeps them from
// displacing what IS reused from L2 (centroid rows, x, a decode step's KV cache).
#ifndef APB7_EVICT_FIRST
#define APB7_EVICT_FIRST 1
#endif
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma3_ef(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint32_t bar,
                                        uint64_t pol) {
#if APB7_EVICT_FIRST
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
        : "memory");
#else
    (void)pol;
    tma3(dst, m, c0, c1, c2, bar);
#endif
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(m), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// B-fragment load: executed only where pred != 0; other lanes keep their
// (zero) registers -- the B operand is block-sparse by construction.
__device__ __forceinline__ void lds128_keep(uint32_t& v0, uint32_t& v1, uint32_t& v2, uint32_t& v3, uint32_t a,
                                            uint32_t pred) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t"
        "@p ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
        : "+r"(v0), "+r"(v1), "+r"(v2), "+r"(v3)
        : "r"(a), "r"(pred));
}
// B-fragment load from global (read-only path): only where pred != 0.
__device__ __forceinline__ void ldg64_keep(uint32_t& v0, uint32_t& v1, const void* p, uint32_t pred) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t"
        "@p ld.global.nc.v2.u32 {%0,%1}, [%2];\n\t}"
        : "+r"(v0), "+r"(v1)
        : "l"(p), "r"(pred));
}
__device__ __forceinline__ uint32_t u4w(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
__device__ __forceinline__ uint32_t lds_table(uint32_t off) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+1024];" : "=r"(v) : "r"(off));
    return v;
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(src_bytes));
}

__device__ __forceinline__ int problem_of(const Launch7& L, int item) {
    int pi = 0;
#pragma unroll 1
    for (int i = 1; i < L.n_prob; ++i)
        if (item >= L.prob[i].item_begin) pi = i;
    return pi;
}
__device__ __forceinline__ int problem_end(const Launch7& L, int pi) {
    return pi + 1 < L.n_prob ? L.prob[pi + 1].item_begin : L.n_items;
}
__device__ __forceinline__ int item_at_cost(const Launch7& L, int64_t target) {
    if (target >= L.total_cost) return L.n_items;
#pragma unroll 1
    for (int i = 0; i < L.n_prob; ++i) {
        const Prob7& P = L.prob[i];
        const int n = problem_end(L, i) - P.item_begin;
        const int64_t end = P.cost_begin + (int64_t)n * P.n_tiles;
        if (target < end) return P.item_begin + (int)((target - P.cost_begin + P.n_tiles - 1) / P.n_tiles);
    }
    return L.n_items;
}

// Decode one lane word into 16 fp16x2 A values: out[p*4 + j] = weights of
// columns (256p + 8t + 2j, +1) of this lane's row (apb_common.cuh networks).
template <int K>
__device__ __forceinline__ void decode_word(const uint32_t* Q, uint32_t off, uint32_t* out) {
    if constexpr (Geo<K>::kPair) {
        uint32_t U[4];
        apb::to_pairs<K>(Q, U);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) out[p * 4 + j] = lds_table(prmt(U[j], off, 0x7604u | (uint32_t)(p << 4)));
    } else {
        uint32_t Wb[8];
        apb::to_bytes<K>(Q, Wb);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const uint32_t sel = 0x7604u | (uint32_t)(p << 4);
                const uint32_t e = lds_table(prmt(Wb[2 * j], off, sel));
                const uint32_t o = lds_table(prmt(Wb[2 * j + 1], off, sel));
                out[p * 4 + j] = e + (o << 16);  // entries are (v, 0): one IMAD packs the pair
            }
    }
}

// NB = batch pairs per launch (m_x <= 2 NB).  NB = 1 stages x in shared memory;
// NB > 1 (small-batch GEMM, engine.py:312-341 with M <= 8) reads its B
// fragments from global memory (L1 / L2 resident) so x never limits smem.
// EPI: the epilogue features (GLU, RMSNorm fold, fused all-gather) are compiled
// in; plain launches use the EPI = false instantiation, whose reduce is exactly
// the plain one (measured: the unused branches cost small launches ~2-3 %).
template <int K, int NB, int CPS, bool EPI>
__global__ void __launch_bounds__(Geo<K, NB, CPS>::kThreads, CPS) gemv7_kernel(const __grid_constant__ Launch7 L) {
    using G = Geo<K, NB, CPS>;
    constexpr int WC = G::kWC, NG = G::kNG;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ep_glu = EPI ? L.glu : 0, ep_norm = EPI ? L.norm_mode : 0, ep_peers = EPI ? L.n_peers : -1;
    if (saddr(smem) != kSmemBase) __trap();  // lds_table folds the table base into the immediate

    const int first = item_at_cost(L, L.total_cost * (int64_t)blockIdx.x / gridDim.x);
    const int last = item_at_cost(L, L.total_cost * (int64_t)(blockIdx.x + 1) / gridDim.x);
    asm volatile("griddepcontrol.launch_dependents;");
    if (first >= last) {
        // RMSNorm producer: the consumer sums ALL n_partials slots, so a CTA
        // without items still writes its (zero) share -- after the PDL wait: a
        // consumer of the previous producer may read the slot until then
        if (EPI && L.norm_mode == 1) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            if (tid == 0) __stcg(L.partials + blockIdx.x, 0.f);
        }
        return;
    }
    if (tid == 0) APB_TL(0);
    const int n_local = last - first;
    const int NST = L.n_stages;

    const uint32_t s_lut = saddr(smem + G::kLut);
    const uint32_t s_ring = saddr(smem + G::kRing);
    uint8_t* const xs = smem + G::kRing + (size_t)NST * G::kStageBytes;  // [2][m_x][padded] fp16
    float* const red = reinterpret_cast<float*>(xs + L.x_bufs * L.xs_bytes);
    const uint32_t bar = saddr(reinterpret_cast<uint8_t*>(red) + G::kRedBytes);
    // spare word after the barriers: the consumer RMSNorm factor (norm_mode 2),
    // computed by compute warp 0 while x is in flight, read by the service warp
    float* const s_norm = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(red) + G::kRedBytes + 16 * NST + 80);
    // the producer's per-CTA sums of resid^2 -> rsqrt(mean + eps), fixed order (one warp)
    auto norm_factor = [&]() {
        float pv[kMaxPartials / 32];
#pragma unroll
        for (int u = 0; u < kMaxPartials / 32; ++u)
            pv[u] = lane + 32 * u < L.n_partials ? __ldcg(L.partials + lane + 32 * u) : 0.f;
        float acc = 0.f;
#pragma unroll
        for (int u = 0; u < kMaxPartials / 32; ++u) acc += pv[u];
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) *s_norm = rsqrtf(acc / (float)L.norm_size + L.norm_eps);
    };
    // barriers (8 B each): full[NST] | empty[NST] | lut_full[2] | lut_empty[2] | table_ready[2] | item_done[2] | x_full[2]
    const uint32_t b_full = bar, b_empty = bar + 8 * NST, b_lfull = bar + 16 * NST, b_lempty = b_lfull + 16,
                   b_tready = b_lfull + 32, b_idone = b_lfull + 48, b_xfull = b_lfull + 64;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(b_full + 8 * i, 1);
            mbar_init(b_empty + 8 * i, 4 * 32);  // every lane of the 4 consumer warps arrives
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(b_lfull + 8 * i, 1);
            mbar_init(b_lempty + 8 * i, 1);
            mbar_init(b_tready + 8 * i, 1);
            mbar_init(b_idone + 8 * i, WC * 32);
            mbar_init(b_xfull + 8 * i, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // activations of problem pi -> x buffer xb (one bulk copy per batch row;
    // columns past cols are masked by the compute warps).  One thread.
    auto issue_x_one = [&](int pi, int xb) {
        const Prob7& P = L.prob[pi];
        const uint32_t bytes = (uint32_t)((P.cols + 7) / 8 * 16);
        mbar_expect_tx(b_xfull + 8 * xb, bytes * L.m_x);
        for (int m = 0; m < L.m_x; ++m)
            bulk_g2s(saddr(xs + xb * L.xs_bytes) + m * P.n_tiles * 2048, P.x + (int64_t)m * P.ldx, bytes,
                     b_xfull + 8 * xb);
    };

    // Lookup-table build for item slot `slot` from its LUT slot.  The service warp
    // builds every table; the first one is built by the service and all compute
    // warps together (they are idle until it exists).
    // k >= 5: the first table (2^k single entries) is built by every compute warp
    // with the service warp (measured: shortens the launch; for the pair tables of
    // k <= 4 the extra code in the compute warps costs more than it saves)
    constexpr bool kCoopFirst = K >= 5 && !G::kMapN;
    // coop: std::true_type for the shared first build (entries split over nbw warps)
    auto build = [&](auto coop, int slot, int bw, int nbw) {  // builder bw of nbw warps
        constexpr bool kCoop = decltype(coop)::value;
        if constexpr (G::kMapN) {
            // rows gg (half 0) and gg+8 (half 1), 4 copies each: one STS.128 per (entry, half)
            const int e4 = lane >> 3, gg = lane & 7, r0 = gg, r1 = gg + 8;
            const uint32_t lut = s_lut + slot * G::kLutSlot;
            const uint32_t dst = saddr(smem) + slot * 65536 + gg * 16;
            if constexpr (G::kPair) {
                uint32_t h0[1 << K], h1[1 << K];
                constexpr int RB = (1 << K) * 2;
#pragma unroll
                for (int c = 0; c < RB / 16; ++c) {
                    const uint4 v0 = lds128(lut + r0 * RB + c * 16), v1 = lds128(lut + r1 * RB + c * 16);
                    const uint32_t a0[4] = {v0.x, v0.y, v0.z, v0.w}, a1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        h0[c * 8 + i] = (i & 1) ? (a0[i >> 1] >> 16) : (a0[i >> 1] & 0xFFFFu);
                        h1[c * 8 + i] = (i & 1) ? (a1[i >> 1] >> 16) : (a1[i >> 1] & 0xFFFFu);
                    }
                }
                constexpr int NH = 1 << (K - 1);
                uint32_t s0[NH], s1[NH], o0[NH], o1[NH];
#pragma unroll
                for (int c = 0; c < NH; ++c) {
                    s0[c] = (e4 & 1) ? h0[2 * c + 1] : h0[2 * c];
                    s1[c] = (e4 & 1) ? h1[2 * c + 1] : h1[2 * c];
                    o0[c] = (e4 & 2) ? h0[2 * c + 1] : h0[2 * c];
                    o1[c] = (e4 & 2) ? h1[2 * c + 1] : h1[2 * c];
                }
#pragma unroll
                for (int i = 0; i < G::kEntries / 4; ++i) {
                    uint32_t ce, co;
                    apb::pair_codes<K - 1>((uint32_t)i, ce, co);
                    const uint32_t v0 = s0[ce] | (o0[co] << 16), v1 = s1[ce] | (o1[co] << 16);
                    const uint32_t a = dst + (4 * i + e4) * 256;
                    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(v0) : "memory");
                    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a + 128), "r"(v1) : "memory");
                }
            } else {
                auto chunk_addr = [&](int r, int cc) -> uint32_t {
                    const int b = cc / 8, ci = cc % 8;
                    if constexpr (K == 5) return lut + r * 64 + ((ci ^ ((r >> 1) & 3)) << 4);
                    else return lut + b * (kRows * 128) + r * 128 + ((ci ^ (r & 7)) << 4);
                };
#pragma unroll 2
                for (int cc = e4; cc < G::kLutHalves / 8; cc += 4) {
                    const uint4 v0 = lds128(chunk_addr(r0, cc)), v1 = lds128(chunk_addr(r1, cc));
                    const uint32_t a0[4] = {v0.x, v0.y, v0.z, v0.w}, a1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint32_t x0 = (i & 1) ? (a0[i >> 1] >> 16) : (a0[i >> 1] & 0xFFFFu);
                        const uint32_t x1 = (i & 1) ? (a1[i >> 1] >> 16) : (a1[i >> 1] & 0xFFFFu);
                        const uint32_t a = dst + (cc * 8 + i) * 256;
                        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(x0) : "memory");
                        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a + 128), "r"(x1) : "memory");
                    }
                }
            }
            return;
        } else {
        // table[entry][slot][lane]: lanes 4g..4g+3 = (row 2g, 2g, 2g+1, 2g+1) -> one
        // 16-byte store per (entry, g) holds both copies of both rows.  Lane
        // (e4 = lane >> 3, gg = lane & 7) writes entries e = e4 (mod 4) of rows 2gg, 2gg+1.
        const int e4 = lane >> 3, gg = lane & 7, r0 = 2 * gg, r1 = r0 + 1;
        const uint32_t lut = s_lut + slot * G::kLutSlot;
        const uint32_t dst = saddr(smem) + slot * 128 + gg * 16;
        if constexpr (G::kPair) {
            uint32_t h0[1 << K], h1[1 << K];
            constexpr int RB = (1 << K) * 2;  // LUT row bytes (16 or 32)
#pragma unroll
            for (int c = 0; c < RB / 16; ++c) {
                const uint4 v0 = lds128(lut + r0 * RB + c * 16), v1 = lds128(lut + r1 * RB + c * 16);
                const uint32_t a0[4] = {v0.x, v0.y, v0.z, v0.w}, a1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    h0[c * 8 + i] = (i & 1) ? (a0[i >> 1] >> 16) : (a0[i >> 1] & 0xFFFFu);
                    h1[c * 8 + i] = (i & 1) ? (a1[i >> 1] >> 16) : (a1[i >> 1] & 0xFFFFu);
                }
            }
            // idx = 4i + e4: pair-index bits 0/1 (= code bit 0 of the even / odd
            // column) come from e4, the rest from i (compile time)
            constexpr int NH = 1 << (K - 1);
            uint32_t s0[NH], s1[NH], o0[NH], o1[NH];
#pragma unroll
            for (int c = 0; c < NH; ++c) {
                s0[c] = (e4 & 1) ? h0[2 * c + 1] : h0[2 * c];
                s1[c] = (e4 & 1) ? h1[2 * c + 1] : h1[2 * c];
                o0[c] = (e4 & 2) ? h0[2 * c + 1] : h0[2 * c];
                o1[c] = (e4 & 2) ? h1[2 * c + 1] : h1[2 * c];
            }
#pragma unroll
            for (int i = 0; i < G::kEntries / 4; ++i) {
                if constexpr (kCoop)
                    if (i % nbw != bw) continue;
                uint32_t ce, co;
                apb::pair_codes<K - 1>((uint32_t)i, ce, co);
                const uint32_t v0 = s0[ce] | (o0[co] << 16), v1 = s1[ce] | (o1[co] << 16);
                asm volatile("st.shared.v4.u32 [%0], {%1,%1,%2,%2};" ::"r"(dst + (4 * i + e4) * 256), "r"(v0), "r"(v1)
                             : "memory");
            }
        } else {
            auto chunk_addr = [&](int r, int cc) -> uint32_t {  // 16-byte chunk cc of LUT row r
                const int b = cc / 8, ci = cc % 8;
                if constexpr (K == 5) return lut + r * 64 + ((ci ^ ((r >> 1) & 3)) << 4);
                else return lut + b * (kRows * 128) + r * 128 + ((ci ^ (r & 7)) << 4);
            };
#pragma unroll 2
            for (int cc = e4 + (kCoop ? 4 * bw : 0); cc < G::kLutHalves / 8; cc += kCoop ? 4 * nbw : 4) {
                const uint4 v0 = lds128(chunk_addr(r0, cc)), v1 = lds128(chunk_addr(r1, cc));
                const uint32_t a0[4] = {v0.x, v0.y, v0.z, v0.w}, a1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t x0 = (i & 1) ? (a0[i >> 1] >> 16) : (a0[i >> 1] & 0xFFFFu);
                    const uint32_t x1 = (i & 1) ? (a1[i >> 1] >> 16) : (a1[i >> 1] & 0xFFFFu);
                    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%2,%2};" ::"r"(dst + (cc * 8 + i) * 256), "r"(x0), "r"(x1)
                                 : "memory");
                }
            }
        }
        }
    };
    if (warp == WC) {
        // ============================ producer (TMA) ============================
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        int slot = 0, ph = 0;  // ring position of the next stage
        int pi = problem_of(L, first), pend = problem_end(L, pi);
#pragma unroll 1
        for (int jl = 0; jl < n_local; ++jl) {
            const int item = first + jl;
            if (item >= pend) {
                pi = problem_of(L, item);
                pend = problem_end(L, pi);
            }
            const Prob7& P = L.prob[pi];
            const int row0 = (item - P.item_begin) * kRows;
            // centroid rows of the item -> lut slot jl & 1
            if (jl >= 2) mbar_wait(b_lempty + 8 * (jl & 1), ((jl - 2) >> 1) & 1);
            mbar_expect_tx(b_lfull + 8 * (jl & 1), G::kLutBytes);
#pragma unroll
            for (int b = 0; b < G::kLutBoxes; ++b)
                tma2(s_lut + (jl & 1) * G::kLutSlot + b * (kRows * G::kLutBox * 2), &L.tm_lut[pi], b * G::kLutBox, row0,
                     b_lfull + 8 * (jl & 1));
            // plane tiles -> ring stages
#pragma unroll 1
            for (int t = 0; t < P.n_tiles; ++t) {
                if (ph > 0) mbar_wait(b_empty + 8 * slot, (ph - 1) & 1);
                mbar_expect_tx(b_full + 8 * slot, G::kStageBytes);
                const uint32_t dst = s_ring + slot * G::kStageBytes;
#pragma unroll
                for (int p = 0; p < K; ++p)
                    tma3_ef(dst + p * 2048, &L.tm_planes[pi], t * kTileBytes, row0, p, b_full + 8 * slot, pol);
                if (++slot == NST) {
                    slot = 0;
                    ++ph;
                }
            }
        }
        APB_TL(6);
        return;
    }

    if (warp == WC + 1) {
        // ========================= service: tables, x, y =========================
        const int g = lane >> 2, q = lane & 3, rho = 2 * g + (q >> 1);
        uint32_t y_written = 0;  // y values this lane stored (fused all-gather accounting)
        float norm_scale = 1.f;  // norm_mode 2: the producer's RMSNorm factor
        float sq_acc = 0.f;      // norm_mode 1: this lane's sum of resid^2
        float resid_pre = 0.f;   // norm_mode 1: resid of row (item row0 + lane), prefetched
        auto reduce = [&](int item, int pi, int slot) {
            const Prob7& P = L.prob[pi];
            const int m_out = L.x_split ? (L.m_x >> 1) : L.m_x;
            const int64_t row0 = (int64_t)(item - P.item_begin) * kRows;
            const float* r = red + slot * (WC * 2 * NB * kRows);
            auto row_sum = [&](int rl, int m) {
                if (L.x_split) {  // batch rows (2m, 2m+1) = (hi, lo) halves of fp32 x
                    float hi = 0.f, lo = 0.f;
#pragma unroll
                    for (int w = 0; w < WC; ++w) hi += r[(w * 2 * NB + 2 * m) * kRows + rl];
#pragma unroll
                    for (int w = 0; w < WC; ++w) lo += r[(w * 2 * NB + 2 * m + 1) * kRows + rl];
                    return L.x_split == 2 ? (hi + lo) * P.xinv[m] : hi + lo;  // scaled pairs: undo 2^e
                }
                float sum = 0.f;
#pragma unroll
                for (int w = 0; w < WC; ++w) sum += r[(w * 2 * NB + m) * kRows + rl];
                return sum;
            };
            auto store = [&](int m, int64_t orow, float v) {
                const int64_t off = (int64_t)m * P.ldy + orow;
                if (L.y_f16) {
                    const __half hv = __float2half_rn(v);
                    reinterpret_cast<__half*>(P.y)[off] = hv;
                    for (int j = 0; j < ep_peers; ++j) reinterpret_cast<__half*>(L.y_peer[pi][j])[off] = hv;
                } else {
                    reinterpret_cast<float*>(P.y)[off] = v;
                    for (int j = 0; j < ep_peers; ++j) reinterpret_cast<float*>(L.y_peer[pi][j])[off] = v;
                }
                ++y_written;
            };
            if (ep_glu) {  // rows (2i, 2i+1) = (gate_i, up_i): y[i] = silu(gate_i . x) * (up_i . x)
                for (int i = lane; i < (kRows / 2) * m_out; i += 32) {
                    const int pr = i & 7, m = i >> 3;
                    const int64_t row = row0 + 2 * pr;
                    if (row >= P.rows) continue;
                    const float gt = norm_scale * row_sum(2 * pr, m), up = norm_scale * row_sum(2 * pr + 1, m);
                    store(m, row >> 1, gt / (1.f + __expf(-gt)) * up);
                }
                return;
            }
            for (int i = lane; i < kRows * m_out; i += 32) {
                const int rl = i & 15, m = i >> 4;
                const int64_t row = row0 + rl;
                if (row >= P.rows) continue;
                if (ep_norm == 1) {  // residual add + the next RMSNorm's numerator (m_out == 1)
                    const float rs = resid_pre + row_sum(rl, m);  // lane == rl: loaded during the compute
                    __stcg(L.resid + row, rs);
                    sq_acc += rs * rs;
                    store(m, row, rs * __half2float(L.norm_w[row]));
                } else {
                    store(m, row, norm_scale * row_sum(rl, m));
                }
            }
        };

        // tables depend only on the weights: they are built before the previous
        // kernel of the stream has finished (PDL); y is written only after it has
        // activations of problem pi -> x buffer xb (one bulk copy per batch row;
        // columns past cols are masked by the compute warps)
        auto issue_x = [&](int pi, int xb) {
            if (NB > 1 || lane != 0) return;
            issue_x_one(pi, xb);
        };
        // tables depend only on the weights: they are built before the previous
        // kernel of the stream has finished (PDL); x is read and y written after
        int pi = problem_of(L, first), pend = problem_end(L, pi), xb = 0;
        int pi_hist[2] = {pi, pi};
        // The first layer's x is issued by compute warp 0 (after its PDL wait), so
        // the first tables -- weights only -- are built even while the previous
        // kernel of the stream is still running.
        bool waited = false;
#pragma unroll 1
        for (int jl = 0; jl < n_local + 2; ++jl) {
            if (jl >= 2) {  // item jl-2 done by every compute warp: reduce it, free its slot
                if (ep_norm == 1) {  // residual rows of this item, fetched while it is computed
                    if (!waited) {
                        asm volatile("griddepcontrol.wait;" ::: "memory");
                        waited = true;
                    }
                    const Prob7& P = L.prob[pi_hist[jl & 1]];
                    const int64_t row = (int64_t)(first + jl - 2 - P.item_begin) * kRows + lane;
                    resid_pre = lane < kRows && row < P.rows ? __ldcg(L.resid + row) : 0.f;
                }
                mbar_wait(b_idone + 8 * (jl & 1), ((jl - 2) >> 1) & 1);
                if (!waited) {  // y of earlier kernels (PDL); compute warp 0 already waited
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    waited = true;
                    if (ep_norm == 2) norm_scale = *s_norm;  // written by compute warp 0 before item 0 was done
                }
                reduce(first + jl - 2, pi_hist[jl & 1], jl & 1);
            }
            if (jl < n_local) {
                const int item = first + jl;
                if (item >= pend) {  // next layer of a grouped launch
                    const int npi = problem_of(L, item);
                    pend = problem_end(L, npi);
                    if (L.prob[npi].xid != L.prob[pi].xid) {  // new activations -> the other buffer
                        xb = L.x_bufs == 2 ? xb ^ 1 : 0;
                        if (!waited) {
                            asm volatile("griddepcontrol.wait;" ::: "memory");
                            waited = true;
                        }
                        issue_x(npi, xb);
                    }
                    pi = npi;
                }
                pi_hist[jl & 1] = pi;
                mbar_wait(b_lfull + 8 * (jl & 1), (jl >> 1) & 1);
                if (kCoopFirst && jl == 0) {
                    build(std::true_type{}, 0, WC, WC + 1);
                    __syncwarp();
                    asm volatile("barrier.sync 1, %0;" ::"r"((WC + 1) * 32) : "memory");  // with the compute warps
                } else {
                    build(std::false_type{}, jl & 1, 0, 1);
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(b_lempty + 8 * (jl & 1));
                    mbar_arrive(b_tready + 8 * (jl & 1));
                }
                if (jl == 0 && lane == 0) APB_TL(1);
            }
        }
        if (ep_norm == 1) {  // this CTA's share of the next RMSNorm's sum of squares
#pragma unroll
            for (int o = 16; o; o >>= 1) sq_acc += __shfl_xor_sync(0xffffffffu, sq_acc, o);
            if (lane == 0) __stcg(L.partials + blockIdx.x, sq_acc);
            // this grid (its size depends on k and the shape) may be smaller than
            // the previous producer's on the same buffer: CTA 0 zeroes the slots no
            // CTA of this grid owns (the service warp has passed the PDL wait)
            if (blockIdx.x == 0)
                for (int i = (int)gridDim.x + lane; i < L.n_partials; i += 32) __stcg(L.partials + i, 0.f);
        }
        if (ep_peers >= 0) {
            // publish: every lane's local + peer stores visible system-wide, then
            // one release-add per rank of the values this CTA wrote
            __threadfence_system();
            uint32_t tot = y_written;
#pragma unroll
            for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
            __syncwarp();
            if (lane <= ep_peers && tot > 0)  // peers' counters, then this rank's own
                asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(L.peer_flag[lane]), "r"(tot) : "memory");
        }
        if (lane == 0) APB_TL(5);
        return;
    }

    // =============================== compute warps ===============================
    if constexpr (G::kMapN) {
        // Batch-in-N mapping: lane (g, q) owns rows g (A rows g) and g + 8 (A rows
        // g + 8) at the same columns; its 16-B chunk c = su + 4(q>>1), 8-B half q&1
        // (words 4c + 2(q&1) + wi); B column n = batch row n (dense: every lane loads
        // x[min(g, m_x-1)] for its columns from L1-resident global memory).
        const int g = lane >> 2, q = lane & 3;
        const int grp = warp >> 2, su = warp & 3;
        const int c = su + 4 * (q >> 1), hf = q & 1;
        const uint32_t po0 = g * 128 + ((c ^ g) << 4) + hf * 8, po1 = po0 + 8 * 128;  // rows g, g+8 (same swizzle)
        const int gm = g < L.m_x ? g : L.m_x - 1;
        const int gm2 = 8 + g < L.m_x ? 8 + g : L.m_x - 1;  // NB == 8: batch rows 8..15 (second MMA)
        constexpr int kBR = 2 * NB;                          // batch rows of the partials
        const int xcol0 = 8 * (4 * c + 2 * hf);  // column of word wi=0, p=0 (+ tile*1024 + 256p + 8wi)
        int pi = problem_of(L, first), pend = problem_end(L, pi);
        int gs = grp, item_gs = 0, slot = grp, ph = 0;
#pragma unroll 1
        for (int jl = 0; jl < n_local; ++jl) {
            const int item = first + jl;
            if (item >= pend) {
                pi = problem_of(L, item);
                pend = problem_end(L, pi);
            }
            const Prob7& P = L.prob[pi];
            const int nt = P.n_tiles;
            const uint16_t* const xrow = P.x + (int64_t)gm * P.ldx + xcol0;
            const uint16_t* const xrow2 = P.x + (int64_t)gm2 * P.ldx + xcol0;
            const int xcols = (int)P.cols - xcol0;
            const int full_tiles = (int)(P.cols / kTileWeights);
            const uint32_t off0 = ((uint32_t)(jl & 1) << 16) | ((uint32_t)lane * 4u), off1 = off0 + 128u;
            float acc[2][4], acc2[2][4];
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
                acc[c2][0] = acc[c2][1] = acc[c2][2] = acc[c2][3] = 0.f;
                acc2[c2][0] = acc2[c2][1] = acc2[c2][2] = acc2[c2][3] = 0.f;
            }
            mbar_sleep(b_tready + 8 * (jl & 1), (jl >> 1) & 1);
            if (jl == 0) {
                asm volatile("griddepcontrol.wait;" ::: "memory");  // x from the previous kernel
                if (ep_norm == 2 && warp == 0) norm_factor();
            }
#pragma unroll 1
            for (; gs < item_gs + nt; gs += NG) {
                const int tile = gs - item_gs;
                mbar_sleep(b_full + 8 * slot, ph);
                const uint32_t sb = s_ring + slot * G::kStageBytes;
                auto run_tile = [&](auto tail) {
                    constexpr bool kTail = decltype(tail)::value;
                    uint2 pa[K], pb[K];
#pragma unroll
                    for (int p = 0; p < K; ++p) {
                        pa[K - 1 - p] = lds64(sb + p * 2048 + po0);
                        pb[K - 1 - p] = lds64(sb + p * 2048 + po1);
                    }
#pragma unroll
                    for (int wi = 0; wi < 2; ++wi) {
                        const int cbase = tile * kTileWeights + 8 * wi;  // + 256p, relative to xcol0
                        uint4 xq[4], xq2[4];
#pragma unroll
                        for (int p = 0; p < 4; ++p) {
                            const int c0 = cbase + 256 * p;
                            const bool past = kTail && c0 >= xcols;  // never read past ldx
                            xq[p] = __ldg(reinterpret_cast<const uint4*>(past ? g_zero_x : xrow + c0));
                            if constexpr (NB == 8) xq2[p] = __ldg(reinterpret_cast<const uint4*>(past ? g_zero_x : xrow2 + c0));
                            if constexpr (kTail) {
                                uint32_t mk[4];
#pragma unroll
                                for (int h = 0; h < 4; ++h)
                                    mk[h] = (c0 + 2 * h < xcols ? 0x0000FFFFu : 0u) | (c0 + 2 * h + 1 < xcols ? 0xFFFF0000u : 0u);
                                xq[p] = make_uint4(xq[p].x & mk[0], xq[p].y & mk[1], xq[p].z & mk[2], xq[p].w & mk[3]);
                                if constexpr (NB == 8)
                                    xq2[p] = make_uint4(xq2[p].x & mk[0], xq2[p].y & mk[1], xq2[p].z & mk[2], xq2[p].w & mk[3]);
                            }
                        }
                        uint32_t Qa[K], Qb[K];
#pragma unroll
                        for (int i = 0; i < K; ++i) {
                            Qa[i] = wi ? pa[i].y : pa[i].x;
                            Qb[i] = wi ? pb[i].y : pb[i].x;
                        }
                        uint32_t a0[16], a1[16];
                        decode_word<K>(Qa, off0, a0);
                        decode_word<K>(Qb, off1, a1);
                        if (wi == 0) {  // every plane register of the stage consumed: release it
                            mbar_arrive(b_empty + 8 * slot);
                            slot += NG;
                            if (slot >= NST) {
                                slot -= NST;
                                ph ^= 1;
                            }
                        }
#pragma unroll
                        for (int p = 0; p < 4; ++p)
#pragma unroll
                            for (int jj = 0; jj < 2; ++jj) {
                                mma16816(acc[p & 1], a0[p * 4 + 2 * jj], a1[p * 4 + 2 * jj], a0[p * 4 + 2 * jj + 1],
                                         a1[p * 4 + 2 * jj + 1], u4w(xq[p], 2 * jj), u4w(xq[p], 2 * jj + 1));
                                if constexpr (NB == 8)  // the same A fragment against batch rows 8..15
                                    mma16816(acc2[p & 1], a0[p * 4 + 2 * jj], a1[p * 4 + 2 * jj],
                                             a0[p * 4 + 2 * jj + 1], a1[p * 4 + 2 * jj + 1], u4w(xq2[p], 2 * jj),
                                             u4w(xq2[p], 2 * jj + 1));
                            }
                    }
                };
                if (tile < full_tiles)
                    run_tile(std::false_type{});
                else
                    run_tile(std::true_type{});
            }
            item_gs += nt;
            // D[g][2q..2q+1] / D[g+8][2q..2q+1]: rows g, g+8 of batch rows 2q, 2q+1
            float* r = red + (jl & 1) * (WC * kBR * kRows) + warp * kBR * kRows;
            r[(2 * q) * kRows + g] = acc[0][0] + acc[1][0];
            r[(2 * q + 1) * kRows + g] = acc[0][1] + acc[1][1];
            r[(2 * q) * kRows + g + 8] = acc[0][2] + acc[1][2];
            r[(2 * q + 1) * kRows + g + 8] = acc[0][3] + acc[1][3];
            if constexpr (NB == 8) {  // batch rows 8 + 2q, 8 + 2q + 1
                r[(8 + 2 * q) * kRows + g] = acc2[0][0] + acc2[1][0];
                r[(8 + 2 * q + 1) * kRows + g] = acc2[0][1] + acc2[1][1];
                r[(8 + 2 * q) * kRows + g + 8] = acc2[0][2] + acc2[1][2];
                r[(8 + 2 * q + 1) * kRows + g + 8] = acc2[0][3] + acc2[1][3];
            }
            mbar_arrive(b_idone + 8 * (jl & 1));
        }
        return;
    }
    // Lane (g, q): row rho = 2g + (q >> 1) of the item, copy cp = q & 1.  Warp su
    // = warp & 3 of its group takes 16-byte chunks su and su + 4 of every stage
    // (tile) row; copy cp reads words 2cp, 2cp+1 of a chunk (LDS.64: rows 0..7 of a
    // phase hit 8 distinct swizzled chunks).  Word t = 4ch + 2cp + wi.
    const int g = lane >> 2, q = lane & 3;
    const int rho = 2 * g + (q >> 1), cp = q & 1;
    const int grp = warp >> 2, su = warp & 3;
    uint32_t plane_off[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) plane_off[j] = rho * 128 + (((su + 4 * j) ^ (rho & 7)) << 4) + cp * 8;
    // B fragment role: column n = g; batch row gm = 2b + (g >> 2) for batch pair b,
    // column set gset = (g >> 1) & 1.  Live lanes read x[gm][tile*1024 + 256p +
    // 8t + 4*gset .. +3] (8 bytes; the 4 live addresses of a load are 8 / 32 B
    // apart -> one wavefront); the others hold zeros (smem path) or read the
    // all-zero array (global path).
    const int gset = (g >> 1) & 1;
    const bool xrole = (q >> 1) == (g & 1);
    uint32_t xlive[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) xlive[b] = (xrole && 2 * b + (g >> 2) < L.m_x) ? 1u : 0u;

    uint32_t xv[NB][8];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[b][i] = 0u;

#ifdef APB_TIMELINE
    long long full_wait = 0, t_begin = clock64();
#endif
    int pi = problem_of(L, first), pend = problem_end(L, pi), xb = 0;
    uint32_t xph = 0;  // bit b: phase parity of x buffer b
    int gs = grp;            // next ring stage of this warp group
    int item_gs = 0;         // first stage of the current item
    int slot = grp, ph = 0;  // ring slot / phase parity of stage gs (NST >= NG)
#pragma unroll 1
    for (int jl = 0; jl < n_local; ++jl) {
        const int item = first + jl;
        bool new_x = jl == 0;
        if (item >= pend) {
            const int npi = problem_of(L, item);
            pend = problem_end(L, npi);
            if (L.prob[npi].xid != L.prob[pi].xid) {
                xb = L.x_bufs == 2 ? xb ^ 1 : 0;
                new_x = true;
            }
            pi = npi;
        }
        const Prob7& P = L.prob[pi];
        const int nt = P.n_tiles;
        // column of word t = 4ch + 2cp + wi: 8t = 32su + 128j + 16cp + 8wi
        const int xcol0 = 32 * su + 16 * cp + 4 * gset;
        const int xcols = (int)P.cols - xcol0;  // column limit relative to the lane's x base
        const int full_tiles = (int)(P.cols / kTileWeights);
        uint32_t xrow_s = 0;                    // NB == 1: shared-memory x of this layer
        const uint16_t* xrow_g[NB];             // NB > 1: global x rows
        if constexpr (NB == 1) {
            xrow_s = saddr(xs + xb * L.xs_bytes) + (uint32_t)((g >> 2) < L.m_x ? (g >> 2) : 0) * (uint32_t)(nt * 2048) +
                     (uint32_t)xcol0 * 2u;
        } else {
#pragma unroll
            for (int b = 0; b < NB; ++b)
                xrow_g[b] = xlive[b] ? P.x + (int64_t)(2 * b + (g >> 2)) * P.ldx + xcol0 : g_zero_x;
        }
        const uint32_t off = (uint32_t)(jl & 1) * 128u + (uint32_t)lane * 4u;
#ifndef APB7_ACC_CHAINS
#define APB7_ACC_CHAINS 2
#endif
        constexpr int kAccChains = NB == 1 ? APB7_ACC_CHAINS : 2;  // independent HMMA accumulator chains
        float acc[NB][kAccChains][4];
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int c2 = 0; c2 < kAccChains; ++c2) acc[b][c2][0] = acc[b][c2][1] = acc[b][c2][2] = acc[b][c2][3] = 0.f;

        if (kCoopFirst && jl == 0) {  // first table: built by all compute warps + the service warp
            mbar_sleep(b_lfull, 0);
            build(std::true_type{}, 0, warp, WC + 1);
            __syncwarp();
            asm volatile("barrier.sync 1, %0;" ::"r"((WC + 1) * 32) : "memory");
        } else {
            mbar_sleep(b_tready + 8 * (jl & 1), (jl >> 1) & 1);  // table of this item
        }
        if (new_x) {
            if constexpr (NB == 1) {  // activations of this layer staged
                if (jl == 0 && warp == 0) {  // first layer: x / y of earlier kernels (PDL), then x
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    if (lane == 0) {
                        issue_x_one(pi, 0);
                        APB_TL(2);
                    }
                    if (ep_norm == 2) norm_factor();  // overlaps the x copy
                }
                mbar_sleep(b_xfull + 8 * xb, (xph >> xb) & 1u);
                xph ^= 1u << xb;
            } else if (jl == 0) {
                asm volatile("griddepcontrol.wait;" ::: "memory");  // x from the previous kernel
                if (ep_norm == 2 && warp == 0) norm_factor();
            }
        }
#pragma unroll 1
        for (; gs < item_gs + nt; gs += NG) {
            const int tile = gs - item_gs;
#ifdef APB_TIMELINE
            {
                const long long w0 = clock64();
                mbar_sleep(b_full + 8 * slot, ph);
                full_wait += clock64() - w0;
            }
#else
            mbar_sleep(b_full + 8 * slot, ph);
#endif
            if (warp == 0 && lane == 0 && gs == 0) APB_TL(3);
            const uint32_t sb = s_ring + slot * G::kStageBytes;
            // one tile of this warp's chunks; TAIL: the last, partial tile of a layer
            // (activation columns >= cols read as zero) -- a separate instantiation, so
            // full tiles carry no per-word-step tail test
            auto run_tile = [&](auto tail) {
                constexpr bool kTail = decltype(tail)::value;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    uint2 pv[K];
#pragma unroll
                    for (int p = 0; p < K; ++p) pv[K - 1 - p] = lds64(sb + p * 2048 + plane_off[j]);  // Q[i] = plane K-1-i
#pragma unroll
                    for (int wi = 0; wi < 2; ++wi) {
                        const int cbase = tile * kTileWeights + 128 * j + 8 * wi;  // + 256p, relative to xcol0
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            uint32_t(&x8)[8] = xv[b];
                            if constexpr (NB == 1) {
                                const uint32_t xa = xrow_s + (uint32_t)cbase * 2u;
#pragma unroll
                                for (int p = 0; p < 4; ++p) lds64_keep(x8[2 * p], x8[2 * p + 1], xa + 512 * p, xlive[0]);
                            } else {
#pragma unroll
                                for (int p = 0; p < 4; ++p) {
                                    const uint16_t* src = xrow_g[b] + cbase + 256 * p;
                                    if (kTail && cbase + 256 * p >= xcols) src = g_zero_x;  // never read past ldx
                                    const uint2 v = __ldg(reinterpret_cast<const uint2*>(src));
                                    x8[2 * p] = v.x;
                                    x8[2 * p + 1] = v.y;
                                }
                            }
                            if constexpr (kTail) {  // columns >= cols are zero
#pragma unroll
                                for (int p = 0; p < 4; ++p) {
                                    const int c0 = cbase + 256 * p;
                                    x8[2 * p] &= (c0 < xcols ? 0x0000FFFFu : 0u) | (c0 + 1 < xcols ? 0xFFFF0000u : 0u);
                                    x8[2 * p + 1] &= (c0 + 2 < xcols ? 0x0000FFFFu : 0u) | (c0 + 3 < xcols ? 0xFFFF0000u : 0u);
                                }
                            }
                        }
                        uint32_t Q[K];
#pragma unroll
                        for (int i = 0; i < K; ++i) Q[i] = wi ? pv[i].y : pv[i].x;
                        uint32_t a[16];
                        decode_word<K>(Q, off, a);
                        if (j == 1 && wi == 0) {  // every plane register of the stage consumed: release it
                            mbar_arrive(b_empty + 8 * slot);
                            slot += NG;
                            if (slot >= NST) {
                                slot -= NST;
                                ph ^= 1;
                            }
                        }
#pragma unroll
                        for (int b = 0; b < NB; ++b)
#pragma unroll
                            for (int p = 0; p < 4; ++p)
                                mma16816(acc[b][kAccChains == 4 ? p : (p & 1)], a[p * 4 + 0], a[p * 4 + 2], a[p * 4 + 1],
                                         a[p * 4 + 3], xv[b][2 * p], xv[b][2 * p + 1]);
                    }
                }
            };
            if (tile < full_tiles)
                run_tile(std::false_type{});
            else
                run_tile(std::true_type{});
        }
        item_gs += nt;
        // rows 2g / 2g+1 of batch row 2b + (q>>1): D[g][2q'] + D[g+8][2q'+2] with q' = q & 2
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            float c[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                c[i] = acc[b][0][i] + acc[b][1][i];
                if constexpr (kAccChains == 4) c[i] += acc[b][2][i] + acc[b][3][i];
            }
            const float o2 = __shfl_xor_sync(0xffffffffu, c[2], 1), o3 = __shfl_xor_sync(0xffffffffu, c[3], 1);
            if ((q & 1) == 0) {
                float* r = red + (jl & 1) * (WC * 2 * NB * kRows) + (warp * 2 * NB + 2 * b + (q >> 1)) * kRows + 2 * g;
                r[0] = c[0] + o2;
                r[1] = c[1] + o3;
            }
        }
        mbar_arrive(b_idone + 8 * (jl & 1));  // all lanes (release orders the partial stores)
        if (warp == 0 && lane == 0 && jl == 0) APB_TL(4);
    }
#ifdef APB_TIMELINE
    if (warp == 0 && lane == 0) {  // slot 7: warp 0's cycles waiting for plane stages / cycles in its loop
        g_tl7[((size_t)(L.tl_launch % 64) * 512 + blockIdx.x) * 8 + 7] =
            ((unsigned long long)full_wait << 32) | (unsigned long long)((clock64() - t_begin) & 0xFFFFFFFFull);
    }
#endif
}

// ---- host side -------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

static bool make_plane_map(CUtensorMap* m, const uint8_t* planes, int n_max, int64_t rows, int64_t row_bytes) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)row_bytes, (cuuint64_t)rows, (cuuint64_t)n_max};
    const cuuint64_t strides[2] = {(cuuint64_t)row_bytes, (cuuint64_t)(rows * row_bytes)};
    const cuuint32_t box[3] = {128, (cuuint32_t)kRows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)planes, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_lut_map(CUtensorMap* m, const uint16_t* lut, int k, int64_t rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const int n = 1 << k, bx = n < 64 ? n : 64;
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)n * 2};
    const cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)kRows};
    const cuuint32_t es[2] = {1, 1};
    const CUtensorMapSwizzle sw =
        k >= 6 ? CU_TENSOR_MAP_SWIZZLE_128B : (k == 5 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE);
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)lut, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

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

constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kSmemLimit2 = 113 * 1024;  // per CTA with two CTAs per SM
constexpr int kMaxStages = 16;

// Two CTAs per SM when an 8-compute-warp CTA with >= 4 ring stages fits in half
// the shared memory: a CTA that finishes early frees half an SM for the next
// kernel of a PDL chain while its neighbour still works, and the work
// granularity halves.  APB7_CPS=1|2 forces the choice (tuning).
template <int K, int NB>
static int choose_cps(const Launch7& L) {
    static const int forced = [] {
        const char* e = std::getenv("APB7_CPS");
        return e ? std::atoi(e) : 0;
    }();
    if (forced == 1) return 1;
    static const int cps1_k = [] {  // tuning: bit K set -> one CTA per SM at bit width K
        const char* e = std::getenv("APB7_CPS1_K");
        return e ? std::atoi(e) : 0;
    }();
    if (cps1_k & (1 << K)) return 1;
    const bool fits2 = NB == 1 && Geo<K, NB, 2>::total(4, L.x_bufs * L.xs_bytes) <= kSmemLimit2;
    if (forced == 2) return fits2 ? 2 : 1;
    // measured: in a PDL chain of decode-sized launches (the bench step) two CTAs
    // per SM win +5 % overall (cross-kernel overlap, granularity); a long
    // isolated launch (> 10 items per SM, e.g. a 28672-row layer) runs ~4 %
    // faster with one 16-warp CTA per SM, except at k = 3.
    const bool long_launch = L.n_items > 10 * sm_count();
    // fewer items than SMs (row shards, small layers): two CTAs per SM would leave
    // each SM ONE 8-warp CTA -- half the decode rate of a 16-warp CTA (measured:
    // 2048 x 28672 at k = 3 took 14.9 us vs 11.1 at k = 4, which runs one CTA per SM)
    const bool few_items = L.n_items < sm_count();
    return fits2 && !few_items && (K == 3 || !long_launch) ? 2 : 1;
}

template <int K, int NB, int CPS, bool EPI>
static int launch(Launch7& L, int flags, cudaStream_t s, bool dry = false) {
    using G = Geo<K, NB, CPS>;
    const size_t limit = CPS == 2 ? kSmemLimit2 : kSmemLimit;
    // ring depth: as many stages as fit (>= 3)
    int nst = kMaxStages;
    while (nst >= G::kNG && G::total(nst, L.x_bufs * L.xs_bytes) > limit) --nst;
    if (nst < G::kNG || nst < 3) return -1;
    if (dry) return APB_OK;  // apb7_plan_create: the launch shape fits
    L.n_stages = nst;
    auto kern = gemv7_kernel<K, NB, CPS, EPI>;
    static std::atomic<unsigned long long> configured{0};
    if (!apb::ensure_smem_optin(kern, (int)kSmemLimit, configured)) return APB_ERR_CUDA;
    int grid = CPS * sm_count();
    if (grid > L.n_items) grid = L.n_items;
    if (L.norm_mode == 1 && grid > L.n_partials) return APB_ERR_PARAM;  // a CTA without a partials slot
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)G::kThreads);
    cfg.dynamicSmemBytes = G::total(nst, L.x_bufs * L.xs_bytes);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (flags & APB_FLAG_PDL) ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, kern, L) != cudaSuccess) return APB_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

}  // namespace apb7

// Called by apb_gemv_grouped (apb_gemv.cu) after argument validation.
// Returns -1 when this kernel does not apply (caller falls back), else a status.
#ifdef APB_TIMELINE
static int g_tl_host_launch = 0;
extern "C" int apb7_read_timeline(unsigned long long* host, int n) {
    return cudaMemcpyFromSymbol(host, apb7::g_tl7, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 5;
}
extern "C" void apb7_timeline_reset(void) { g_tl_host_launch = 0; }
#endif

namespace apb7 {
int apb7_build(Launch7& L, int& nb, int n, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
               const int64_t* cols, const int64_t* padded, int k, const uint16_t* const* lut,
               const uint16_t* const* x, int m_x, const int64_t* ldx, int64_t x_off, int x_split, void* const* y,
               int y_dtype, const int64_t* ldy, int64_t y_off, int flags, int n_peers, void* const* y_peers,
               uint32_t* const* peer_flags, const apb_norm_epilogue* norm);
int apb7_dispatch(Launch7& L, int k, int nb, int flags, cudaStream_t s, bool dry);
}  // namespace apb7

extern "C" int apb7_try_gemv(int n, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
                             const int64_t* cols, const int64_t* padded, int k, const uint16_t* const* lut,
                             const uint16_t* const* x, int m_x, const int64_t* ldx, int64_t x_off, int x_split,
                             void* const* y, int y_dtype, const int64_t* ldy, int64_t y_off, int flags, void* stream,
                             int n_peers, void* const* y_peers, uint32_t* const* peer_flags,
                             const apb_norm_epilogue* norm) {
    using namespace apb7;
    static const bool disabled = [] {
        const char* e = std::getenv("APB_GEMV_V7");
        return e && e[0] == '0';
    }();
    // batch rows: <= 2 row-copy mapping (x in smem), 3..8 batch-in-N mapping
    // (measured faster than the two-batch-pair row-copy path from 3 rows up)
    if (disabled) return -1;
    static thread_local Launch7 L;  // ~7 KB: kept off the stack
    int nb = 0;
    const int rc = apb7::apb7_build(L, nb, n, planes, n_max, rows, cols, padded, k, lut, x, m_x, ldx, x_off, x_split, y,
                                    y_dtype, ldy, y_off, flags, n_peers, y_peers, peer_flags, norm);
    if (rc != 0) return rc;
    return apb7::apb7_dispatch(L, k, nb, flags, (cudaStream_t)stream, false);
}

namespace apb7 {
// Activation identity: layers fed the same x (q/k/v, gate/up) stage it once.
// From the problems' CURRENT x pointers (re-run when a plan is re-pointed).
static void assign_xids(Launch7& L) {
    int n_xid = 0;
    for (int i = 0; i < L.n_prob; ++i) {
        Prob7& P = L.prob[i];
        P.xid = i;
        for (int j = 0; j < i; ++j) {
            const Prob7& Q = L.prob[j];
            if (Q.x == P.x && Q.ldx == P.ldx && Q.cols == P.cols) {
                P.xid = Q.xid;
                break;
            }
        }
        if (P.xid == i) ++n_xid;
    }
    L.x_bufs = n_xid == 1 ? 1 : 2;
}

// Launch7 of a call (tensor maps encoded, partition fixed); -1 when this kernel
// does not apply.  No argument validation beyond that (the callers validate).
int apb7_build(Launch7& L, int& nb, int n, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
               const int64_t* cols, const int64_t* padded, int k, const uint16_t* const* lut,
               const uint16_t* const* x, int m_x, const int64_t* ldx, int64_t x_off, int x_split, void* const* y,
               int y_dtype, const int64_t* ldy, int64_t y_off, int flags, int n_peers, void* const* y_peers,
               uint32_t* const* peer_flags, const apb_norm_epilogue* norm) {
    if (k < 3 || k > 8 || m_x > 16 || n > kMaxProb || n_peers > kMaxPeers - 1) return -1;
    for (int i = 0; i < n; ++i)
        if (padded[i] > kMaxCols) return -1;
    std::memset(&L, 0, sizeof(L));
    L.n_prob = n;
    L.m_x = m_x;
    L.x_split = x_split;
    L.y_f16 = y_dtype == APB_DTYPE_F16;
    L.glu = (flags & APB_FLAG_GLU) ? 1 : 0;
    if (norm && norm->mode) {
        L.norm_mode = norm->mode;
        L.resid = norm->resid;
        L.norm_w = reinterpret_cast<const __half*>(norm->norm_w);
        L.partials = norm->partials;
        L.n_partials = norm->n_partials < kMaxPartials ? norm->n_partials : kMaxPartials;
        L.norm_size = norm->norm_size;
        L.norm_eps = norm->eps;
    }
    int items = 0, max_tiles = 0;
    int64_t cost = 0;
    const int esz = y_dtype == APB_DTYPE_F16 ? 2 : 4;
    for (int i = 0; i < n; ++i) {
        Prob7& P = L.prob[i];
        const int64_t row_bytes = padded[i] / 8;
        if (!make_plane_map(&L.tm_planes[i], planes[i], n_max[i], rows[i], row_bytes)) return -1;
        if (!make_lut_map(&L.tm_lut[i], lut[i], k, rows[i])) return -1;
        P.x = x[i] + x_off * ldx[i];
        P.xinv = x_split == 2 ? reinterpret_cast<const float*>(x[i] + (int64_t)m_x * ldx[i]) + x_off / 2 : nullptr;
        P.y = reinterpret_cast<uint8_t*>(y[i]) + y_off * ldy[i] * esz;
        for (int j = 0; j < n_peers; ++j)  // the same region of every peer's output
            L.y_peer[i][j] = reinterpret_cast<uint8_t*>(y_peers[(size_t)i * n_peers + j]) + y_off * ldy[i] * esz;
        P.rows = rows[i];
        P.cols = cols[i];
        P.ldx = ldx[i];
        P.ldy = ldy[i];
        P.n_tiles = (int)(padded[i] / kTileWeights);
        P.item_begin = items;
        P.cost_begin = cost;
        const int ni = (int)((rows[i] + kRows - 1) / kRows);
        items += ni;
        cost += (int64_t)ni * P.n_tiles;
        if (P.n_tiles > max_tiles) max_tiles = P.n_tiles;
    }
    L.n_items = items;
    L.total_cost = cost;
    L.xs_bytes = (int64_t)m_x * max_tiles * 2048;
    assign_xids(L);
    L.n_peers = peer_flags ? n_peers : -1;  // -1: no fused gather at all
    if (peer_flags)
        for (int j = 0; j <= n_peers; ++j) L.peer_flag[j] = peer_flags[j];
#ifdef APB_TIMELINE
    L.tl_launch = g_tl_host_launch++;
#endif
#ifndef APB7_NB2_MAX
#define APB7_NB2_MAX 2
#endif
    nb = m_x <= 2 ? 1 : (m_x <= APB7_NB2_MAX ? 2 : (m_x <= 8 ? 4 : 8));
    if (nb > 1) L.xs_bytes = 0;
    return 0;
}

int apb7_dispatch(Launch7& L, int k, int nb, int flags, cudaStream_t s, bool dry) {
    const bool epi = L.glu || L.norm_mode || L.n_peers >= 0;
    switch (k * 16 + nb) {
#define APB7_L(K, NB, CPS) \
    (epi ? launch<K, NB, CPS, true>(L, flags, s, dry) : launch<K, NB, CPS, false>(L, flags, s, dry))
#define APB7_CASE(K)                                                           \
    case K * 16 + 1: return choose_cps<K, 1>(L) == 2 ? APB7_L(K, 1, 2) : APB7_L(K, 1, 1); \
    case K * 16 + 2: return APB7_L(K, 2, 1);                                    \
    case K * 16 + 4: return APB7_L(K, 4, 1);                                    \
    case K * 16 + 8: return APB7_L(K, 8, 1);
        APB7_CASE(3)
        APB7_CASE(4)
        APB7_CASE(5)
        APB7_CASE(6)
        APB7_CASE(7)
        APB7_CASE(8)
#undef APB7_CASE
#undef APB7_L
    }
    return -1;
}
}  // namespace apb7

// ---- caller-owned launch plans: everything but the activation / output
// pointers prepared once (validation, tensor-map encoding, partition) --------
struct ApbGemvPlan7 {
    apb7::Launch7 L;
    int k, nb, flags, n;
    int64_t esz;
};

extern "C" void* apb7_plan_create(int n, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
                                  const int64_t* cols, const int64_t* padded, int k, const uint16_t* const* lut,
                                  const uint16_t* const* x, int m_x, const int64_t* ldx, int x_split, void* const* y,
                                  int y_dtype, const int64_t* ldy, int flags) {
    auto* p = new (std::nothrow) ApbGemvPlan7;
    if (!p) return nullptr;
    int nb = 0;
    if (apb7::apb7_build(p->L, nb, n, planes, n_max, rows, cols, padded, k, lut, x, m_x, ldx, 0, x_split, y, y_dtype,
                         ldy, 0, flags, 0, nullptr, nullptr, nullptr) != 0 ||
        apb7::apb7_dispatch(p->L, k, nb, flags, nullptr, true) != APB_OK) {  // e.g. x too large to stage
        delete p;
        return nullptr;
    }
    p->k = k;
    p->nb = nb;
    p->flags = flags;
    p->n = n;
    p->esz = y_dtype == APB_DTYPE_F16 ? 2 : 4;
    return p;
}

extern "C" int apb_gemv_plan_launch(void* plan, const uint16_t* const* x, void* const* y, void* stream) {
    auto* p = static_cast<ApbGemvPlan7*>(plan);
    if (!p) return APB_ERR_PARAM;
    for (int i = 0; i < p->n; ++i) {
        if (x && (!x[i] || ((uintptr_t)x[i] & 15))) return APB_ERR_PARAM;
        if (y && !y[i]) return APB_ERR_PARAM;
    }
    for (int i = 0; i < p->n; ++i) {
        apb7::Prob7& P = p->L.prob[i];
        if (x) {
            P.x = x[i];
            if (p->L.x_split == 2) P.xinv = reinterpret_cast<const float*>(x[i] + (int64_t)p->L.m_x * P.ldx);
        }
        if (y) P.y = y[i];
    }
    // the staging decision (one shared x buffer or two) follows the new pointers
    if (x) apb7::assign_xids(p->L);
    const int rc = apb7::apb7_dispatch(p->L, p->k, p->nb, p->flags, (cudaStream_t)stream, false);
    return rc == -1 ? APB_ERR_PARAM : rc;  // the re-pointed x no longer fits the staging buffers
}

extern "C" void apb_gemv_plan_destroy(void* plan) { delete static_cast<ApbGemvPlan7*>(plan); }

