// apb_dense_tc.cu -- the dense (M > dense_threshold) path of engine.gemm
// (reference engine.py:343-354: dequantize + fp32 GEMM; PAPER.md:443 runs it as
// a separate dequantisation + cuBLAS) as ONE Blackwell kernel: the k-bit
// weights are decoded from the top k bitplanes + the per-row fp16 centroid
// table and written straight into TENSOR MEMORY (tcgen05.st) as the A operand
// of tcgen05.mma (A from TMEM, B from shared memory), the activations arrive
// by TMA, the fp32 accumulator lives in tensor memory.  No dense weight tensor
// ever exists in HBM or shared memory.
//
// Numerics: the decoded weights are fp16 table entries (exact); fp32
// activations are carried as scaled fp16 (hi, lo) row pairs (apb_dense_prep_x:
// exact power-of-two row scale, hi + lo holds ~22 significant bits) and both
// products accumulate in fp32 in the same MMA, the pair summed and unscaled in
// the epilogue -- fp32-accurate like the reference (tests: 1e-5 vs fp64).
//
// CTA tile: 128 weight rows (UMMA M) x BN = 128 or 256 activation rows (UMMA N),
// K in blocks of 64 columns.  Warp roles:
//   warp 0    TMA producer: activation tiles (box {64, BN}, SW128) and plane
//             chunks (box {16 B, 128 rows, k planes} = two K blocks),
//   warp 1    TMEM allocation + the single-thread tcgen05.mma issuer,
//   warps 2-17 decoders: warp (row quarter q = warp % 4 = its TMEM lane quarter,
//             lane word h, K-block parity); thread = weight row; the decoded
//             fp16 pairs go to TMEM columns [BN + 32 slot + 16 h, +16) with one
//             tcgen05.st.32x32b.x16; then all 16 run the epilogue (tcgen05.ld -> y).
// Why TMEM for A: the kernel is shared-memory bound (LUT lookups + the tensor
// core's operand reads); staging A in shared memory cost a store and an MMA
// read per decoded weight (r2 profile: LSU 59 % + TC 30 % of the data path),
// TMEM takes both off it (M = 64 / 512 / 2048: 0.053 / 0.144 / 0.444 ms with A
// in shared memory -> 0.041 / 0.102 / 0.352 ms).
// The K order inside a 1024-column tile follows the bitplane lane words: K block
// v holds words 2v, 2v+1, element e = 32h + 8p + b of a block is column
// 256p + 8(2v+h) + b -- apb_dense_prep_x writes the activations in that order.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>

#include "../../include/anyprec_b200.h"
#include "apb_common.cuh"

namespace apbd {
using apb::prmt;

constexpr int BM = 128, BK = 64;
#ifndef APBD_PAIR_SLOTS
#define APBD_PAIR_SLOTS 8
#endif
#ifndef APBD_ONE256_SLOTS
#define APBD_ONE256_SLOTS 4  // measured: 2 slots 0.345 ms, 4 slots 0.342, 8 slots 0.346 (11008x4096, M = 2048)
#endif
constexpr int kDecWarps = 16;  // (row quarter q, word h, K-block parity) -- 4 per SM sub-partition
constexpr int kThreads = (2 + kDecWarps) * 32;
constexpr int kSmemBase = 1024;  // sm_100 reserves the first 1 KB of the shared window
// dynamic shared memory layout (offsets from the 1024-aligned base), per N tile
template <int BN, int K>
struct Lay {
    static constexpr int kXStages = BN == 256 ? 4 : 6;
    static_assert(BN == 32 || BN == 64 || BN == 128 || BN == 256, "UMMA N tile");
    static constexpr int kOffX = 0;                              // activation tiles (BN x 128 B)
    // centroid table: u32 [2^k][128 rows] (k <= 7), u16 (k = 8)
    static constexpr int kTableBytes = (1 << K) * (K <= 7 ? 4 : 2) * BM;
    // plane chunk ring: as many K x 2 KB stages as the budget leaves (2..8): each
    // stage covers two K blocks, and DRAM latency must hide behind the others
    static constexpr int kPStride = K * 2048;
    static constexpr int kPBudget = 227 * 1024 - 512 - kXStages * BN * 128 - kTableBytes;
    static constexpr int kPStages = kPBudget / kPStride > 8 ? 8 : kPBudget / kPStride;
    static_assert(kPStages >= 2, "plane ring");
    static constexpr int kOffP = kOffX + kXStages * BN * 128;    // plane chunks
    static constexpr int kOffT = kOffP + kPStages * kPStride;    // centroid table
    static constexpr int kOffB = (kOffT + kTableBytes + 15) / 16 * 16;  // mbarriers + TMEM address
    static constexpr int kBytes = kOffB + 512;
    static constexpr uint32_t kTable = (uint32_t)(kSmemBase + kOffT);  // absolute (LDS immediate)
    // tensor memory: D = columns [0, BN) (fp32), decoded A slots of 32 columns each
    // (128 lanes = weight rows x 64 K as packed fp16 pairs) after it
    static constexpr int kTmemCols = BN == 256 ? 512 : 256;  // power of two >= columns used
    // decoded A slots (32 TMEM columns each): 4 with the 128-wide N tile (small
    // batches are decode-bound: four K blocks in flight, each decoder warp owns
    // every 4th K block), 2 with the 256-wide tile (TMEM: 256 + 2 x 32 <= 512)
    static constexpr int kASlots = BN <= 128 ? 4 : 2;
    static_assert(BN + 32 * kASlots <= kTmemCols, "tensor memory budget");
    static constexpr uint32_t kColA = BN;
};

struct DenseParams {
    CUtensorMap tm_x;       // permuted activations [Mx][Cp] fp16
    CUtensorMap tm_planes;  // [n_max][R][Cp/8] u8
    const __half* lut;      // [R][2^k]
    float* y;               // [m_out][ldy] fp32
    const float* inv;       // pairs: 1 / row scale per output row
    float* ws;              // split-K: raw fp32 accumulator tiles [splits][mx][rows]
    int64_t rows, ldy;
    int mx, m_out, n_kb, pairs;  // n_kb: K blocks per split (even)
    int splits;
    int pair;  // CTA pairs (tm_x box = half the N tile per CTA)
};

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
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(m), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// table lookups: the table base is the LDS immediate
template <uint32_t T>
__device__ __forceinline__ uint32_t lds_t32(uint32_t off) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(off), "n"(T));
    return v;
}
template <uint32_t T>
__device__ __forceinline__ uint32_t lds_t16(uint32_t off) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1+%2];" : "=h"(v) : "r"(off), "n"(T));
    return v;
}
// UMMA shared-memory descriptor, K-major, 128-byte swizzle: 8-row x 128-B atoms
// stacked at SBO = 1024 B, version 1 (sm_100), layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr_) {
    return (uint64_t)((saddr_ >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, N >> 3, M >> 4
template <int BN, int MM = BM>
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(MM >> 4) << 24);

// A from tensor memory (the decoders' tcgen05.st), B from shared memory (TMA).
// PAIR: a CTA pair (cta_group::2, M = 256): A = both CTAs' TMEM lanes at the same
// column, B = both CTAs' shared-memory halves (BN / 2 activation rows each) at
// the same offset; issued by the pair's even CTA only.
template <int BN, bool PAIR>
__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t accumulate) {
    if constexpr (PAIR)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b), "n"(kIdesc<BN, 2 * BM>), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b), "n"(kIdesc<BN>), "r"(accumulate));
}
// PAIR: the arrive lands on the barrier at the same offset in BOTH CTAs of the pair
template <bool PAIR>
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    if constexpr (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
            "h"((uint16_t)3)
            : "memory");
    else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// wait for a phase completed by arrivals from the other CTA of a pair (cluster-scope acquire)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
// the even CTA of the pair's copy of a shared-memory address (cluster window: rank bit 24)
__device__ __forceinline__ uint32_t pair_leader(uint32_t a) { return a & 0xFEFFFFFFu; }
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#ifdef APBD_TL
// timing builds (tools/dense_tl.py): per-CTA globaltimer stamps / issuer wait cycles
__device__ unsigned long long g_tld[8192 * 10];
#define APBD_STAMP(i)                                                                                          \
    do {                                                                                                       \
        unsigned long long t_;                                                                                 \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                                \
        g_tld[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 10 + (i)] = t_;              \
    } while (0)
#define APBD_SET(i, v) g_tld[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 10 + (i)] = (v)
#else
#define APBD_STAMP(i) \
    do {              \
    } while (0)
#define APBD_SET(i, v) \
    do {               \
    } while (0)
#endif

template <int K, int BN, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1) dense_tc_kernel(const __grid_constant__ DenseParams P) {
    using Y = Lay<BN, K>;
    // PAIR: 4 A slots (TMEM 256 + 4 x 32 <= 512) -- a slot now waits on both CTAs' decoders
    // PAIR: half-height activation stages, twice as many in the same bytes
    constexpr int kXStages = PAIR ? 2 * Y::kXStages : Y::kXStages,
                  kASlots = PAIR ? APBD_PAIR_SLOTS : (BN == 256 ? APBD_ONE256_SLOTS : Y::kASlots),
                  kPStages = Y::kPStages;
    constexpr int kXStage = (PAIR ? BN / 2 : BN) * 128;  // bytes of one activation stage in this CTA
    static_assert(BN + 32 * kASlots <= Y::kTmemCols, "tensor memory budget");
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the table base is an LDS immediate (+ the CTA's cluster rank at bit 24, carried in rr below)
    if ((saddr(smem) & 0xFFFFFFu) != kSmemBase) __trap();
    if (threadIdx.x == 0) APBD_STAMP(0);
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    const int n0 = blockIdx.y * BN;
    uint32_t rank = 0;  // PAIR: rank in the CTA pair (clusters of 2 along the row tiles)
    if constexpr (PAIR) asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const bool issuer_cta = !PAIR || rank == 0;
    constexpr int kXRows = PAIR ? BN / 2 : BN;  // activation rows this CTA stages per K block
    const uint32_t sX = saddr(smem + Y::kOffX), sP = saddr(smem + Y::kOffP);
    const uint32_t bar = saddr(smem + Y::kOffB);
    // barriers (8 B each): x_full[8] x_empty[8] a_full[4] a_empty[4] p_full[8] p_empty[8] d_full
    static_assert(kXStages <= 8 && kASlots <= 8 && kPStages <= 8, "barrier layout");
    const uint32_t b_xf = bar, b_xe = bar + 64, b_af = bar + 128, b_ae = bar + 192, b_pf = bar + 256,
                   b_pe = bar + 320, b_d = bar + 384;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Y::kOffB + 400);
    constexpr int kPlaneBytes = Y::kPStride;  // one plane chunk stage: 16 B x 128 rows x K planes

    if (threadIdx.x == 0) {
        for (int i = 0; i < kXStages; ++i) {
            mbar_init(b_xf + 8 * i, 1);
            mbar_init(b_xe + 8 * i, 1);
        }
        for (int i = 0; i < kASlots; ++i) {
            // the K block's decoder threads; PAIR: one arrive per decoder warp of both CTAs
            mbar_init(b_af + 8 * i, PAIR ? 2 * (kASlots >= 4 ? 4 : 8) : (kASlots >= 4 ? 4 : 8) * 32);
            mbar_init(b_ae + 8 * i, 1);
        }
        for (int i = 0; i < kPStages; ++i) {
            mbar_init(b_pf + 8 * i, 1);
            mbar_init(b_pe + 8 * i, (kASlots >= 4 ? 8 : kDecWarps) * 32);  // decoders of its two K blocks
        }
        mbar_init(b_d, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // D[128 lanes][BN] fp32 + the decoded A slots
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tmem_slot)),
                         "n"(Y::kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tmem_slot)),
                         "n"(Y::kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if constexpr (PAIR)
        cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA arrive / TMA
    else
        __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) APBD_STAMP(1);
    const int n_kb = P.n_kb;                  // this CTA's K blocks (split-K: blockIdx.z's share)
    const int kb0 = (int)blockIdx.z * n_kb;  // first global K block (even)

    if (warp == 0) {
        // ================================ TMA producers ================================
        // lane 0 streams plane chunks, lane 1 activation tiles: independent rings, so a
        // full activation ring (waiting on the MMA) never stalls the plane prefetch
        if (lane == 0) {
            for (int ps = 0; ps < (n_kb >> 1); ++ps) {  // plane chunk ps = K blocks 2ps, 2ps+1
                const int s = ps % kPStages;
                if (ps >= kPStages) mbar_wait(b_pe + 8 * s, ((ps / kPStages) - 1) & 1);
                mbar_expect_tx(b_pf + 8 * s, kPlaneBytes);
                tma3(sP + s * Y::kPStride, &P.tm_planes, 16 * ((kb0 >> 1) + ps), (int)row0, 0, b_pf + 8 * s);
            }
        } else if (lane == 1) {
            for (int kb = 0; kb < n_kb; ++kb) {
                const int s = kb % kXStages;
                if (kb >= kXStages) mbar_wait(b_xe + 8 * s, ((kb / kXStages) - 1) & 1);
                if constexpr (PAIR) {
                    // each CTA stages its half of the tile; both halves complete on the even
                    // CTA's barrier, which expects the whole tile
                    if (rank == 0) mbar_expect_tx(b_xf + 8 * s, BN * 128);
                    asm volatile(
                        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                            sX + s * kXStage),
                        "l"(&P.tm_x), "r"((kb0 + kb) * BK), "r"(n0 + (int)rank * kXRows), "r"(pair_leader(b_xf + 8 * s))
                        : "memory");
                } else {
                    mbar_expect_tx(b_xf + 8 * s, BN * 128);
                    tma2(sX + s * kXStage, &P.tm_x, (kb0 + kb) * BK, n0, b_xf + 8 * s);
                }
            }
        }
    } else if (warp == 1) {
        // ============================ tcgen05.mma issuer ============================
        if (lane == 0 && issuer_cta) {
#ifdef APBD_TL
            long long wa = 0, wx = 0;
#endif
            for (int kb = 0; kb < n_kb; ++kb) {
                const int sa = kb % kASlots, sx = kb % kXStages;
#ifdef APBD_TL
                long long c0 = clock64();
                mbar_wait(b_af + 8 * sa, (kb / kASlots) & 1);
                long long c1 = clock64();
                mbar_wait(b_xf + 8 * sx, (kb / kXStages) & 1);
                wa += c1 - c0;
                wx += clock64() - c1;
                if (kb == 0) APBD_STAMP(2);
#else
                if constexpr (PAIR)
                    mbar_wait_cluster(b_af + 8 * sa, (kb / kASlots) & 1);
                else
                    mbar_wait(b_af + 8 * sa, (kb / kASlots) & 1);
                mbar_wait(b_xf + 8 * sx, (kb / kXStages) & 1);
#endif
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t dx = sw128_desc(sX + sx * kXStage);
                const uint32_t ta = tmem + Y::kColA + 32u * (uint32_t)sa;
#pragma unroll
                for (int ks = 0; ks < BK / 16; ++ks)  // K = 16 per MMA: 8 TMEM columns of A, +32 B of B's swizzle atom
                    umma_f16_ts<BN, PAIR>(tmem, ta + 8u * (uint32_t)ks, dx + 2 * ks, (kb | ks) != 0);
                umma_commit<PAIR>(b_ae + 8 * sa);  // the decoded tile and the x tile may be overwritten
                umma_commit<PAIR>(b_xe + 8 * sx);
            }
            umma_commit<PAIR>(b_d);  // accumulator complete
            APBD_STAMP(3);
#ifdef APBD_TL
            APBD_SET(7, (unsigned long long)wa);
            APBD_SET(8, (unsigned long long)wx);
#endif
        }
    } else {
        // =================== decoders, then the epilogue ===================
        // decode warp dw: rows 32q..32q+31 (q = warp & 3, the TMEM lane quarter this
        // warp may write / read).  2 A slots: lane word h of every K block with parity
        // par; 4 A slots: both lane words of every K block kb = ph (mod 4)
        const int dw = warp - 2, q4 = warp & 3;
        const int h = kASlots >= 4 ? 0 : (dw >> 2) & 1, par = kASlots >= 4 ? dw >> 2 : dw >> 3;
        constexpr int kWords = kASlots >= 4 ? 2 : 1;
        const int r = 32 * q4 + lane;
        const int64_t grow = row0 + r;
        // this row's centroid table: u32 [entry][128 rows] (k <= 7), u16 (k = 8); the
        // 4 warps of a row quarter split the entries
        {
            const __half* src = P.lut + (grow < P.rows ? grow : 0) * (int64_t)(1 << K);
            const int part = dw >> 2;
#pragma unroll 4
            for (int e = part; e < (1 << K); e += 4) {
                const uint16_t v = grow < P.rows ? __half_as_ushort(src[e]) : (uint16_t)0;
                if constexpr (K <= 7)
                    *reinterpret_cast<uint32_t*>(smem + Y::kOffT + (e * BM + r) * 4) = v;
                else
                    *reinterpret_cast<uint16_t*>(smem + Y::kOffT + (e * BM + r) * 2) = v;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kDecWarps * 32) : "memory");  // table complete
        if (warp == 2 && lane == 0) APBD_STAMP(6);
        // byte 0 of the table address; bytes 2-3 carry this CTA's shared-window rank bit
        // (bit 24 of the address after the u32 path's << 1), kept by the PRMT below
        const uint32_t rr = ((uint32_t)r << 1) | ((saddr(smem) & 0xFF000000u) >> (K <= 7 ? 1 : 0));
        // this warp's TMEM lane quarter; A slot columns of word h
        const uint32_t t_row = tmem + ((uint32_t)(32 * q4) << 16) + Y::kColA + 16u * (uint32_t)h;
        for (int kb = par; kb < n_kb; kb += (kASlots >= 4 ? 4 : 2)) {
            // this row's lane word(s) of K block kb: plane chunk stage kb / 2, words 2 (kb & 1) + h (+1)
            const int ps = kb >> 1, s = ps % kPStages;
            mbar_wait(b_pf + 8 * s, (ps / kPStages) & 1);
            uint32_t Q[kWords][K];
#pragma unroll
            for (int i = 0; i < K; ++i) {  // Q[.][i] = plane K-1-i (LSB plane first)
                const uint32_t a = sP + s * Y::kPStride + (K - 1 - i) * 2048 + r * 16 + (2 * (kb & 1) + h) * 4;
                if constexpr (kWords == 2) {
                    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(Q[0][i]), "=r"(Q[kWords - 1][i]) : "r"(a));
                } else {
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(Q[0][i]) : "r"(a));
                }
            }
            mbar_arrive(b_pe + 8 * s);
            const int sa = kb % kASlots;
#pragma unroll
            for (int w = 0; w < kWords; ++w) {
                uint32_t W[8];
                apb::to_bytes<K>(Q[w], W);  // W[b] byte p = code of column 256p + 8t + b
                uint32_t v[16];             // K elements 32h + 8p + b as fp16 pairs: column 4p + b/2 of word h
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int b = 0; b < 8; b += 2) {
                        const uint32_t a0 = prmt(W[b], rr, 0x7604u | (uint32_t)(p << 4));  // code << 8 | r << 1
                        const uint32_t a1 = prmt(W[b + 1], rr, 0x7604u | (uint32_t)(p << 4));
                        uint32_t lo, hi;
                        if constexpr (K <= 7) {
                            lo = lds_t32<Y::kTable>(a0 << 1);
                            hi = lds_t32<Y::kTable>(a1 << 1);
                        } else {
                            lo = lds_t16<Y::kTable>(a0);
                            hi = lds_t16<Y::kTable>(a1);
                        }
                        v[4 * p + b / 2] = lo | (hi << 16);
                    }
                if (w == 0) {  // decoded in registers while the MMA may still read the slot: wait only to store
                    if (kb >= kASlots) mbar_wait(b_ae + 8 * sa, ((kb / kASlots) - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                        t_row + 32u * (uint32_t)sa + 16u * (uint32_t)w),
                    "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                    "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                    : "memory");
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            if constexpr (PAIR) {  // the even CTA issues the pair's MMA: one cluster-scope arrive per warp
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(pair_leader(b_af + 8 * sa))
                                 : "memory");
            } else
                mbar_arrive(b_af + 8 * sa);
        }
        // ------------------------------------ epilogue ------------------------------------
        // the 4 warp groups (dw >> 2) split the BN accumulator columns
        mbar_wait(b_d, 0);
        if (warp == 2 && lane == 0) APBD_STAMP(4);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        constexpr int kCols = BN / 4;                  // accumulator columns per warp group
        constexpr int kChunk = kCols < 32 ? kCols : 32;  // tcgen05.ld .x8 / .x16 / .x32
#pragma unroll 1
        for (int c0 = (dw >> 2) * kCols; c0 < ((dw >> 2) + 1) * kCols; c0 += kChunk) {
            uint32_t d[32];
            const uint32_t ta = tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)c0;
            if constexpr (kChunk == 32) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                      "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]),
                      "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]),
                      "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]),
                      "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
                    : "r"(ta));
            } else if constexpr (kChunk == 16) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                      "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]),
                      "=r"(d[15])
                    : "r"(ta));
            } else {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
                               "=r"(d[7])
                             : "r"(ta));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (grow < P.rows && P.splits > 1) {  // split-K: raw partial tile, summed by split_sum_kernel
#pragma unroll
                for (int c = 0; c < kChunk; ++c) {
                    const int n = n0 + c0 + c;
                    if (n < P.mx) P.ws[((int64_t)blockIdx.z * P.mx + n) * P.rows + grow] = __uint_as_float(d[c]);
                }
            } else if (grow < P.rows) {
                if (P.pairs) {  // columns (2i, 2i+1) = (hi, lo) of output row (n0 + c) / 2
#pragma unroll
                    for (int c = 0; c < kChunk; c += 2) {
                        const int m = (n0 + c0 + c) >> 1;
                        if (m < P.m_out)
                            P.y[(int64_t)m * P.ldy + grow] =
                                (__uint_as_float(d[c]) + __uint_as_float(d[c + 1])) * P.inv[m];
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < kChunk; ++c) {
                        const int m = n0 + c0 + c;
                        if (m < P.m_out) P.y[(int64_t)m * P.ldy + grow] = __uint_as_float(d[c]);
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if constexpr (PAIR)
        cluster_sync_all();  // no CTA of the pair leaves while the other may still signal it
    else
        __syncthreads();
    if (threadIdx.x == 0) {
        APBD_STAMP(5);
#ifdef APBD_TL
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        APBD_SET(9, smid);
#endif
    }
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Y::kTmemCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Y::kTmemCols));
    }
}

#ifdef APBD_TL
extern "C" int apbd_read_timeline(unsigned long long* host, int n) {
    return cudaMemcpyFromSymbol(host, g_tld, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 5;
}
#endif

// Activations in the kernel's K order (one CTA per input row): fp16 rows copied,
// or fp32 rows split into scaled (hi, lo) pairs at rows (2i, 2i+1) with 1 / scale
// in inv[i]; columns >= cols are zero.
template <bool F32>
__global__ void __launch_bounds__(256) prep_x_kernel(const void* __restrict__ x, int cols, int64_t ldx,
                                                     __half* __restrict__ xp, int64_t cp, float* __restrict__ inv) {
    const int row = blockIdx.x, t = threadIdx.x;
    float scale = 1.f;
    if constexpr (F32) {
        __shared__ float red[8];
        const float* xr = reinterpret_cast<const float*>(x) + (int64_t)row * ldx;
        float a = 0.f;
        for (int i = t; i < cols; i += 256) a = fmaxf(a, fabsf(xr[i]));
#pragma unroll
        for (int o = 16; o; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
        if ((t & 31) == 0) red[t >> 5] = a;
        __syncthreads();
        a = red[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) a = fmaxf(a, red[w]);
        if (a > 0.f && isfinite(a)) {
            int e;
            frexpf(a, &e);
            scale = ldexpf(1.f, min(max(15 - e, -126), 126));  // max |x| * scale in [2^14, 2^15)
        }
        if (t == 0) inv[row] = 1.f / scale;
    }
    for (int64_t j = t; j < cp; j += 256) {
        const int64_t T = j >> 10;
        const int w = (int)(j & 1023), v = w >> 6, e = w & 63;
        const int64_t c = (T << 10) + 256 * ((e >> 3) & 3) + 16 * v + 8 * (e >> 5) + (e & 7);
        if constexpr (F32) {
            const float xv = c < cols ? reinterpret_cast<const float*>(x)[(int64_t)row * ldx + c] * scale : 0.f;
            const __half h = __float2half_rn(xv);
            xp[(int64_t)(2 * row) * cp + j] = h;
            xp[(int64_t)(2 * row + 1) * cp + j] = __float2half_rn(xv - __half2float(h));
        } else {
            xp[(int64_t)row * cp + j] =
                c < cols ? reinterpret_cast<const __half*>(x)[(int64_t)row * ldx + c] : __ushort_as_half(0);
        }
    }
}

// split-K epilogue: y = sum over splits (fixed order: deterministic) of the raw
// accumulator tiles, (hi, lo) columns added and unscaled for pairs.
__global__ void __launch_bounds__(256) split_sum_kernel(const float* __restrict__ ws, int splits, int mx, int64_t rows,
                                                        int pairs, const float* __restrict__ inv, float* __restrict__ y,
                                                        int64_t ldy, int m_out) {
    const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= (int64_t)m_out * rows) return;
    const int m = (int)(i / rows);
    const int64_t r = i - (int64_t)m * rows;
    float acc = 0.f;
    for (int z = 0; z < splits; ++z) {
        const float* t = ws + (int64_t)z * mx * rows;
        acc += pairs ? t[(int64_t)(2 * m) * rows + r] + t[(int64_t)(2 * m + 1) * rows + r] : t[(int64_t)m * rows + r];
    }
    y[(int64_t)m * ldy + r] = pairs ? acc * inv[m] : acc;
}

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

template <int K, int BN, bool PAIR>
static int launch_bn(DenseParams& P, int64_t rows, cudaStream_t s) {
    static std::atomic<unsigned long long> configured{0};
    static_assert(Lay<BN, K>::kBytes <= 227 * 1024, "shared memory budget");
    auto kern = dense_tc_kernel<K, BN, PAIR>;
    if (!apb::ensure_smem_optin(kern, Lay<BN, K>::kBytes, configured)) return APB_ERR_CUDA;
    int64_t row_tiles = (rows + BM - 1) / BM;
    if (PAIR) row_tiles = (row_tiles + 1) / 2 * 2;  // whole CTA pairs (an all-padding tile reads zeros, stores nothing)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)row_tiles, (unsigned)((P.mx + BN - 1) / BN), (unsigned)P.splits);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Lay<BN, K>::kBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = PAIR ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, kern, P) != cudaSuccess) return APB_ERR_CUDA;
    if (P.splits > 1) {
        const int64_t n = (int64_t)P.m_out * rows;
        split_sum_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P.ws, P.splits, P.mx, rows, P.pairs, P.inv, P.y,
                                                                     P.ldy, P.m_out);
    }
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}
// N tile: the activation rows rounded up to 32 / 64 / 128, or 256 above 128 (a
// decoded weight tile then feeds twice the MMA work); small batches stage only
// the rows they have (the activation tile is shared-memory traffic per K block)
static int pick_bn(int64_t mx) { return mx > 128 ? 256 : (mx > 64 ? 128 : (mx > 32 ? 64 : 32)); }
// CTA pairs (cta_group::2, M = 256) for the 256-wide N tile without split-K:
// each SM of a pair stages and reads half of every activation tile.  Opt-in
// (APB_DENSE_PAIR=1): correct (tests) but measured ~15 % slower than one CTA
// per tile -- every K block then waits for both CTAs' decoders
// (profiles/r2_dense_overlap.md).
static bool pair_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("APB_DENSE_PAIR");
        return e && e[0] == '1';
    }();
    return on;
}
template <int K>
static int launch(DenseParams& P, int64_t rows, cudaStream_t s) {
    switch (pick_bn(P.mx)) {
        case 32: return launch_bn<K, 32, false>(P, rows, s);
        case 64: return launch_bn<K, 64, false>(P, rows, s);
        case 128: return launch_bn<K, 128, false>(P, rows, s);
    }
    if (P.pair) return launch_bn<K, 256, true>(P, rows, s);
    return launch_bn<K, 256, false>(P, rows, s);
}

}  // namespace apbd

extern "C" int apb_dense_prep_x(const void* x, int x_dtype, int64_t m, int64_t cols, int64_t ldx, uint16_t* xp,
                                int64_t padded_cols, float* inv, void* stream) {
    if (!x || !xp || (x_dtype == APB_DTYPE_F32 && !inv)) return APB_ERR_PARAM;
    if (x_dtype != APB_DTYPE_F32 && x_dtype != APB_DTYPE_F16) return APB_ERR_PARAM;
    if (m <= 0 || cols <= 0 || ldx < cols || padded_cols < cols || padded_cols % 1024 || m > INT32_MAX ||
        cols > INT32_MAX)
        return APB_ERR_SHAPE;
    cudaStream_t s = (cudaStream_t)stream;
    if (x_dtype == APB_DTYPE_F32)
        apbd::prep_x_kernel<true><<<(unsigned)m, 256, 0, s>>>(x, (int)cols, ldx, (__half*)xp, padded_cols, inv);
    else
        apbd::prep_x_kernel<false><<<(unsigned)m, 256, 0, s>>>(x, (int)cols, ldx, (__half*)xp, padded_cols, inv);
    return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA;
}

// Split-K factor for a launch of row_blocks x n_tiles output tiles over n_kb K
// blocks: enough CTAs to cover the SMs (deterministic: fixed-order sum).
static int choose_splits(int64_t tiles, int n_kb, int sms) {
    int s = 1;
    while (tiles * s * 2 <= (int64_t)sms && s < 8 && n_kb % (4 * s) == 0 && n_kb / (2 * s) >= 8) s *= 2;  // one wave
    return s;
}

extern "C" int64_t apb_gemm_dense_tc_workspace(int64_t rows, int64_t padded_cols, int64_t mx) {
    if (rows <= 0 || padded_cols <= 0 || mx <= 0) return 0;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int bn = apbd::pick_bn(mx);
    const int64_t tiles = ((rows + apbd::BM - 1) / apbd::BM) * ((mx + bn - 1) / bn);
    const int sp = choose_splits(tiles, (int)(padded_cols / apbd::BK), sms);
    return sp > 1 ? (int64_t)sp * mx * rows * 4 : 0;
}

extern "C" int apb_gemm_dense_tc(const uint8_t* planes, int n_max, int64_t rows, int64_t cols, int64_t padded_cols,
                                 int k, const uint16_t* lut, const uint16_t* xp, int64_t mx, int pairs,
                                 const float* inv, float* y, int64_t ldy, float* ws, int64_t ws_bytes,
                                 void* stream) {
    using namespace apbd;
    if (!planes || !lut || !xp || !y || (pairs && !inv)) return APB_ERR_PARAM;
    if (k < 2 || k > n_max || n_max > 8) return APB_ERR_PARAM;
    if (rows <= 0 || cols <= 0 || padded_cols < cols || padded_cols % 1024 || mx <= 0 || (pairs && (mx & 1)))
        return APB_ERR_SHAPE;
    const int64_t m_out = pairs ? mx / 2 : mx;
    if (ldy < rows || mx > INT32_MAX) return APB_ERR_SHAPE;
    if (((uintptr_t)planes & 15) || ((uintptr_t)xp & 15)) return APB_ERR_PARAM;  // TMA global addresses
    if ((mx + pick_bn(mx) - 1) / pick_bn(mx) > 65535) return APB_ERR_SHAPE;       // grid.y
    if (ws && ((uintptr_t)ws & 3)) return APB_ERR_PARAM;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return APB_ERR_CUDA;
    DenseParams P = {};
    {
        int sms = 148, dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int bn = pick_bn(mx);
        const int64_t tiles = ((rows + BM - 1) / BM) * ((mx + bn - 1) / bn);
        int sp = choose_splits(tiles, (int)(padded_cols / BK), sms);
        if (sp > 1 && (!ws || ws_bytes < (int64_t)sp * mx * rows * 4)) sp = 1;  // no workspace: one pass
        P.splits = sp;
        P.ws = ws;
        P.n_kb = (int)(padded_cols / BK) / sp;
    }
    P.pair = pick_bn(mx) == 256 && P.splits == 1 && rows > BM && pair_enabled() ? 1 : 0;
    {
        const cuuint64_t dims[2] = {(cuuint64_t)padded_cols, (cuuint64_t)mx};
        const cuuint64_t strides[1] = {(cuuint64_t)padded_cols * 2};
        const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)(pick_bn(mx) >> P.pair)}, es[2] = {1, 1};  // N tile / CTA
        if (enc(&P.tm_x, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)xp, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return APB_ERR_CUDA;
    }
    {
        const int64_t rb = padded_cols / 8;
        const cuuint64_t dims[3] = {(cuuint64_t)rb, (cuuint64_t)rows, (cuuint64_t)n_max};
        const cuuint64_t strides[2] = {(cuuint64_t)rb, (cuuint64_t)(rows * rb)};
        const cuuint32_t box[3] = {16, (cuuint32_t)BM, (cuuint32_t)k}, es[3] = {1, 1, 1};
        if (enc(&P.tm_planes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)planes, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return APB_ERR_CUDA;
    }
    P.lut = reinterpret_cast<const __half*>(lut);
    P.y = y;
    P.inv = inv;
    P.rows = rows;
    P.ldy = ldy;
    P.mx = (int)mx;
    P.m_out = (int)m_out;
    P.pairs = pairs ? 1 : 0;
    cudaStream_t s = (cudaStream_t)stream;
    switch (k) {
        case 2: return launch<2>(P, rows, s);
        case 3: return launch<3>(P, rows, s);
        case 4: return launch<4>(P, rows, s);
        case 5: return launch<5>(P, rows, s);
        case 6: return launch<6>(P, rows, s);
        case 7: return launch<7>(P, rows, s);
        case 8: return launch<8>(P, rows, s);
    }
    return APB_ERR_PARAM;
}
