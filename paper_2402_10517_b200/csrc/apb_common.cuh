// apb_common.cuh -- shared device helpers for the B200 bitplane kernels.
//
// Geometry of the reference layout (bitplane.py:23-37, engine.py:187-195):
//   a 1024-weight tile is 128 bytes per plane; in the permuted layout the
//   32-bit little-endian word of lane t (bytes 4t..4t+3) holds, in byte j,
//   bit i, the code bit of weight 256*j + 8*t + i.  So bit position b of a
//   lane word (b = 8j + i) is column 256*(b>>3) + 8*t + (b&7) of the tile.
//
// Bit networks.  Both take Q[i] = the lane word of code bit i (LSB plane
// first, i.e. Q[i] = plane k-1-i, as engine.py:90-91 feeds its transpose) and
// gather every weight's code bits together with masked 1/2/4-bit interleaves
// (select-form delta swaps: one LOP3 plus one shift each, the shift on the
// FMA pipe when it is a left shift).
//
//   to_bytes<KB>: W[b] byte p = code of bit position 8p + b (b = 0..7).
//     For k = 5..8 this is exactly transpose_any_width's B = 8 output
//     (engine.py:75-92: word g, field s = code of bitpos s*B + g).
//   to_pairs<KB> (k <= 4): U[j] byte p = "pair index" of bit positions
//     (8p + 2j, 8p + 2j + 1) = two ADJACENT columns, with pair-index bit 2i =
//     code bit i of the even column and bit 2i+1 = code bit i of the odd
//     column.  This is the paper's merged lookup (PAPER.md:298-300,
//     engine.py:95-120, 220-236) generalised to k <= 4 and re-arranged so the
//     pair matches an fp16x2 activation pair in memory.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace apb {

// Host side: the dynamic shared-memory opt-in is a per-DEVICE function
// attribute; one flag bit per device (a process may drive several GPUs).
#include <atomic>
#include <cuda_runtime.h>
template <typename Kern>
static inline bool ensure_smem_optin(Kern kern, int bytes, std::atomic<unsigned long long>& done) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return true;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
    if (bit) done.fetch_or(bit, std::memory_order_release);
    return true;
}

constexpr int kTileWeights = 1024;
constexpr int kTileBytes = 128;

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

// Bitwise select: bits of a where m = 1, bits of b where m = 0 (one LOP3).
__device__ __forceinline__ uint32_t sel(uint32_t m, uint32_t a, uint32_t b) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "r"(m));
    return r;
}

// One select-form delta swap stage between a "low" word X and a "high" word
// Y with group width d and mask m (m = groups of d ones, e.g. 0x33333333):
//   lo_out = (X & m) | ((Y << d) & ~m)    high_out = ((X >> d) & m) | (Y & ~m)
// LIVE_X / LIVE_Y say whether X / Y can be non-zero (compile time), so zero
// planes of k < 8 cost nothing.
// Logical right shift.  (Measured: moving it to the FMA pipe as the high
// word of X * 2^(32-D) -- IMAD.HI -- is slower on B200 than SHF on the ALU.)
template <int D>
__device__ __forceinline__ uint32_t shr_fma(uint32_t X) {
    return X >> D;
}

template <bool LX, bool LY, int D>
__device__ __forceinline__ void interleave(uint32_t X, uint32_t Y, uint32_t m, uint32_t& lo,
                                           uint32_t& hi) {
    if constexpr (LX && LY) {
        lo = sel(m, X, Y << D);
        hi = sel(m, shr_fma<D>(X), Y);
    } else if constexpr (LX) {
        lo = X & m;
        hi = shr_fma<D>(X) & m;
    } else if constexpr (LY) {
        lo = (Y << D) & ~m;
        hi = Y & ~m;
    } else {
        lo = 0u;
        hi = 0u;
    }
}

template <int KB>
__device__ __forceinline__ void to_bytes(const uint32_t* Q, uint32_t* W) {
    // Level 1: planes (2a, 2a+1), 1-bit groups.  E: bitpos 2n, O: bitpos 2n+1.
    uint32_t E[4], O[4];
#define APB_L1(a)                                                                          \
    interleave<(2 * (a) < KB), (2 * (a) + 1 < KB), 1>((2 * (a) < KB) ? Q[(2 * (a)) % KB] : 0u, \
                                                      (2 * (a) + 1 < KB) ? Q[(2 * (a) + 1) % KB] : 0u, \
                                                      0x55555555u, E[a], O[a]);
    APB_L1(0) APB_L1(1) APB_L1(2) APB_L1(3)
#undef APB_L1
    constexpr bool L0 = KB > 0, L1 = KB > 2, L2 = KB > 4, L3 = KB > 6;  // plane-pair liveness
    // Level 2: plane pairs -> nibbles.  N[b0][c][b1]: bitpos 4n + b0 + 2 b1, planes 4c..4c+3.
    uint32_t N[2][2][2];
    interleave<L0, L1, 2>(E[0], E[1], 0x33333333u, N[0][0][0], N[0][0][1]);
    interleave<L0, L1, 2>(O[0], O[1], 0x33333333u, N[1][0][0], N[1][0][1]);
    interleave<L2, L3, 2>(E[2], E[3], 0x33333333u, N[0][1][0], N[0][1][1]);
    interleave<L2, L3, 2>(O[2], O[3], 0x33333333u, N[1][1][0], N[1][1][1]);
    // Level 3: nibbles -> bytes.  W[b] byte p: bitpos 8p + b.
    constexpr bool LA = L0 || L1, LB = L2 || L3;
#pragma unroll
    for (int b0 = 0; b0 < 2; ++b0)
#pragma unroll
        for (int b1 = 0; b1 < 2; ++b1)
            interleave<LA, LB, 4>(N[b0][0][b1], N[b0][1][b1], 0x0F0F0F0Fu, W[b0 + 2 * b1],
                                  W[4 + b0 + 2 * b1]);
}

template <int KB>
__device__ __forceinline__ void to_pairs(const uint32_t* Q, uint32_t* U) {
    static_assert(KB >= 1 && KB <= 4, "pair network covers k <= 4");
    const uint32_t A = Q[0], B = Q[(1) % KB], C = Q[(2) % KB], D = Q[(3) % KB];
    uint32_t D1, E1, D2, E2;
    // 2-bit column groups of planes (0,1) and (2,3): nibble n = bitpos (4n,4n+1) / (4n+2,4n+3)
    interleave<true, (KB > 1), 2>(A, B, 0x33333333u, D1, E1);
    interleave<(KB > 2), (KB > 3), 2>(C, D, 0x33333333u, D2, E2);
    // nibbles -> bytes: U[j] byte p = pair index of bitpos (8p+2j, 8p+2j+1)
    interleave<true, (KB > 2), 4>(D1, D2, 0x0F0F0F0Fu, U[0], U[2]);
    interleave<true, (KB > 2), 4>(E1, E2, 0x0F0F0F0Fu, U[1], U[3]);
}

// Pair index -> (even code, odd code), inverse of the to_pairs bit layout.
template <int K>
__host__ __device__ __forceinline__ void pair_codes(uint32_t idx, uint32_t& ce, uint32_t& co) {
    ce = 0;
    co = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        ce |= ((idx >> (2 * i)) & 1u) << i;
        co |= ((idx >> (2 * i + 1)) & 1u) << i;
    }
}

// 4x4 byte transpose: out[j] byte i = in[i] byte j.
__device__ __forceinline__ void byte_transpose4(const uint32_t* in, uint32_t* out) {
    const uint32_t t01l = prmt(in[0], in[1], 0x5140u);  // [a0 b0 a1 b1]
    const uint32_t t01h = prmt(in[0], in[1], 0x7362u);  // [a2 b2 a3 b3]
    const uint32_t t23l = prmt(in[2], in[3], 0x5140u);
    const uint32_t t23h = prmt(in[2], in[3], 0x7362u);
    out[0] = prmt(t01l, t23l, 0x5410u);
    out[1] = prmt(t01l, t23l, 0x7632u);
    out[2] = prmt(t01h, t23h, 0x5410u);
    out[3] = prmt(t01h, t23h, 0x7632u);
}

__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint2 ldg_stream8(const void* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t ldg_stream4(const void* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

}  // namespace apb
