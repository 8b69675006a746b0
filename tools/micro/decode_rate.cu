// Microbenchmark: compute ceiling of the GEMV inner loop with everything
// resident in shared memory (no TMA, no HBM): weights decoded per SM-cycle for
//   MAP 0: the round-1 "row-copy" lane mapping of gemv7 (16-row items, 2 lanes
//          per row, 2 table copies per row, 8 live x lanes, LDS.64 x per word)
//   MAP 1: "lane = row" mapping (32-row items, 1 table copy per row, lanes of
//          a quad q process words t0+2q / t0+2q+1 as MMA column sets A / B,
//          x as one LDS.128 per live lane per two HMMAs)
// k = 3..8; pair tables for k <= 4, single (v, 0) tables for k >= 5 (PACK=1: one
// IMAD per pair; PACK=0: separate (v,0) / (0,v) tables and one HMMA per half).
// Usage: decode_rate  (prints one line per variant)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include "../../paper_2402_10517_b200/csrc/apb_common.cuh"

using apb::prmt;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds64_keep(uint32_t& v0, uint32_t& v1, uint32_t a, uint32_t pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t@p ld.shared.v2.u32 {%0,%1}, [%2];\n\t}"
                 : "+r"(v0), "+r"(v1) : "r"(a), "r"(pred));
}
__device__ __forceinline__ void lds128_keep(uint32_t& v0, uint32_t& v1, uint32_t& v2, uint32_t& v3, uint32_t a, uint32_t pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t@p ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
                 : "+r"(v0), "+r"(v1), "+r"(v2), "+r"(v3) : "r"(a), "r"(pred));
}
template <int IMM>
__device__ __forceinline__ uint32_t lds_t(uint32_t off) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(off), "n"(IMM));
    return v;
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

constexpr int kTableOff = 1024;   // table region
constexpr int kTable2 = 65536;    // second (0, v) table for PACK = 0
constexpr int kPlaneOff = 140 * 1024;
constexpr int kXOff = 136 * 1024;

// decode one lane word into 16 fp16x2 values (pairs) -- PACK variants for k >= 5
template <int K, int PACK>
__device__ __forceinline__ void decode(const uint32_t* Q, uint32_t off, uint32_t* out, uint32_t* out2) {
    if constexpr (K <= 4) {
        uint32_t U[4];
        apb::to_pairs<K>(Q, U);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) out[p * 4 + j] = lds_t<kTableOff>(prmt(U[j], off, 0x7604u | (uint32_t)(p << 4)));
    } else {
        uint32_t Wb[8];
        apb::to_bytes<K>(Q, Wb);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const uint32_t sel = 0x7604u | (uint32_t)(p << 4);
                const uint32_t e = lds_t<kTableOff>(prmt(Wb[2 * j], off, sel));
                if constexpr (PACK) {
                    const uint32_t o = lds_t<kTableOff>(prmt(Wb[2 * j + 1], off, sel));
                    out[p * 4 + j] = e + (o << 16);
                } else {
                    out[p * 4 + j] = e;
                    out2[p * 4 + j] = lds_t<kTableOff + kTable2>(prmt(Wb[2 * j + 1], off, sel));
                }
            }
    }
}

// MAP 0: round-1 mapping.  Each warp: group grp = warp/4 of NG, su = warp&3; a
// "stage" = 16 rows x 128 B x K planes (K*2 KB); warps loop over NST stages.
template <int K, int PACK>
__global__ void __launch_bounds__(512, 1) map0(int iters, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3, rho = 2 * g + (q >> 1), cp = q & 1, su = warp & 3;
    const int NST = 4;
    uint32_t plane_off[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) plane_off[j] = rho * 128 + (((su + 4 * j) ^ (rho & 7)) << 4) + cp * 8;
    const int gset = (g >> 1) & 1;
    const uint32_t xlive = (q >> 1) == (g & 1) && (g >> 2) == 0;
    const uint32_t xrow = saddr(smem + kXOff) + (uint32_t)(32 * su + 16 * cp + 4 * gset) * 2u;
    const uint32_t off = (uint32_t)lane * 4u;
    uint32_t xv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float acc[2][4] = {};
    const uint32_t ring = saddr(smem + kPlaneOff);
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        const uint32_t sb = ring + (uint32_t)((it + (warp >> 2)) % NST) * (K * 2048);
        const int tile = it & 3;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            uint2 pv[K];
#pragma unroll
            for (int p = 0; p < K; ++p) pv[K - 1 - p] = lds64(sb + p * 2048 + plane_off[j]);
#pragma unroll
            for (int wi = 0; wi < 2; ++wi) {
                const uint32_t xa = xrow + (uint32_t)(tile * 1024 + 128 * j + 8 * wi) * 2u;
#pragma unroll
                for (int p = 0; p < 4; ++p) lds64_keep(xv[2 * p], xv[2 * p + 1], xa + 512 * p, xlive);
                uint32_t Q[K];
#pragma unroll
                for (int i = 0; i < K; ++i) Q[i] = wi ? pv[i].y : pv[i].x;
                uint32_t a[16], a2[16];
                decode<K, PACK>(Q, off, a, a2);
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    mma16816(acc[p & 1], a[p * 4 + 0], a[p * 4 + 2], a[p * 4 + 1], a[p * 4 + 3], xv[2 * p], xv[2 * p + 1]);
                    if constexpr (K >= 5 && !PACK)
                        mma16816(acc[p & 1], a2[p * 4 + 0], a2[p * 4 + 2], a2[p * 4 + 1], a2[p * 4 + 3], xv[2 * p], xv[2 * p + 1]);
                }
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 4; ++i) s += acc[0][i] + acc[1][i];
    out[blockIdx.x * blockDim.x + tid] = s;
    if (tid == 0) out[1 << 20 | blockIdx.x] = (float)(t1 - t0);
}

// MAP 0 + a concurrent HBM stream from the last two warps of the CTA:
// MODE 1: LDG.128 (L1::no_allocate) streaming, MODE 2: cp.async.bulk (TMA) into
// a smem scratch ring.  Measures whether plane bytes arriving through the L1TEX
// data path or TMA writes take shared-memory bandwidth from the LUT lookups.
__device__ __forceinline__ void mbar_init2(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait2(uint32_t a, uint32_t parity) {
    // try_wait with a suspend-time hint: the waiting thread sleeps in the barrier unit
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t@!p bra W_%=;\n\t}" ::"r"(a), "r"(parity), "r"(1000000) : "memory");
}
__device__ CUtensorMap g_tmap_c;
__device__ const CUtensorMap* g_tmap;
template <int K, int MODE, int SZ = 4096>
__global__ void __launch_bounds__(640, 1) map0s(int iters, float* out, const uint4* src, size_t n16) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ int done_cnt;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) done_cnt = 0;
    __syncthreads();
    volatile int* stop = &done_cnt;
    const long long tstart = clock64();
    if (warp >= 16) {
        if (MODE == 2 && warp > 16) return;
        if (MODE == 0) return;
        if (MODE == 6) {  // control: one thread polling the stop flag with nanosleep, no copies
            if (warp != 16 || lane != 0) return;
            while (*stop < 16) __nanosleep(2000);
            out[(1 << 21) + blockIdx.x * 2] = 0.f;
            return;
        }
        uint32_t accx = 0;
        size_t i = ((size_t)blockIdx.x * 2 + (warp - 16)) * 32 * 8 + lane;
        const size_t stride = (size_t)gridDim.x * 2 * 32 * 8;
        if (MODE == 1 || MODE == 3) {
            // MODE 1: coalesced (a warp reads 512 contiguous bytes per LDG.128)
            // MODE 3: row-strided (lane l reads 16 B of "row" l, rows 1 KB apart: 32 lines per instruction)
            long long bytes = 0;
            const int sw = warp - 16;  // 0..3
            const char* base = (const char*)src;
            const size_t total = n16 * 16 - (1 << 20);
            size_t pos = ((size_t)blockIdx.x * 4 + sw) * 65536;
            const size_t step = (size_t)gridDim.x * 4 * 65536;
            while (*stop < 16) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const size_t o = MODE == 1 ? pos + u * 512 + lane * 16 : pos + (size_t)lane * 1024 + u * 16;
                    uint4 v = apb::ldg_stream16(base + o);
                    accx ^= v.x ^ v.w;
                }
                pos += MODE == 1 ? 4096 : 32768;
                if (pos + 65536 >= total) pos = ((size_t)blockIdx.x * 4 + sw) * 65536;
                bytes += 8 * 512;
            }
            if (lane == 0) atomicAdd(out + (1 << 21) + blockIdx.x * 2, (float)bytes);
        } else {
            if (warp != 16 || lane != 0) return;
            // 16 x 4 KB ring at [kXOff - 64 KB, kXOff), barriers after the planes region
            constexpr int NR = 65536 / SZ > 16 ? 16 : 65536 / SZ;
            const uint32_t ring = saddr(smem + kXOff - 65536), bar = saddr(smem + kPlaneOff - 256);
            for (int j = 0; j < NR; ++j) mbar_init2(bar + 8 * j, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            long long bytes = 0;
            int it = 0;
            size_t off = (size_t)blockIdx.x * 4096;
            int row = blockIdx.x * 16;
            while (*stop < 16) {
                const int j = it % NR;
                if (it >= NR) mbar_wait2(bar + 8 * j, ((it / NR) - 1) & 1);
                asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;\n\t}" ::"r"(bar + 8 * j), "r"(MODE == 2 ? SZ : 4096) : "memory");
                if (MODE == 2) {
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(ring + SZ * j),
                                 "l"((const char*)src + off % (n16 * 16 - SZ)), "r"(SZ), "r"(bar + 8 * j) : "memory");
                } else {
                    // two 2 KB boxes {128 B, 16 rows, 1 plane} of a [8 planes][rows][1024 B] u8 tensor, 128B swizzle
                    for (int h = 0; h < 2; ++h)
                        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(ring + 4096 * j + 2048 * h),
                                     "l"(g_tmap), "r"((int)((it * 2 + h) % 8) * 128), "r"(row % 65536), "r"(h), "r"(bar + 8 * j) : "memory");
                    row += 16 * 148;
                }
                off += (size_t)gridDim.x * (MODE == 2 ? SZ : 4096);
                bytes += MODE == 2 ? SZ : 4096;
                ++it;
            }
            for (int j = 0; j < NR && j < it; ++j) mbar_wait2(bar + 8 * ((it - 1 - j) % NR), ((it - 1 - j) / NR) & 1);
            out[(1 << 21) + blockIdx.x * 2] = (float)bytes;
            return;
        }
        out[blockIdx.x * blockDim.x + tid] = (float)accx;
        return;
    }
    const int g = lane >> 2, q = lane & 3, rho = 2 * g + (q >> 1), cp = q & 1, su = warp & 3;
    const int NST = 4;
    uint32_t plane_off[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) plane_off[j] = rho * 128 + (((su + 4 * j) ^ (rho & 7)) << 4) + cp * 8;
    const int gset = (g >> 1) & 1;
    const uint32_t xlive = (q >> 1) == (g & 1) && (g >> 2) == 0;
    const uint32_t xrow = saddr(smem + kXOff) + (uint32_t)(32 * su + 16 * cp + 4 * gset) * 2u;
    const uint32_t off = (uint32_t)lane * 4u;
    uint32_t xv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float acc[2][4] = {};
    const uint32_t ringp = saddr(smem + kPlaneOff);
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        const uint32_t sb = ringp + (uint32_t)((it + (warp >> 2)) % NST) * (K * 2048);
        const int tile = it & 3;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            uint2 pv[K];
#pragma unroll
            for (int p = 0; p < K; ++p) pv[K - 1 - p] = lds64(sb + p * 2048 + plane_off[j]);
#pragma unroll
            for (int wi = 0; wi < 2; ++wi) {
                const uint32_t xa = xrow + (uint32_t)(tile * 1024 + 128 * j + 8 * wi) * 2u;
#pragma unroll
                for (int p = 0; p < 4; ++p) lds64_keep(xv[2 * p], xv[2 * p + 1], xa + 512 * p, xlive);
                uint32_t Q[K];
#pragma unroll
                for (int i = 0; i < K; ++i) Q[i] = wi ? pv[i].y : pv[i].x;
                uint32_t a[16], a2[16];
                decode<K, 1>(Q, off, a, a2);
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    mma16816(acc[p & 1], a[p * 4 + 0], a[p * 4 + 2], a[p * 4 + 1], a[p * 4 + 3], xv[2 * p], xv[2 * p + 1]);
            }
        }
    }
    float s = 0;
    for (int i = 0; i < 4; ++i) s += acc[0][i] + acc[1][i];
    out[blockIdx.x * blockDim.x + tid] = s;
    __syncwarp();
    if (lane == 0) {
        out[(1 << 20) + blockIdx.x * 16 + warp] = (float)(clock64() - tstart);
        atomicAdd((int*)&done_cnt, 1);
    }
}

// MAP 1: lane = row.  lane (g, q) owns row 8q + ((g + 4(q>>1)) & 7) of a 32-row
// item; per step the quad q takes words t0+2q (set A) / t0+2q+1 (set B) of its
// row; a "stage" = 32 rows x 128 B x K planes; 4 steps (t0 = 0, 8, 16, 24) per
// stage split over the 4 warps of a group -> one step per warp per stage.
template <int K, int PACK>
__global__ void __launch_bounds__(512, 1) map1(int iters, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3, su = warp & 3;
    const int row = 8 * q + ((g + 4 * (q >> 1)) & 7);
    const int NST = 2;
    // words t0+2q, t0+2q+1 with t0 = 8 su: 16-B chunk 2su + (q>>1), half q&1
    const uint32_t plane_off = row * 128 + ((((2 * su + (q >> 1))) ^ (row & 7)) << 4) + (q & 1) * 8;
    // live x lanes: set A col n: (g = n, q = n); set B col n+4: (g = n+4, q = n)
    const int xn = g & 3;
    const uint32_t xlive = q == xn;
    const uint32_t xsetb = g >> 2;  // 0: set A (word t0+2q), 1: set B (t0+2q+1)
    const uint32_t xbase = saddr(smem + kXOff) + (uint32_t)(8 * (8 * su + 2 * xn + xsetb)) * 2u;
    const uint32_t off = (uint32_t)lane * 4u;
    uint32_t xv[4][4] = {};
    float acc[2][4] = {};
    const uint32_t ring = saddr(smem + kPlaneOff);
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        const uint32_t sb = ring + (uint32_t)((it + (warp >> 2)) % NST) * (K * 4096);
        const int tile = it & 3;
        uint2 pv[K];
#pragma unroll
        for (int p = 0; p < K; ++p) pv[K - 1 - p] = lds64(sb + p * 4096 + plane_off);
        // x: column 256p + 8t + 0..7 for p = 0..3 (t = word of this lane's quad / set)
#pragma unroll
        for (int p = 0; p < 4; ++p)
            lds128_keep(xv[p][0], xv[p][1], xv[p][2], xv[p][3], xbase + (uint32_t)(tile * 1024 + 256 * p) * 2u, xlive);
        uint32_t QA[K], QB[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            QA[i] = pv[i].x;
            QB[i] = pv[i].y;
        }
        uint32_t aA[16], aB[16], aA2[16], aB2[16];
        decode<K, PACK>(QA, off, aA, aA2);
        decode<K, PACK>(QB, off, aB, aB2);
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                mma16816(acc[hh], aA[p * 4 + 2 * hh], aB[p * 4 + 2 * hh], aA[p * 4 + 2 * hh + 1], aB[p * 4 + 2 * hh + 1],
                         xv[p][2 * hh], xv[p][2 * hh + 1]);
                if constexpr (K >= 5 && !PACK)
                    mma16816(acc[hh], aA2[p * 4 + 2 * hh], aB2[p * 4 + 2 * hh], aA2[p * 4 + 2 * hh + 1],
                             aB2[p * 4 + 2 * hh + 1], xv[p][2 * hh], xv[p][2 * hh + 1]);
            }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 4; ++i) s += acc[0][i] + acc[1][i];
    out[blockIdx.x * blockDim.x + tid] = s;
    if (tid == 0) out[1 << 20 | blockIdx.x] = (float)(t1 - t0);
}

__global__ void fill(uint32_t* p, int n) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x) {
        uint32_t h = i * 2654435761u;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        p[i] = h & 0x3BFF3BFFu;
    }
}

template <typename F>
static int run(const char* name, F kern, int K, int weights_per_iter_warp, int warps, int cps) {
    const int smem = 227 * 1024 / cps - 1024;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    float* out;
    CK(cudaMalloc(&out, (2 << 20) * 4));
    const int iters = 4000;
    kern<<<148 * cps, warps * 32, smem>>>(16, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<148 * cps, warps * 32, smem>>>(iters, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double w = (double)148 * cps * warps * iters * weights_per_iter_warp;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cyc = ms * 1e-3 * clk * 1e3;
    const double wpc = w / 148 / cyc;
    const double need = 6544.3e9 * 8.0 / K / (148.0 * clk * 1e3);  // w/clk/SM at the HBM peak
    printf("%-22s k=%d warps=%2d x%d CTA: %6.1f w/clk/SM  -> %5.1f%% of HBM-peak rate  (%.3f ms)\n", name, K, warps, cps, wpc,
           100.0 * wpc / need, ms);
    cudaFree(out);
    return 0;
}

template <int K, int PACK>
static void suite() {
    // MAP 0: per warp-iteration 2 j x 2 wi x 32 lanes x 32 weights = 4096
    run("map0 rowcopy", map0<K, PACK>, K, 4096, 16, 1);
    // MAP 1: per warp-iteration 2 words x 32 lanes x 32 = 2048
    run("map1 lane=row", map1<K, PACK>, K, 2048, 16, 1);
}

template <int K, int MODE, int SZ = 4096>
static int run_stream(const char* name) {
    const int smem = 227 * 1024 - 2048;
    auto kern = map0s<K, MODE, SZ>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    float* out;
    CK(cudaMalloc(&out, (4 << 20) * 4));
    size_t n16 = (size_t)1 << 26;  // 1 GiB
    uint4* src;
    CK(cudaMalloc(&src, n16 * 16));
    CK(cudaMemset(src, 1, n16 * 16));
    const int iters = 4000;
    CK(cudaMemset(out, 0, (4 << 20) * 4));
    kern<<<148, 640, smem>>>(16, out, src, n16);
    CK(cudaDeviceSynchronize());
    CK(cudaMemset(out, 0, (4 << 20) * 4));
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<148, 640, smem>>>(iters, out, src, n16);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    static float h[(1 << 21) + 512];
    CK(cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost));
    double cyc = 0, bytes = 0;
    for (int c = 0; c < 148; ++c) {
        for (int w = 0; w < 16; ++w) cyc = std::max(cyc, (double)h[(1 << 20) + c * 16 + w]);
        bytes += h[(1 << 21) + c * 2];
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double wpc = (double)16 * iters * 4096 / cyc;  // per SM
    printf("%-26s k=%d compute %6.1f w/clk/SM (%.0f cyc)  stream %.0f GB/s over %.3f ms (%.1f B/clk/SM)\n", name, K, wpc, cyc,
           bytes / (ms * 1e-3) * 1e-9, ms, bytes / 148 / (ms * 1e-3 * clk * 1e3));
    cudaFree(out);
    cudaFree(src);
    return 0;
}


// MAP 0 with a compact shared-memory layout (table | x | planes) so that CPS CTAs
// of W warps fit per SM: tests the shipped configuration (2 CTAs x 8 warps, <= 96 regs)
template <int K, int W, int CPS>
__global__ void __launch_bounds__(W * 32, CPS) map0c(int iters, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kTab = (K <= 4 ? (1 << (2 * K)) : (1 << K)) * 256;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3, rho = 2 * g + (q >> 1), cp = q & 1, su = warp & 3;
    const int NST = 4;
    uint32_t plane_off[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) plane_off[j] = rho * 128 + (((su + 4 * j) ^ (rho & 7)) << 4) + cp * 8;
    const int gset = (g >> 1) & 1;
    const uint32_t xlive = (q >> 1) == (g & 1) && (g >> 2) == 0;
    const uint32_t xrow = saddr(smem + kTab) + (uint32_t)(32 * su + 16 * cp + 4 * gset) * 2u;
    const uint32_t off = (uint32_t)lane * 4u;
    uint32_t xv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float acc[2][4] = {};
    const uint32_t ring = saddr(smem + kTab + 8192);
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        const uint32_t sb = ring + (uint32_t)((it + (warp >> 2)) % NST) * (K * 2048);
        const int tile = it & 3;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            uint2 pv[K];
#pragma unroll
            for (int p = 0; p < K; ++p) pv[K - 1 - p] = lds64(sb + p * 2048 + plane_off[j]);
#pragma unroll
            for (int wi = 0; wi < 2; ++wi) {
                const uint32_t xa = xrow + (uint32_t)(tile * 1024 + 128 * j + 8 * wi) * 2u;
#pragma unroll
                for (int p = 0; p < 4; ++p) lds64_keep(xv[2 * p], xv[2 * p + 1], xa + 512 * p, xlive);
                uint32_t Q[K];
#pragma unroll
                for (int i = 0; i < K; ++i) Q[i] = wi ? pv[i].y : pv[i].x;
                uint32_t a[16], a2[16];
                decode<K, 1>(Q, off, a, a2);
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    mma16816(acc[p & 1], a[p * 4 + 0], a[p * 4 + 2], a[p * 4 + 1], a[p * 4 + 3], xv[2 * p], xv[2 * p + 1]);
            }
        }
    }
    long long t1 = clock64();
    float sacc = 0;
    for (int i = 0; i < 4; ++i) sacc += acc[0][i] + acc[1][i];
    out[blockIdx.x * blockDim.x + tid] = sacc;
    if (tid == 0) out[1 << 20 | blockIdx.x] = (float)(t1 - t0);
}

template <int K, int W, int CPS>
static int run_c(const char* name) {
    constexpr int kTab = (K <= 4 ? (1 << (2 * K)) : (1 << K)) * 256;
    const int smem = kTab + 8192 + 4 * K * 2048 + 1024;
    auto kern = map0c<K, W, CPS>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    float* out;
    CK(cudaMalloc(&out, (2 << 20) * 4));
    const int iters = 4000;
    kern<<<148 * CPS, W * 32, smem>>>(16, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<148 * CPS, W * 32, smem>>>(iters, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double w = (double)148 * CPS * W * iters * 4096;
    const double wpc = w / 148 / (ms * 1e-3 * clk * 1e3);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    printf("%-28s k=%d %d CTA x %2d warps (%d regs, %d B smem): %6.1f w/clk/SM\n", name, K, CPS, W, fa.numRegs, smem, wpc);
    cudaFree(out);
    return 0;
}

int main() {
    uint32_t* dummy;
    cudaMalloc(&dummy, 4);
    // profiles/r2_cta_shape.txt (CTAs per SM x warps) and r2_cta8.txt (8-warp CTAs)
    run_c<3, 16, 1>("compact 1x16");
    run_c<3, 8, 1>("compact 1x8");
    run_c<3, 8, 2>("compact 2x8 (shipped shape)");
    run_c<3, 16, 2>("compact 2x16");
    run_c<5, 8, 2>("compact 2x8");
    run_c<5, 16, 1>("compact 1x16");
    run_c<5, 8, 1>("compact 1x8");
    run_c<8, 12, 1>("compact 1x12");
    run_c<8, 8, 1>("compact 1x8");
    return 0;
}
