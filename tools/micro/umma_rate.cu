// umma_rate.cu -- tcgen05.mma kind::f16 issue rate on one B200, per SM, with the
// A operand in tensor memory ("ts", what apb_dense_tc.cu does) or in shared
// memory ("ss"), M = 128, N = 256 / 128, K = 16 per instruction, fp32 accumulate.
// One CTA per SM, one elected thread issues NITER x 4 MMAs into one accumulator
// (the dense kernel's per-K-block pattern), one commit at the end; clock64 around
// the issue + wait.  Operand contents are garbage (rate only).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_rate umma_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
template <int BN>
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

template <int BN, bool A_TMEM>
__global__ void __launch_bounds__(128, 1) umma_kernel(int niter, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    const uint32_t sA = saddr(smem), sB = saddr(smem + 16384);  // A: 128 x 64 K (16 KB), B: BN x 64 K
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        const uint64_t db = sw128_desc(sB), da = sw128_desc(sA);
        const uint32_t ta = tmem + 256;  // A columns after a 256-column accumulator
        const long long t0 = clock64();
        for (int it = 0; it < niter; ++it) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint32_t acc = (it | ks) != 0;
                if constexpr (A_TMEM) {
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                        "r"(ta + 8u * ks), "l"(db + 2 * ks), "n"(kIdesc<BN>), "r"(acc));
                } else {
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                        "l"(da + 2 * ks), "l"(db + 2 * ks), "n"(kIdesc<BN>), "r"(acc));
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, 1000000;\n\t"
            "@!p bra W_%=;\n\t}" ::"r"(saddr(&bar))
            : "memory");
        cycles[blockIdx.x] = (unsigned long long)(clock64() - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int BN, bool A_TMEM>
static void run(const char* name) {
    const int sms = 148, niter = 4096;
    unsigned long long* d;
    cudaMalloc(&d, sms * sizeof(unsigned long long));
    auto k = umma_kernel<BN, A_TMEM>;
    const int smem = 16384 + BN * 128 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<sms, 128, smem>>>(16, d);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<sms, 128, smem>>>(niter, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i] / sms;
    const double flop_per_mma = 2.0 * 128 * BN * 16;
    const double n_mma = 4.0 * niter;
    printf("%-28s %s: %7.1f cycles / MMA (128x%dx16), %6.0f flop/clk/SM, %7.1f TFLOP/s device (event %.3f ms)\n", name,
           cudaGetErrorString(cudaGetLastError()), mean / n_mma, BN, flop_per_mma * n_mma / mean,
           flop_per_mma * n_mma * sms / (ms * 1e-3) / 1e12, ms);
    cudaFree(d);
}

int main() {
    run<256, true>("A in TMEM, N = 256");
    run<256, false>("A in smem, N = 256");
    run<128, true>("A in TMEM, N = 128");
    run<128, false>("A in smem, N = 128");
    return 0;
}
