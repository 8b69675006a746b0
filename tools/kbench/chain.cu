// chain: per-launch / per-CTA timeline of one bench step (24 GEMV launches:
// per k = 3..8: grouped q/k/v | o | grouped gate/up | down, PDL, CUDA graph),
// instrumented v7 build (APB_TIMELINE).  Prints, per launch: first CTA start,
// last CTA end, gap to the previous launch's end, and phase medians.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../include/anyprec_b200.h"
extern "C" int apb7_read_timeline(unsigned long long* host, int n);
extern "C" void apb7_timeline_reset(void);
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)
__global__ void fill(uint8_t* p, size_t n, uint32_t s) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { uint32_t h = (uint32_t)i * 2654435761u ^ s; h ^= h >> 13; h *= 0x5bd1e995u; p[i] = (uint8_t)(h >> 8); } }
struct Lay { int64_t R, C, Cp; uint8_t* planes; uint16_t* lut; uint16_t* x; float* y; };
int main() {
    cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int64_t shp[7][2] = {{4096,4096},{4096,4096},{4096,4096},{4096,4096},{11008,4096},{11008,4096},{4096,11008}};
    const int NC = 4;
    std::vector<std::vector<Lay>> cp(NC);
    for (int c = 0; c < NC; ++c) for (int i = 0; i < 7; ++i) {
        Lay L; L.R = shp[i][0]; L.C = shp[i][1]; L.Cp = apb_pad_columns(L.C);
        CK(cudaMalloc(&L.planes, 8 * L.R * L.Cp / 8)); fill<<<512,256>>>(L.planes, 8 * L.R * L.Cp / 8, c * 7 + i);
        CK(cudaMalloc(&L.lut, L.R * 256 * 2)); fill<<<512,256>>>((uint8_t*)L.lut, L.R * 512, 99 + i);
        CK(cudaMalloc(&L.x, L.C * 2)); CK(cudaMemset(L.x, 0, L.C * 2));
        CK(cudaMalloc(&L.y, L.R * 4));
        cp[c].push_back(L);
    }
    const int groups[4][3] = {{0,1,2},{3,-1,-1},{4,5,-1},{6,-1,-1}};
    auto step = [&]() {
        int li = 0;
        for (int k = 3; k <= 8; ++k) for (int gi = 0; gi < 4; ++gi, ++li) {
            std::vector<Lay>& set = cp[li % NC];
            const uint8_t* pl[3]; int nm[3]; int64_t r[3], cc[3], pd[3], ldx[3], ldy[3]; const uint16_t* lt[3]; const uint16_t* xx[3]; void* yy[3];
            int n = 0;
            for (int j = 0; j < 3; ++j) { int id = groups[gi][j]; if (id < 0) continue; Lay& L = set[id];
                pl[n] = L.planes; nm[n] = 8; r[n] = L.R; cc[n] = L.C; pd[n] = L.Cp; lt[n] = L.lut; xx[n] = set[groups[gi][0]].x; ldx[n] = L.C; yy[n] = L.y; ldy[n] = L.R; ++n; }
            int rc = apb_gemv_grouped(n, pl, nm, r, cc, pd, k, lt, xx, 1, ldx, 0, yy, APB_DTYPE_F32, ldy, APB_FLAG_PDL, s);
            if (rc) { fprintf(stderr, "rc %d\n", rc); exit(1); }
        }
    };
    step(); CK(cudaStreamSynchronize(s));
    apb7_timeline_reset();
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal)); step(); CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); CK(cudaGraphLaunch(ge, s)); cudaEventRecord(b, s); CK(cudaStreamSynchronize(s));
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> t(64 * 512 * 8);
    apb7_read_timeline(t.data(), 64 * 512 * 8);
    printf("step %.1f us (event)\n", ms * 1e3);
    const char* nm[] = {"qkv", "o", "gu", "down"};
    unsigned long long t00 = ~0ull, prev_end = 0;
    for (int l = 0; l < 24; ++l) for (int c = 0; c < 512; ++c) { unsigned long long v = t[((size_t)l * 512 + c) * 8]; if (v && v < t00) t00 = v; }
    double sum_span = 0;
    for (int l = 0; l < 24; ++l) {
        std::vector<double> st, en, tb, s0;
        for (int c = 0; c < 512; ++c) {
            const unsigned long long* p = &t[((size_t)l * 512 + c) * 8];
            if (!p[0]) continue;
            st.push_back((p[0] - t00) / 1e3); en.push_back((p[5] - t00) / 1e3);
            tb.push_back((p[1] - p[0]) / 1e3); s0.push_back((p[3] - p[0]) / 1e3);
        }
        if (st.empty()) continue;
        std::sort(st.begin(), st.end()); std::sort(en.begin(), en.end()); std::sort(tb.begin(), tb.end()); std::sort(s0.begin(), s0.end());
        double start = st.front(), end = en.back();
        printf("k%d %-4s ctas %3zu start %7.2f end %7.2f span %6.2f | gap %5.2f | cta start spread %5.2f | table0 %4.2f stage0 %4.2f | end spread (med..max) %5.2f..%5.2f\n",
               3 + l / 4, nm[l % 4], st.size(), start, end, end - start, l ? start - prev_end / 1e3 : 0.0, st.back() - st.front(),
               tb[tb.size() / 2], s0[s0.size() / 2], en[en.size() / 2] - start, end - start);
        prev_end = (unsigned long long)(end * 1e3);
        sum_span += end - start;
    }
    printf("sum of spans %.1f us\n", sum_span);
    for (int l : {8, 9, 10, 11, 20, 22}) {
        printf("launch %d (k%d %s): blockIdx: start / stage0 / end (us from launch first start)\n", l, 3 + l / 4, nm[l % 4]);
        double s0 = 1e30;
        for (int c = 0; c < 512; ++c) { const unsigned long long* p = &t[((size_t)l * 512 + c) * 8]; if (p[0]) s0 = std::min(s0, (p[0] - t00) / 1e3); }
        for (int c = 0; c < 512; c += 12) {
            const unsigned long long* p = &t[((size_t)l * 512 + c) * 8];
            if (!p[0]) continue;
            printf("  %3d %6.2f %6.2f %6.2f\n", c, (p[0] - t00) / 1e3 - s0, (p[3] - t00) / 1e3 - s0, (p[5] - t00) / 1e3 - s0);
        }
    }
}
