// apb_quant.cu -- the offline any-precision quantizer on the GPU (SURVEY.md
// section 8(f) row 4): sensitivity-weighted exact 1-D k-means seed at n_min
// bits by dynamic programming, then one exact weighted 2-means split per
// extra bit up to n_max (reference quantizer.py:370-435 / :515-531,
// clustering.py:89-302).  Bit-exact with the reference: every float64
// expression is evaluated in the reference's order with round-to-nearest and
// no FMA contraction (this file is compiled with -fmad=false), prefix sums are
// sequential like np.cumsum, and the two numpy reductions the reference uses
// are reproduced with numpy's own association (pairwise_sum below).
//
// Layout: one CTA per output channel (row); the per-row working set lives in
// a caller-provided workspace.  The caller supplies the stable argsort of every
// row (torch.sort(stable=True) on device).
//
//   prefix_kernel : thread per row: sorted values / weights, inclusive prefix
//                   sums (w, w*v, w*v*v) with a leading zero, distinct count
//   seed_kernel   : CTA per row: _dp_boundaries (clustering.py:89-197) with
//                   k_eff = min(distinct, 2^n_min) clusters
//   level_kernel  : CTA per row, once per bit-width k = n_min..n_max: interval
//                   means (clustering.py:60-83 + quantizer.py:244-259), fp16
//                   table, weighted SSE against it (quantizer.py:272-278),
//                   level codes, and for k < n_max the 2-means split of every
//                   interval (clustering.py:252-302)
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/anyprec_b200.h"

namespace {

constexpr double kTiny = 4.9406564584124654e-324;  // clustering.py:86, smallest subnormal
constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLevelBits = 8;                   // quantizer.py:28 MAX_BITS
constexpr int kMaxIntervals = 1 << kMaxLevelBits;
constexpr int kLeafMax = 128;                      // numpy PW_BLOCKSIZE
constexpr int kMaxLeaves = 512;                    // parallel SSE leaves: rows up to 32K wide

// Per-row workspace slices (element offsets are computed by Ws).
struct Ws {
    int n, k_seed, n_max;
    size_t row_bytes;
    size_t off_sv, off_sw, off_pw, off_pwv, off_pwv2, off_d0, off_d1, off_args, off_bounds, off_means, off_parents,
        off_distinct;
    __host__ __device__ Ws(int n_, int k_seed_, int n_max_) : n(n_), k_seed(k_seed_), n_max(n_max_) {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t r = o;
            o += (bytes + 15) & ~(size_t)15;
            return r;
        };
        off_sv = take(sizeof(double) * n);
        off_sw = take(sizeof(double) * n);
        off_pw = take(sizeof(double) * (n + 1));
        off_pwv = take(sizeof(double) * (n + 1));
        off_pwv2 = take(sizeof(double) * (n + 1));
        off_d0 = take(sizeof(double) * (n + 1));
        off_d1 = take(sizeof(double) * (n + 1));
        off_args = take(sizeof(int) * (size_t)(k_seed > 2 ? k_seed - 2 : 0) * n);
        off_bounds = take(sizeof(int) * ((1 << n_max) + 1) * 2);
        off_means = take(sizeof(double) * (1 << n_max));
        off_parents = take(sizeof(double) * (1 << n_max));
        off_distinct = take(sizeof(int));
        row_bytes = o;
    }
};

template <typename T>
__device__ __forceinline__ T* slice(void* ws, const Ws& W, int row, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(ws) + (size_t)row * W.row_bytes + off);
}

// ---- numpy's pairwise summation (loops_utils.h.src, PW_BLOCKSIZE 128) ---------
// f(i) yields element i.  n < 8: plain loop from 0; n <= 128: eight strided
// accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the
// remainder; else split at n/2 rounded down to a multiple of 8.
template <typename F>
__device__ double pw_leaf(const F& f, int64_t a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += f(a + i);
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(a + j);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] += f(a + i + j);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += f(a + i);
    return res;
}

template <typename F>
__device__ double pairwise_sum(const F& f, int64_t a, int64_t n) {
    // explicit stack: depth <= log2(n / 64) + 1
    if (n <= kLeafMax) return pw_leaf(f, a, n);
    struct Frame {
        int64_t a, n;
        double left;
        int state;
    } st[40];
    int sp = 0;
    st[0] = {a, n, 0.0, 0};
    double ret = 0.0;
    while (true) {
        Frame& fr = st[sp];
        if (fr.n <= kLeafMax) {
            ret = pw_leaf(f, fr.a, fr.n);
            if (sp == 0) return ret;
            --sp;
            continue;
        }
        int64_t n2 = fr.n / 2;
        n2 -= n2 % 8;
        if (fr.state == 0) {
            fr.state = 1;
            st[++sp] = {fr.a, n2, 0.0, 0};
        } else if (fr.state == 1) {
            fr.left = ret;
            fr.state = 2;
            st[++sp] = {fr.a + n2, fr.n - n2, 0.0, 0};
        } else {
            ret = fr.left + ret;
            if (sp == 0) return ret;
            --sp;
        }
    }
}

// np.add.reduceat over one segment: the first element, then the pairwise sum
// of the rest (the reduce inner loop adds into the copied first element).
template <typename F>
__device__ double reduceat_sum(const F& f, int64_t a, int64_t n) {
    if (n == 1) return f(a);
    return f(a) + pairwise_sum(f, a + 1, n - 1);
}

// Weighted mean of sorted positions [a, a + len) (clustering.py:60-83): the
// reduceat sums of w and w*v; zero total weight -> the plain mean; empty -> NaN.
__device__ double interval_mean(const double* sv, const double* sw, int a, int len) {
    if (len <= 0) return NAN;
    const double sum_w = reduceat_sum([&](int64_t i) { return sw[i]; }, a, len);
    const double sum_wv = reduceat_sum([&](int64_t i) { return sw[i] * sv[i]; }, a, len);
    if (sum_w > 0.0) return sum_wv / sum_w;
    const double sum_v = reduceat_sum([&](int64_t i) { return sv[i]; }, a, len);
    return sum_v / (double)len;
}

// (value, index) argmin with first-index tie break, as np.minimum.reduceat
// followed by the first position equal to the minimum.
__device__ __forceinline__ void argmin_merge(double& v, int& i, double v2, int i2) {
    if (v2 < v || (v2 == v && i2 < i)) {
        v = v2;
        i = i2;
    }
}
__device__ __forceinline__ void warp_argmin(double& v, int& i) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
        argmin_merge(v, i, v2, i2);
    }
}

// ------------------------------------------------------------------------------
__global__ void prefix_kernel(const double* __restrict__ w, const double* __restrict__ s,
                              const int64_t* __restrict__ order, int rows, Ws W, void* ws) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int n = W.n;
    const double* wr = w + (int64_t)r * n;
    const double* sr = s + (int64_t)r * n;
    const int64_t* orr = order + (int64_t)r * n;
    double* sv = slice<double>(ws, W, r, W.off_sv);
    double* sw = slice<double>(ws, W, r, W.off_sw);
    double* pw = slice<double>(ws, W, r, W.off_pw);
    double* pwv = slice<double>(ws, W, r, W.off_pwv);
    double* pwv2 = slice<double>(ws, W, r, W.off_pwv2);
    // clustering.py:31-43: cumsum of w, w*v, w*v*v (evaluated left to right)
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, prev = 0.0;
    int distinct = 1;
    pw[0] = pwv[0] = pwv2[0] = 0.0;
    for (int p = 0; p < n; ++p) {
        const int64_t o = orr[p];
        const double v = wr[o], x = sr[o];
        sv[p] = v;
        sw[p] = x;
        const double xv = x * v;
        a0 += x;
        a1 += xv;
        a2 += xv * v;
        pw[p + 1] = a0;
        pwv[p + 1] = a1;
        pwv2[p + 1] = a2;
        if (p > 0 && v - prev > 0.0) ++distinct;  // clustering.py:200-201
        prev = v;
    }
    *slice<int>(ws, W, r, W.off_distinct) = distinct;
}

// One DP layer candidate: dist over prefix j with m-1 clusters plus the cost of
// the last cluster [j, b), b = the prefix end whose sums are (e0, e1, e2)
// (clustering.py:120-127).
__device__ __forceinline__ double dp_cand(const double* pw, const double* pwv, const double* pwv2,
                                          const double* dist, int j, double e0, double e1, double e2) {
    const double dw = e0 - pw[j];
    const double dwv = e1 - pwv[j];
    const double dwv2 = e2 - pwv2[j];
    double cost = dwv2 - dwv * dwv / fmax(dw, kTiny);
    cost += dist[j];
    return cost;
}

// argmin over j in [jlo, jhi] by the calling warp
__device__ __forceinline__ void warp_scan(const double* pw, const double* pwv, const double* pwv2,
                                          const double* dist, int jlo, int jhi, int b, double& best, int& jstar) {
    const int lane = threadIdx.x & 31;
    const double e0 = pw[b], e1 = pwv[b], e2 = pwv2[b];
    double v = INFINITY;
    int i = INT32_MAX;
    bool any = false;
    for (int j = jlo + lane; j <= jhi; j += 32) {
        const double c = dp_cand(pw, pwv, pwv2, dist, j, e0, e1, e2);
        if (!any) {
            v = c;
            i = j;
            any = true;
        } else {
            argmin_merge(v, i, c, j);
        }
    }
    warp_argmin(v, i);
    best = v;
    jstar = i;
}

__global__ void __launch_bounds__(kThreads) seed_kernel(int rows, Ws W, void* ws) {
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int n = W.n, k = W.k_seed;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* pw = slice<double>(ws, W, r, W.off_pw);
    const double* pwv = slice<double>(ws, W, r, W.off_pwv);
    const double* pwv2 = slice<double>(ws, W, r, W.off_pwv2);
    double* dist = slice<double>(ws, W, r, W.off_d0);
    double* ndist = slice<double>(ws, W, r, W.off_d1);
    int* args = slice<int>(ws, W, r, W.off_args);
    int* bounds = slice<int>(ws, W, r, W.off_bounds);
    const int distinct = *slice<int>(ws, W, r, W.off_distinct);
    const int keff = min(distinct, k);  // quantizer.py:224-237
    __shared__ double s_best[kWarps];
    __shared__ int s_arg[kWarps];

    for (int c = threadIdx.x; c <= k; c += kThreads) bounds[c] = c == 0 ? 0 : n;
    if (keff == 1) return;
    __syncthreads();
    // layer 1: one cluster over every prefix (clustering.py:116-117)
    for (int t = threadIdx.x; t <= n; t += kThreads)
        dist[t] = t == 0 ? INFINITY : pwv2[t] - pwv[t] * pwv[t] / fmax(pw[t], kTiny);
    __syncthreads();
    for (int m = 2; m < keff; ++m) {
        int* arg = args + (size_t)(m - 2) * n;
        for (int t = threadIdx.x; t <= n; t += kThreads) ndist[t] = INFINITY;
        __syncthreads();
        // divide and conquer over i = mid in [m-1, n-1], level by level: a node's
        // j-range is [arg of the ancestor ending just left of it (or m-1), arg of
        // the ancestor just right of it (or n-1)], clipped to j <= mid
        for (int level = 0;; ++level) {
            const int64_t n_nodes = (int64_t)1 << level;
            bool any = false;
            for (int64_t q0 = 0; q0 < n_nodes; q0 += kWarps) {
                const int64_t q = q0 + warp;
                int lo = m - 1, hi = n - 1;
                bool live = q < n_nodes;
                for (int b = level - 1; b >= 0 && live; --b) {
                    const int mid = (lo + hi) >> 1;
                    if ((q >> b) & 1) lo = mid + 1;
                    else hi = mid - 1;
                    live = lo <= hi;
                }
                if (!live) continue;
                any = true;
                const int mid = (lo + hi) >> 1;
                const int jlo = lo > m - 1 ? arg[lo - 1] : m - 1;
                const int jhi = min(hi < n - 1 ? arg[hi + 1] : n - 1, mid);
                double best;
                int jstar;
                warp_scan(pw, pwv, pwv2, dist, jlo, jhi, mid + 1, best, jstar);
                if (lane == 0) {
                    ndist[mid + 1] = best;
                    arg[mid] = jstar;
                }
            }
            if (!__syncthreads_or(any)) break;  // no live node at this depth: layer done
        }
        double* t = dist;
        dist = ndist;
        ndist = t;
    }
    // final layer: one scan over j in [keff-1, n-1] ending at n (clustering.py:173-189)
    {
        const double e0 = pw[n], e1 = pwv[n], e2 = pwv2[n];
        double v = INFINITY;
        int i = INT32_MAX;
        bool any = false;
        for (int j = keff - 1 + (int)threadIdx.x; j <= n - 1; j += kThreads) {
            const double c = dp_cand(pw, pwv, pwv2, dist, j, e0, e1, e2);
            if (!any) {
                v = c;
                i = j;
                any = true;
            } else {
                argmin_merge(v, i, c, j);
            }
        }
        warp_argmin(v, i);
        if (lane == 0) {
            s_best[warp] = v;
            s_arg[warp] = i;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double bv = s_best[0];
            int bi = s_arg[0];
            for (int w2 = 1; w2 < kWarps; ++w2) argmin_merge(bv, bi, s_best[w2], s_arg[w2]);
            // traceback (clustering.py:191-196)
            bounds[keff - 1] = bi;
            int idx = bi - 1;
            for (int m = keff - 1; m >= 2; --m) {
                const int jm = args[(size_t)(m - 2) * n + idx];
                bounds[m - 1] = jm;
                idx = jm - 1;
            }
        }
    }
}

// k-bit level of one row: bounds (2^k + 1 entries) in slot `cur` of the row's
// bounds area; writes the fp16 table, the SSE, optional level codes and, when
// split != 0, the 2^(k+1) + 1 split bounds into the other slot.
__global__ void __launch_bounds__(kThreads) level_kernel(int rows, Ws W, void* ws, int kbits, int cur, int seed,
                                                         int split, int only_split, uint16_t* __restrict__ table,
                                                         double* __restrict__ sse, uint8_t* __restrict__ codes_a,
                                                         uint8_t* __restrict__ codes_b,
                                                         const int64_t* __restrict__ order) {
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int n = W.n, m = 1 << kbits;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* sv = slice<double>(ws, W, r, W.off_sv);
    const double* sw = slice<double>(ws, W, r, W.off_sw);
    const double* pw = slice<double>(ws, W, r, W.off_pw);
    const double* pwv = slice<double>(ws, W, r, W.off_pwv);
    const double* pwv2 = slice<double>(ws, W, r, W.off_pwv2);
    int* bounds_area = slice<int>(ws, W, r, W.off_bounds);
    const int bstride = (1 << W.n_max) + 1;
    const int* bounds = bounds_area + cur * bstride;
    int* nbounds = bounds_area + (cur ^ 1) * bstride;
    double* means = slice<double>(ws, W, r, W.off_means);
    double* parents = slice<double>(ws, W, r, W.off_parents);

    __shared__ int sb[kMaxIntervals + 1];
    __shared__ double t64[kMaxIntervals];
    __shared__ double leaf[kMaxLeaves];
    for (int c = threadIdx.x; c <= m; c += kThreads) sb[c] = bounds[c];
    __syncthreads();
    if (!only_split) {  // (continue_upscale's first step only splits the stored level)
        // interval means (clustering.py:60-83): reduceat sums of w, w*v, v
        for (int c = threadIdx.x; c < m; c += kThreads) means[c] = interval_mean(sv, sw, sb[c], sb[c + 1] - sb[c]);
        __syncthreads();
        // empty intervals (quantizer.py:244-259): seed -> copy the previous column;
        // otherwise -> the parent's float64 centroid
        if (seed) {
            if (threadIdx.x == 0)
                for (int c = 1; c < m; ++c)
                    if (isnan(means[c])) means[c] = means[c - 1];
        } else {
            for (int c = threadIdx.x; c < m; c += kThreads)
                if (isnan(means[c])) means[c] = parents[c >> 1];
        }
        __syncthreads();
        for (int c = threadIdx.x; c < m; c += kThreads) {
            const __half h = __double2half(means[c]);
            if (table) table[(int64_t)r * m + c] = __half_as_ushort(h);
            t64[c] = (double)__half2float(h);
            parents[c] = means[c];  // the next level's parents
        }
        __syncthreads();
        // weighted SSE against the fp16 table (quantizer.py:272-278): np.sum over the
        // row of (w * diff) * diff -- pairwise; leaves of <= 128 summed in parallel
        {
            auto code_of = [&](int64_t p) {
                int lo = 0, hi = m - 1;  // last c with sb[c] <= p and sb[c+1] > p
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sb[mid] <= p) lo = mid;
                    else hi = mid - 1;
                }
                return lo;
            };
            auto term = [&](int64_t p) {
                const double d = sv[p] - t64[code_of(p)];
                return sw[p] * d * d;
            };
            // enumerate the leaves of numpy's split tree (left to right)
            __shared__ int64_t leaf_a[kMaxLeaves], leaf_n[kMaxLeaves];
            __shared__ int n_leaves;
            if (threadIdx.x == 0) {
                int cnt = 0;
                int64_t sa[40], sn[40];
                int sp = 0;
                sa[0] = 0;
                sn[0] = n;
                while (sp >= 0) {
                    const int64_t a = sa[sp], len = sn[sp];
                    --sp;
                    if (len <= kLeafMax || cnt >= kMaxLeaves) {
                        leaf_a[cnt] = a;
                        leaf_n[cnt] = len;
                        ++cnt;
                    } else {
                        int64_t n2 = len / 2;
                        n2 -= n2 % 8;
                        // push right first so the left is processed first
                        ++sp;
                        sa[sp] = a + n2;
                        sn[sp] = len - n2;
                        ++sp;
                        sa[sp] = a;
                        sn[sp] = n2;
                    }
                }
                n_leaves = cnt;
            }
            __syncthreads();
            const bool small = n <= kMaxLeaves * kLeafMax / 2;  // every leaf of the split tree is >= 64
            if (small) {
                for (int l = threadIdx.x; l < n_leaves; l += kThreads) leaf[l] = pw_leaf(term, leaf_a[l], leaf_n[l]);
                __syncthreads();
                if (threadIdx.x == 0) {
                    // recombine in the split tree's order
                    struct F2 {
                        int64_t n;
                        double left;
                        int state;
                    } st[40];
                    int sp = 0, li = 0;
                    st[0] = {(int64_t)n, 0.0, 0};
                    double ret = 0.0;
                    while (true) {
                        F2& fr = st[sp];
                        if (fr.n <= kLeafMax) {
                            ret = leaf[li++];
                            if (sp == 0) break;
                            --sp;
                            continue;
                        }
                        int64_t n2 = fr.n / 2;
                        n2 -= n2 % 8;
                        if (fr.state == 0) {
                            fr.state = 1;
                            st[++sp] = {n2, 0.0, 0};
                        } else if (fr.state == 1) {
                            fr.left = ret;
                            fr.state = 2;
                            st[++sp] = {fr.n - n2, 0.0, 0};
                        } else {
                            ret = fr.left + ret;
                            if (sp == 0) break;
                            --sp;
                        }
                    }
                    if (sse) sse[r] = ret;
                }
            } else if (threadIdx.x == 0 && sse) {
                sse[r] = pairwise_sum(term, 0, n);
            }
        }
        // codes of this level (scattered back through the sort order)
        if (codes_a || codes_b) {
            const int64_t* orr = order + (int64_t)r * n;
            for (int c = warp; c < m; c += kWarps)
                for (int p = sb[c] + lane; p < sb[c + 1]; p += 32) {
                    const int64_t o = (int64_t)r * n + orr[p];
                    if (codes_a) codes_a[o] = (uint8_t)c;
                    if (codes_b) codes_b[o] = (uint8_t)c;
                }
        }
    }
    if (!split) return;
    // 2-means split of every interval (clustering.py:252-302): warp per interval
    for (int c = warp; c < m; c += kWarps) {
        const int b0 = sb[c], b1 = sb[c + 1], len = b1 - b0;
        int s = b1;
        const bool splittable = len >= 2 && sv[max(b1 - 1, 0)] > sv[min(b0, n - 1)];
        if (splittable) {
            const double lo_w = pw[b0], lo_wv = pwv[b0], lo_wv2 = pwv2[b0];
            const double hi_w = pw[b1], hi_wv = pwv[b1], hi_wv2 = pwv2[b1];
            double v = INFINITY;
            int i = INT32_MAX;
            bool any = false;
            for (int p = b0 + lane; p < b1; p += 32) {
                double cost;
                if (p == b0) {
                    cost = INFINITY;  // a split at the start leaves the left child empty
                } else {
                    const double dlw = pw[p] - lo_w;
                    const double dlv = pwv[p] - lo_wv;
                    cost = (pwv2[p] - lo_wv2) - dlv * dlv / fmax(dlw, kTiny);
                    const double drw = hi_w - pw[p];
                    const double drv = hi_wv - pwv[p];
                    cost += (hi_wv2 - pwv2[p]) - drv * drv / fmax(drw, kTiny);
                }
                if (!any) {
                    v = cost;
                    i = p;
                    any = true;
                } else {
                    argmin_merge(v, i, cost, p);
                }
            }
            warp_argmin(v, i);
            s = i;
        }
        if (lane == 0) {
            nbounds[2 * c] = b0;
            nbounds[2 * c + 1] = s;
            if (c == m - 1) nbounds[2 * m] = sb[m];  // out[:, 0::2] = bounds
        }
    }
}

// continue_upscale (quantizer.py:469-484): the stored k0-bit codes in sorted
// order must be non-decreasing (value-contiguous clusters); their counts give
// the k0-level interval bounds (slot 0), and the fp16 table of k0 (as float64)
// is the parent of the first split (quantizer.py:484).
__global__ void __launch_bounds__(kThreads) bounds_from_codes_kernel(int rows, Ws W, void* ws,
                                                                     const uint8_t* __restrict__ codes, int k0,
                                                                     const int64_t* __restrict__ order,
                                                                     const uint16_t* __restrict__ table,
                                                                     int* __restrict__ bad,
                                                                     const double* __restrict__ parents64) {
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int n = W.n, m = 1 << k0;
    __shared__ int cnt[kMaxIntervals];
    for (int c = threadIdx.x; c < m; c += kThreads) cnt[c] = 0;
    __syncthreads();
    const uint8_t* cr = codes + (int64_t)r * n;
    const int64_t* orr = order + (int64_t)r * n;
    bool ok = true;
    for (int p = threadIdx.x; p < n; p += kThreads) {
        const int c = cr[orr[p]];
        if (c >= m || (p > 0 && c < cr[orr[p - 1]])) ok = false;
        else atomicAdd(&cnt[c], 1);
    }
    if (!ok) atomicOr(bad, 1);
    __syncthreads();
    int* bounds = slice<int>(ws, W, r, W.off_bounds);  // slot 0
    double* parents = slice<double>(ws, W, r, W.off_parents);
    if (threadIdx.x == 0) {
        int acc = 0;
        bounds[0] = 0;
        for (int c = 0; c < m; ++c) {
            acc += cnt[c];
            bounds[c + 1] = acc;
        }
    }
    for (int c = threadIdx.x; c < m; c += kThreads)
        parents[c] = parents64 ? parents64[(int64_t)r * m + c]
                               : (double)__half2float(__ushort_as_half(table[(int64_t)r * m + c]));
}

// continue_upscale's error record of the EXISTING levels (quantizer.py:499-503):
// np.sum(s * (w - table_k[codes >> shift]) ** 2, axis=1) over the row in its
// original column order -- numpy's pairwise summation, one thread per row.
__global__ void sse_levels_kernel(const double* __restrict__ w, const double* __restrict__ s,
                                  const uint8_t* __restrict__ codes, int shift, const uint16_t* __restrict__ table,
                                  int k, int rows, int n, double* __restrict__ sse) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int64_t base = (int64_t)r * n;
    const uint16_t* tr = table + ((int64_t)r << k);
    auto term = [&](int64_t i) {
        const double deq = (double)__half2float(__ushort_as_half(tr[codes[base + i] >> shift]));
        const double d = w[base + i] - deq;
        return s[base + i] * (d * d);
    };
    sse[r] = pairwise_sum(term, 0, n);
}

// cluster_rows + the seed centroids (clustering.py:204-227, quantizer.py:224-259,
// kmeans_1d_weighted quantizer.py:122-157) for any cluster count k: the DP
// bounds of every row, float64 interval means with empty trailing intervals
// copying the previous column, and the interval index of every element in the
// row's original order.  One CTA per row.
__global__ void __launch_bounds__(kThreads) cluster_out_kernel(int rows, Ws W, void* ws, int k,
                                                               const int64_t* __restrict__ order,
                                                               int* __restrict__ bounds_out,
                                                               double* __restrict__ means_out,
                                                               int* __restrict__ codes_out) {
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int n = W.n;
    const double* sv = slice<double>(ws, W, r, W.off_sv);
    const double* sw = slice<double>(ws, W, r, W.off_sw);
    const int* b = slice<int>(ws, W, r, W.off_bounds);
    double* mr = means_out + (int64_t)r * k;
    for (int c = threadIdx.x; c <= k; c += kThreads) bounds_out[(int64_t)r * (k + 1) + c] = b[c];
    for (int c = threadIdx.x; c < k; c += kThreads) mr[c] = interval_mean(sv, sw, b[c], b[c + 1] - b[c]);
    __syncthreads();
    if (threadIdx.x == 0)
        for (int c = 1; c < k; ++c)
            if (isnan(mr[c])) mr[c] = mr[c - 1];
    if (codes_out) {
        const int64_t* orr = order + (int64_t)r * n;
        for (int c = threadIdx.x >> 5; c < k; c += kThreads / 32)
            for (int p = b[c] + (threadIdx.x & 31); p < b[c + 1]; p += 32) codes_out[(int64_t)r * n + orr[p]] = c;
    }
}

// _upscale_general (quantizer.py:344-367): codes that are not value-contiguous.
// Every cluster b is split by its own exact weighted 2-means
// (kmeans_1d_weighted of its members, weights -> 1 when they sum to 0): the
// row arrives sorted by (code, value) (ties by position), each warp takes whole
// clusters, builds their fresh prefix sums from 0 (as the per-cluster k-means
// does), scans the k = 2 DP's last layer and writes codes 2b / 2b+1 and the two
// centroids; fewer than two distinct members -> all 2b, both centroids = their
// mean; an empty cluster -> both = the parent centroid.
__global__ void __launch_bounds__(kThreads) upscale_general_kernel(
    const double* __restrict__ w, const double* __restrict__ s, const int64_t* __restrict__ gorder,
    const uint8_t* __restrict__ codes_in, const double* __restrict__ parents, int rows, int n, int k0,
    uint8_t* __restrict__ codes_out, double* __restrict__ means_out, double* __restrict__ scratch) {
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int m = 1 << k0, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t* go = gorder + (int64_t)r * n;
    const double* wr = w + (int64_t)r * n;
    const double* sr = s + (int64_t)r * n;
    const uint8_t* cr = codes_in + (int64_t)r * n;
    // scratch per row: sv, sw [n] and pw / pwv / pwv2 [n + m + 1] (cluster b's prefix at start_b + b)
    const int64_t stride = 2 * (int64_t)n + 3 * ((int64_t)n + m + 1);
    double* sv = scratch + (int64_t)r * stride;
    double* sw = sv + n;
    double* pw = sw + n;
    double* pwv = pw + (n + m + 1);
    double* pwv2 = pwv + (n + m + 1);
    __shared__ int start[kMaxIntervals + 1];
    if (threadIdx.x == 0) {  // clusters are contiguous in (code, value) order
        int c = 0;
        for (int p = 0; p < n; ++p)
            while (c <= (int)cr[go[p]]) start[c++] = p;
        while (c <= m) start[c++] = n;
    }
    __syncthreads();
    for (int b = warp; b < m; b += kThreads / 32) {
        const int a = start[b], len = start[b + 1] - a;
        double* outm = means_out + (int64_t)r * 2 * m;
        if (len == 0) {
            if (lane == 0) outm[2 * b] = outm[2 * b + 1] = parents[(int64_t)r * m + b];
            continue;
        }
        // members in value order, weights (or ones when they sum to 0)
        bool any_w = false;
        for (int i = lane; i < len; i += 32) any_w |= sr[go[a + i]] > 0.0;
        any_w = __any_sync(0xffffffffu, any_w);
        for (int i = lane; i < len; i += 32) {
            const int64_t o = go[a + i];
            sv[a + i] = wr[o];
            sw[a + i] = any_w ? sr[o] : 1.0;
        }
        __syncwarp();
        const int pb = a + b;  // this cluster's prefix slice
        int distinct = 1;
        if (lane == 0) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0;
            pw[pb] = pwv[pb] = pwv2[pb] = 0.0;
            for (int i = 0; i < len; ++i) {
                const double v = sv[a + i], x = sw[a + i], xv = x * v;
                a0 += x;
                a1 += xv;
                a2 += xv * v;
                pw[pb + i + 1] = a0;
                pwv[pb + i + 1] = a1;
                pwv2[pb + i + 1] = a2;
                if (i > 0 && v - sv[a + i - 1] > 0.0) ++distinct;
            }
        }
        distinct = __shfl_sync(0xffffffffu, distinct, 0);
        __syncwarp();
        int split = len;  // padded: every member in the low child
        if (distinct >= 2) {
            const double e0 = pw[pb + len], e1 = pwv[pb + len], e2 = pwv2[pb + len];
            double v = INFINITY;
            int i = INT32_MAX;
            bool first = true;
            for (int j = 1 + lane; j <= len - 1; j += 32) {
                const double d1 = pwv2[pb + j] - pwv[pb + j] * pwv[pb + j] / fmax(pw[pb + j], kTiny);
                const double dw = e0 - pw[pb + j], dwv = e1 - pwv[pb + j], dwv2 = e2 - pwv2[pb + j];
                double c = dwv2 - dwv * dwv / fmax(dw, kTiny);
                c += d1;
                if (first) {
                    v = c;
                    i = j;
                    first = false;
                } else {
                    argmin_merge(v, i, c, j);
                }
            }
            warp_argmin(v, i);
            split = i;
        }
        if (lane == 0) {
            const double lo = interval_mean(sv + a, sw + a, 0, split);
            const double hi = split < len ? interval_mean(sv + a, sw + a, split, len - split) : lo;
            outm[2 * b] = lo;
            outm[2 * b + 1] = hi;
        }
        for (int i2 = lane; i2 < len; i2 += 32)
            codes_out[(int64_t)r * n + go[a + i2]] = (uint8_t)(2 * b + (i2 >= split ? 1 : 0));
    }
}

int finish() { return cudaGetLastError() == cudaSuccess ? APB_OK : APB_ERR_CUDA; }

}  // namespace

extern "C" int64_t apb_quant_workspace(int rows, int n, int n_min, int n_max) {
    if (rows <= 0 || n <= 0 || n_min < 2 || n_min > n_max || n_max > kMaxLevelBits) return -1;
    return (int64_t)rows * (int64_t)Ws(n, 1 << n_min, n_max).row_bytes;
}

extern "C" int apb_quant_build(const double* weights, const double* sens, const int64_t* order, int rows, int n,
                               int n_min, int n_max, uint8_t* codes, uint16_t* tables, double* sse,
                               uint8_t* level_codes, void* workspace, int64_t workspace_bytes, void* stream) {
    if (!weights || !sens || !order || !codes || !tables || !sse || !workspace) return APB_ERR_PARAM;
    const int64_t need = apb_quant_workspace(rows, n, n_min, n_max);
    if (need < 0) return rows <= 0 || n <= 0 ? APB_ERR_SHAPE : APB_ERR_PARAM;
    if (workspace_bytes < need || ((uintptr_t)workspace & 15)) return APB_ERR_PARAM;
    cudaStream_t st = (cudaStream_t)stream;
    const Ws W(n, 1 << n_min, n_max);
    prefix_kernel<<<(rows + 127) / 128, 128, 0, st>>>(weights, sens, order, rows, W, workspace);
    seed_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace);
    int cur = 0;
    int64_t toff = 0;
    for (int k = n_min; k <= n_max; ++k) {
        const int last = k == n_max;
        uint8_t* lc = level_codes ? level_codes + (int64_t)(k - n_min) * rows * n : nullptr;
        level_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, k, cur, k == n_min, !last, 0, tables + toff,
                                                 sse + (int64_t)(k - n_min) * rows, lc, last ? codes : nullptr,
                                                 order);
        toff += (int64_t)rows << k;
        cur ^= 1;
    }
    return finish();
}

extern "C" int apb_quant_continue(const double* weights, const double* sens, const int64_t* order,
                                  const uint8_t* codes_in, const uint16_t* table_k0, int rows, int n, int k0,
                                  int new_n_max, uint8_t* codes, uint16_t* tables, double* sse, int* bad,
                                  void* workspace, int64_t workspace_bytes, void* stream) {
    if (!weights || !sens || !order || !codes_in || !table_k0 || !codes || !tables || !sse || !bad || !workspace)
        return APB_ERR_PARAM;
    if (rows <= 0 || n <= 0) return APB_ERR_SHAPE;
    if (k0 < 2 || new_n_max <= k0 || new_n_max > kMaxLevelBits) return APB_ERR_PARAM;
    const int64_t need = apb_quant_workspace(rows, n, 2, new_n_max);
    if (workspace_bytes < need || ((uintptr_t)workspace & 15)) return APB_ERR_PARAM;
    cudaStream_t st = (cudaStream_t)stream;
    const Ws W(n, 1 << 2, new_n_max);  // no DP here
    prefix_kernel<<<(rows + 127) / 128, 128, 0, st>>>(weights, sens, order, rows, W, workspace);
    bounds_from_codes_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, codes_in, k0, order, table_k0, bad,
                                                         nullptr);
    level_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, k0, 0, 0, 1, 1, nullptr, nullptr, nullptr, nullptr,
                                             order);
    int cur = 1;
    int64_t toff = 0;
    for (int k = k0 + 1; k <= new_n_max; ++k) {
        const int last = k == new_n_max;
        level_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, k, cur, 0, !last, 0, tables + toff,
                                                 sse + (int64_t)(k - k0 - 1) * rows, nullptr, last ? codes : nullptr,
                                                 order);
        toff += (int64_t)rows << k;
        cur ^= 1;
    }
    return finish();
}

extern "C" int apb_quant_sse_levels(const double* weights, const double* sens, const uint8_t* codes, int shift,
                                    const uint16_t* table_k, int k, int rows, int n, double* sse, void* stream) {
    if (!weights || !sens || !codes || !table_k || !sse) return APB_ERR_PARAM;
    if (rows <= 0 || n <= 0) return APB_ERR_SHAPE;
    if (k < 1 || k > kMaxLevelBits || shift < 0 || shift > 7) return APB_ERR_PARAM;
    sse_levels_kernel<<<(rows + 127) / 128, 128, 0, (cudaStream_t)stream>>>(weights, sens, codes, shift, table_k, k,
                                                                            rows, n, sse);
    return finish();
}

// Workspace for apb_quant_cluster: the DP keeps k - 2 argmin rows per channel.
extern "C" int64_t apb_quant_cluster_workspace(int rows, int n, int k) {
    if (rows <= 0 || n <= 0 || k < 1 || k > 4096) return -1;
    int nb = 1;
    while ((1 << nb) < k) ++nb;  // bounds area of 2^nb + 1 entries
    return (int64_t)rows * (int64_t)Ws(n, k, nb).row_bytes;
}

extern "C" int apb_quant_cluster(const double* weights, const double* sens, const int64_t* order, int rows, int n,
                                 int k, int* bounds, double* means, int* codes, void* workspace,
                                 int64_t workspace_bytes, void* stream) {
    if (!weights || !sens || !order || !bounds || !means || !workspace) return APB_ERR_PARAM;
    const int64_t need = apb_quant_cluster_workspace(rows, n, k);
    if (need < 0) return rows <= 0 || n <= 0 ? APB_ERR_SHAPE : APB_ERR_PARAM;
    if (workspace_bytes < need || ((uintptr_t)workspace & 15)) return APB_ERR_PARAM;
    int nb = 1;
    while ((1 << nb) < k) ++nb;
    cudaStream_t st = (cudaStream_t)stream;
    const Ws W(n, k, nb);
    prefix_kernel<<<(rows + 127) / 128, 128, 0, st>>>(weights, sens, order, rows, W, workspace);
    seed_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace);
    cluster_out_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, k, order, bounds, means, codes);
    return finish();
}

// upscale (quantizer.py:310-341), value-contiguous codes: the k0-level bounds
// from the codes, the channel's float64 centroids as parents, one split, the
// new level's float64 means (means [rows][2^(k0+1)]) and codes.
extern "C" int apb_quant_upscale(const double* weights, const double* sens, const int64_t* order,
                                 const uint8_t* codes_in, const double* parents, int rows, int n, int k0,
                                 uint8_t* codes, double* means, int* bad, void* workspace, int64_t workspace_bytes,
                                 void* stream) {
    if (!weights || !sens || !order || !codes_in || !parents || !codes || !means || !bad || !workspace)
        return APB_ERR_PARAM;
    if (rows <= 0 || n <= 0) return APB_ERR_SHAPE;
    if (k0 < 1 || k0 >= kMaxLevelBits) return APB_ERR_PARAM;
    const int64_t need = apb_quant_workspace(rows, n, 2, k0 + 1);
    if (workspace_bytes < need || ((uintptr_t)workspace & 15)) return APB_ERR_PARAM;
    cudaStream_t st = (cudaStream_t)stream;
    const Ws W(n, 1 << 2, k0 + 1);
    prefix_kernel<<<(rows + 127) / 128, 128, 0, st>>>(weights, sens, order, rows, W, workspace);
    bounds_from_codes_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, codes_in, k0, order, nullptr, bad, parents);
    level_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, k0, 0, 0, 1, 1, nullptr, nullptr, nullptr, nullptr,
                                             order);
    level_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, k0 + 1, 1, 0, 0, 0, nullptr, nullptr, nullptr, codes,
                                             order);
    const size_t mb = sizeof(double) << (k0 + 1);
    if (cudaMemcpy2DAsync(means, mb, static_cast<char*>(workspace) + W.off_parents, W.row_bytes, mb, rows,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return APB_ERR_CUDA;
    return finish();
}

// _upscale_general (quantizer.py:344-367): gorder = each row's stable sort by
// (code, value); scratch >= rows * (2n + 3(n + 2^k0 + 1)) doubles.
extern "C" int apb_quant_upscale_general(const double* weights, const double* sens, const int64_t* gorder,
                                         const uint8_t* codes_in, const double* parents, int rows, int n, int k0,
                                         uint8_t* codes, double* means, double* scratch, void* stream) {
    if (!weights || !sens || !gorder || !codes_in || !parents || !codes || !means || !scratch) return APB_ERR_PARAM;
    if (rows <= 0 || n <= 0) return APB_ERR_SHAPE;
    if (k0 < 1 || k0 >= kMaxLevelBits) return APB_ERR_PARAM;
    upscale_general_kernel<<<rows, kThreads, 0, (cudaStream_t)stream>>>(weights, sens, gorder, codes_in, parents, rows,
                                                                        n, k0, codes, means, scratch);
    return finish();
}

// split_boundaries (clustering.py:252-302) on caller bounds: rows of already
// sorted (sv, sw) with identity order, their bounds [rows][m+1] (m a power of
// two <= 256), out [rows][2m+1].
__global__ void load_bounds_kernel(int rows, Ws W, void* ws, int m, const int* __restrict__ bounds) {
    const int r = blockIdx.x;
    if (r >= rows) return;
    int* b = slice<int>(ws, W, r, W.off_bounds);
    for (int c = threadIdx.x; c <= m; c += blockDim.x) b[c] = bounds[(int64_t)r * (m + 1) + c];
}
__global__ void store_bounds_kernel(int rows, Ws W, void* ws, int m, int* __restrict__ out) {
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int* b = slice<int>(ws, W, r, W.off_bounds) + ((1 << W.n_max) + 1);  // slot 1
    for (int c = threadIdx.x; c <= 2 * m; c += blockDim.x) out[(int64_t)r * (2 * m + 1) + c] = b[c];
}

extern "C" int apb_quant_split(const double* sv, const double* sw, const int64_t* identity, int rows, int n,
                               int log2m, const int* bounds, int* out, void* workspace, int64_t workspace_bytes,
                               void* stream) {
    if (!sv || !sw || !identity || !bounds || !out || !workspace) return APB_ERR_PARAM;
    if (rows <= 0 || n <= 0) return APB_ERR_SHAPE;
    if (log2m < 0 || log2m >= kMaxLevelBits) return APB_ERR_PARAM;
    const int64_t need = apb_quant_workspace(rows, n, 2, log2m + 1);
    if (workspace_bytes < need || ((uintptr_t)workspace & 15)) return APB_ERR_PARAM;
    cudaStream_t st = (cudaStream_t)stream;
    const Ws W(n, 1 << 2, log2m + 1);
    const int m = 1 << log2m;
    prefix_kernel<<<(rows + 127) / 128, 128, 0, st>>>(sv, sw, identity, rows, W, workspace);
    load_bounds_kernel<<<rows, 128, 0, st>>>(rows, W, workspace, m, bounds);
    level_kernel<<<rows, kThreads, 0, st>>>(rows, W, workspace, log2m, 0, 0, 1, 1, nullptr, nullptr, nullptr,
                                             nullptr, identity);
    store_bounds_kernel<<<rows, 128, 0, st>>>(rows, W, workspace, m, out);
    return finish();
}
