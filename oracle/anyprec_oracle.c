/*
 * anyprec_oracle.c -- CPU restatement of the reference bitplane hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle and the CPU
 * baseline; it is never linked into, called by or shipped with the product
 * path (paper_2402_10517_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.
 *
 * It restates, step by step, the word-parallel algorithm of the reference
 * package anyprec 0.1.0 (/root/reference/pkg/src/anyprec):
 *   - bitplane.py:72-73    pad_columns
 *   - bitplane.py:76-100   pack_bitplanes   (MSB-first planes, little bit order)
 *   - bitplane.py:103-118  unpack_codes     (prefix codes from planes[:k])
 *   - bitplane.py:121-136  permute / inverse permute (out[4t+j] = in[32j+t])
 *   - engine.py:48-72      bit_transpose    (masked delta swaps, d = 1,2,4)
 *   - engine.py:75-92      transpose_any_width (LSB plane first, B = 2/4/8)
 *   - engine.py:198-209    _extract_codes   (shift + mask per field)
 *   - engine.py:212-246    _dequant_values  (incl. merged 3-bit pair table)
 *   - engine.py:187-195    _weight_order    (bitpos j of lane t -> weight)
 *   - engine.py:284-309    gemv  (fp32 per-tile dot, then fp32 sum over tiles)
 *   - engine.py:312-341    gemm  quantized path (M <= dense_threshold)
 *   - engine.py:357-362    dequantize
 * Parity of this restatement is pinned against vectors produced by the
 * reference itself (tests/golden/make_golden.py -> the npz fixtures in tests/golden).
 *
 * Row-range threading ("row-range work partitioning is
 * permitted") is bit-identical to the serial result because every row is
 * computed independently in a fixed order.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TILE_WEIGHTS 1024
#define TILE_BYTES 128
#define LANES 32

enum { ORA_OK = 0, ORA_SHAPE = 1, ORA_PARAM = 2, ORA_LAYOUT = 3, ORA_CODE_RANGE = 4 };

/* bitplane.py:72-73 */
long long ora_pad_columns(long long cols) { return ((cols + TILE_WEIGHTS - 1) / TILE_WEIGHTS) * TILE_WEIGHTS; }

/* IEEE binary16 -> binary32, exact (numpy float16.astype(float32)). */
static float half_to_float(uint16_t h) {
    uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    uint32_t exp = (h >> 10) & 0x1Fu;
    uint32_t man = h & 0x3FFu;
    uint32_t bits;
    if (exp == 0) {
        if (man == 0) {
            bits = sign;
        } else { /* subnormal: normalise */
            int e = -1;
            do { e++; man <<= 1; } while ((man & 0x400u) == 0);
            man &= 0x3FFu;
            bits = sign | ((uint32_t)(127 - 15 - e) << 23) | (man << 13);
        }
    } else if (exp == 31) {
        bits = sign | 0x7F800000u | (man << 13);
    } else {
        bits = sign | ((exp + 127 - 15) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

void ora_half_to_float(const uint16_t* in, float* out, long long n) {
    for (long long i = 0; i < n; i++) out[i] = half_to_float(in[i]);
}

/* bitplane.py:76-100: codes (rows, cols) -> planes (n_max, rows, padded/8),
 * LINEAR layout.  Plane p holds code bit n_max-1-p; byte b bit i = weight 8b+i
 * (np.packbits(..., bitorder="little")).  Padded tail packs as zero. */
int ora_pack_bitplanes(const uint8_t* codes, long long rows, long long cols, long long ld,
                       int n_max, uint8_t* planes) {
    if (rows <= 0 || cols <= 0) return ORA_SHAPE;
    if (n_max < 1 || n_max > 8) return ORA_PARAM;
    for (long long r = 0; r < rows; r++) {
        uint8_t acc = 0;
        for (long long c = 0; c < cols; c++) acc |= codes[r * ld + c];
        if (acc >> n_max) return ORA_CODE_RANGE; /* bitplane.py:90-91 */
    }
    long long padded = ora_pad_columns(cols);
    long long rb = padded / 8;
    memset(planes, 0, (size_t)(n_max * rows * rb));
    for (long long r = 0; r < rows; r++)
        for (long long b = 0; b < (cols + 7) / 8; b++) {
            /* byte b of every plane = bits of weights 8b..8b+7 (packbits little) */
            uint8_t out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int i = 0; i < 8 && 8 * b + i < cols; i++) {
                uint8_t code = codes[r * ld + 8 * b + i];
                for (int p = 0; p < n_max; p++) /* plane p = code bit n_max-1-p (MSB first) */
                    out[p] |= (uint8_t)(((code >> (n_max - 1 - p)) & 1u) << i);
            }
            for (int p = 0; p < n_max; p++) planes[((long long)p * rows + r) * rb + b] = out[p];
        }
    return ORA_OK;
}

/* bitplane.py:31-36: out[4t + j] = in[32j + t] */
static int perm_src(int pos) { return 32 * (pos & 3) + (pos >> 2); }

/* bitplane.py:121-136: per-tile byte permutation (inverse when inverse != 0). */
void ora_permute(const uint8_t* in, uint8_t* out, long long n_planes, long long rows,
                 long long padded, int inverse) {
    long long rb = padded / 8, tiles = padded / TILE_WEIGHTS;
    for (long long pr = 0; pr < n_planes * rows; pr++)
        for (long long t = 0; t < tiles; t++) {
            const uint8_t* src = in + pr * rb + t * TILE_BYTES;
            uint8_t* dst = out + pr * rb + t * TILE_BYTES;
            for (int pos = 0; pos < TILE_BYTES; pos++) {
                if (!inverse) dst[pos] = src[perm_src(pos)];
                else dst[perm_src(pos)] = src[pos];
            }
        }
}

/* bitplane.py:103-118: k-bit prefix codes from planes[:k] only. */
int ora_unpack_codes(const uint8_t* planes, long long rows, long long cols, long long padded,
                     int n_max, int permuted, int k, uint8_t* codes, long long ld) {
    if (k < 1 || k > n_max) return ORA_PARAM;
    long long rb = padded / 8;
    for (long long r = 0; r < rows; r++)
        for (long long c = 0; c < cols; c++) {
            long long byte = c >> 3;
            if (permuted) { /* inverse permutation of the byte position */
                long long t = byte / TILE_BYTES, b = byte % TILE_BYTES;
                /* linear byte b = 32j + lane  ->  permuted position 4*lane + j */
                byte = t * TILE_BYTES + 4 * (b % 32) + (b / 32);
            }
            uint8_t code = 0;
            for (int p = 0; p < k; p++) {
                uint8_t bit = (planes[((long long)p * rows + r) * rb + byte] >> (c & 7)) & 1u;
                code |= (uint8_t)(bit << (k - 1 - p));
            }
            codes[r * ld + c] = code;
        }
    return ORA_OK;
}

/* engine.py:35-46: masks by (B, d) */
static uint32_t swap_mask(int d) { return d == 1 ? 0x55555555u : d == 2 ? 0x33333333u : 0x0F0F0F0Fu; }

/* engine.py:48-72: in-place transpose of the B x B bit blocks of B words. */
static void bit_transpose_group(uint32_t* w, int b) {
    for (int d = 1; d < b; d <<= 1) {
        uint32_t mask = swap_mask(d);
        for (int r = 0; r < b; r++) {
            if (r & d) continue;
            uint32_t t = ((w[r] >> d) ^ w[r + d]) & mask;
            w[r] ^= t << d;
            w[r + d] ^= t;
        }
    }
}

/* engine.py:48-72 over arrays: words is (B, n) row-major. */
int ora_bit_transpose(uint32_t* words, int b, long long n) {
    if (b != 2 && b != 4 && b != 8) return ORA_PARAM;
    uint32_t w[8];
    for (long long i = 0; i < n; i++) {
        for (int r = 0; r < b; r++) w[r] = words[r * n + i];
        bit_transpose_group(w, b);
        for (int r = 0; r < b; r++) words[r * n + i] = w[r];
    }
    return ORA_OK;
}

static int width_for(int k) { return k <= 2 ? 2 : (k <= 4 ? 4 : 8); }

/* engine.py:75-92: plane words (k, n), MSB plane first -> (B, n). */
int ora_transpose_any_width(const uint32_t* plane_words, int k, long long n, uint32_t* out) {
    if (k < 2 || k > 8) return ORA_PARAM;
    int b = width_for(k);
    uint32_t w[8];
    for (long long i = 0; i < n; i++) {
        for (int r = 0; r < b; r++) w[r] = 0;
        for (int bit = 0; bit < k; bit++) w[bit] = plane_words[(long long)(k - 1 - bit) * n + i];
        bit_transpose_group(w, b);
        for (int r = 0; r < b; r++) out[(long long)r * n + i] = w[r];
    }
    return ORA_OK;
}

/* ---- GEMV / GEMM ------------------------------------------------------- */

typedef struct {
    const uint8_t* planes; /* permuted, (n_max, rows, padded/8) */
    long long rows, cols, padded;
    int n_max, k, merged, m;
    const float* lut32; /* (rows, 2^k) fp32 (tables32[k], engine.py:160-163) */
    const float* x;     /* (m, padded) fp32, zero padded (_prep_x) */
    float* y;           /* (m, rows) */
    long long r0, r1;
} job_t;

/* engine.py:212-246 + 187-195 for one (row, tile): decoded fp32 values in
 * WEIGHT order (vals[1024]). */
static void dequant_tile(const job_t* J, long long r, long long tile, float* vals) {
    const int k = J->k, b = width_for(k);
    const long long rb = J->padded / 8;
    const float* lut = J->lut32 + r * (1LL << k);
    for (int lane = 0; lane < LANES; lane++) {
        /* engine.py:180-184: little-endian u32 lane word from planes[:k] */
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int bit = 0; bit < k; bit++) {
            const uint8_t* src = J->planes + ((long long)(k - 1 - bit) * J->rows + r) * rb +
                                 tile * TILE_BYTES + 4 * lane;
            w[bit] = (uint32_t)src[0] | ((uint32_t)src[1] << 8) | ((uint32_t)src[2] << 16) |
                     ((uint32_t)src[3] << 24);
        }
        bit_transpose_group(w, b); /* engine.py:75-92 */
        float lanewise[32];
        if (J->merged) {
            /* engine.py:220-236: idx6 = (lo << 3) | hi -> (c_lo, c_hi) */
            for (int g = 0; g < 4; g++)
                for (int p = 0; p < 4; p++) {
                    uint32_t lo = (w[g] >> (8 * p)) & 7u, hi = (w[g] >> (8 * p + 4)) & 7u;
                    uint32_t idx6 = (lo << 3) | hi;
                    lanewise[8 * p + g] = lut[idx6 >> 3];     /* entries[8i+j][0] = c_i */
                    lanewise[8 * p + 4 + g] = lut[idx6 & 7u]; /* entries[8i+j][1] = c_j */
                }
        } else {
            /* engine.py:198-209: out[j] = (tw[j % B] >> (j // B) * B) & (2^B - 1) */
            uint32_t mask = (1u << b) - 1u;
            for (int j = 0; j < 32; j++) lanewise[j] = lut[(w[j % b] >> ((j / b) * b)) & mask];
        }
        /* engine.py:187-195: bit position j of lane t -> weight 256(j>>3)+8t+(j&7) */
        for (int j = 0; j < 32; j++) vals[256 * (j >> 3) + 8 * lane + (j & 7)] = lanewise[j];
    }
}

static void* gemm_worker(void* arg) {
    const job_t* J = (const job_t*)arg;
    const long long tiles = J->padded / TILE_WEIGHTS;
    float vals[TILE_WEIGHTS];
    float* partial = (float*)malloc(sizeof(float) * (size_t)(tiles * J->m));
    for (long long r = J->r0; r < J->r1; r++) {
        for (long long t = 0; t < tiles; t++) {
            dequant_tile(J, r, t, vals);
            /* engine.py:307-308 / 339-340: per-tile fp32 dot products */
            for (int m = 0; m < J->m; m++) {
                const float* xt = J->x + (long long)m * J->padded + t * TILE_WEIGHTS;
                float acc = 0.0f;
                for (int c = 0; c < TILE_WEIGHTS; c++) acc += vals[c] * xt[c];
                partial[m * tiles + t] = acc;
            }
        }
        /* engine.py:309 / 341: float32 sum over tiles, fixed order */
        for (int m = 0; m < J->m; m++) {
            float s = 0.0f;
            for (long long t = 0; t < tiles; t++) s += partial[m * tiles + t];
            J->y[(long long)m * J->rows + r] = s;
        }
    }
    free(partial);
    return NULL;
}

/* engine.py:284-309 (m == 1) and 312-341 (quantized path, any m).
 * planes: permuted (n_max, rows, padded/8); lut16: (rows, 2^k) fp16 bits;
 * x: (m, cols) fp32 (caller applies the activations_fp16 rounding);
 * y: (m, rows) fp32.  nthreads <= 0 means 1. */
int ora_gemm(const uint8_t* planes, long long rows, long long cols, long long padded, int n_max,
             int k, const uint16_t* lut16, const float* x, int m, float* y, int merged,
             int nthreads) {
    if (k < 2 || k > n_max || k > 8) return ORA_PARAM;
    if (merged && k != 3) return ORA_PARAM; /* engine.py:225-226 */
    if (m < 1) return ORA_SHAPE;
    if (nthreads < 1) nthreads = 1;
    long long nl = rows * (1LL << k);
    float* lut32 = (float*)malloc(sizeof(float) * (size_t)nl);
    float* xp = (float*)calloc((size_t)(m * padded), sizeof(float));
    ora_half_to_float(lut16, lut32, nl);
    for (int i = 0; i < m; i++) memcpy(xp + (long long)i * padded, x + (long long)i * cols, sizeof(float) * (size_t)cols);
    if (nthreads > rows) nthreads = (int)rows;
    job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int i = 0; i < nthreads; i++) {
        job_t* J = &jobs[i];
        J->planes = planes; J->rows = rows; J->cols = cols; J->padded = padded;
        J->n_max = n_max; J->k = k; J->merged = merged; J->m = m;
        J->lut32 = lut32; J->x = xp; J->y = y;
        J->r0 = rows * i / nthreads; J->r1 = rows * (i + 1) / nthreads;
        if (nthreads == 1) gemm_worker(J);
        else pthread_create(&th[i], NULL, gemm_worker, J);
    }
    if (nthreads > 1)
        for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    free(th); free(jobs); free(xp); free(lut32);
    return ORA_OK;
}

/* engine.py:357-362: dense fp32 weights from parent codes and table k. */
int ora_dequantize(const uint8_t* codes, long long rows, long long cols, long long ld, int n_max,
                   int k, const uint16_t* lut16, float* out) {
    if (k < 1 || k > n_max) return ORA_PARAM;
    for (long long r = 0; r < rows; r++)
        for (long long c = 0; c < cols; c++) {
            uint8_t code = (uint8_t)(codes[r * ld + c] >> (n_max - k)); /* quantizer.py:115-119 */
            out[r * cols + c] = half_to_float(lut16[r * (1LL << k) + code]);
        }
    return ORA_OK;
}
