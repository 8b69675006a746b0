/*
 * anyprec_b200.h -- C ABI of the B200-native bitplane any-precision hot path.
 *
 * Drop-in boundary for the reference package anyprec 0.1.0.  The reference has
 * no FFI: its "operator API" is the module-level Python functions of
 * anyprec.bitplane and anyprec.engine.  Each entry point below replaces one of
 * them (file:line under /root/reference/pkg/src/anyprec/) and is what a
 * ctypes / cffi binding added to the reference would call.
 *
 * Conventions
 *   - All pointers are DEVICE pointers (cudaMalloc / torch CUDA storage) unless
 *     a parameter name starts with h_.  The library never allocates device
 *     memory inside a call and keeps no global mutable state besides a one-time
 *     kernel attribute setup; every call is reentrant from many host threads.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Kernels are launched on it; calls do not synchronise.
 *   - Planes: uint8 [n_max][rows][padded_cols/8]; plane p holds code bit
 *     n_max-1-p (MSB first, bitplane.py:76-100); byte b bit i = weight 8b+i;
 *     padded_cols = ceil(cols/1024)*1024 (bitplane.py:72-73).  "permuted"
 *     layout applies out[4t+j] = in[32j+t] inside every 128-byte tile
 *     (bitplane.py:31-37, 121-130) and is what the GEMV reads.
 *   - Centroid tables: IEEE fp16 bit patterns, uint16 [rows][1<<k], one table
 *     per bit-width k (quantizer.py:75-119 AnyPrecisionLayer.centroid_tables[k]).
 *   - Activations: fp16 [m][ldx], ldx % 8 == 0, 16-byte aligned base.
 *   - Return value: APB_OK or an apb_status error code; validation happens on
 *     the host before any launch (engine.py:263-281 raise-before-compute).
 */
#ifndef ANYPREC_B200_H
#define ANYPREC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python shim maps them onto the reference exception
 * classes of errors.py:4-35. */
typedef enum {
    APB_OK = 0,
    APB_ERR_SHAPE = 1,      /* ShapeError      (errors.py:8-9)   */
    APB_ERR_PARAM = 2,      /* ParameterError  (errors.py:12-13) */
    APB_ERR_LAYOUT = 3,     /* LayoutError     (errors.py:20-21) */
    APB_ERR_CODE_RANGE = 4, /* CodeRangeError  (errors.py:16-17) */
    APB_ERR_CUDA = 5,       /* CUDA launch / runtime failure    */
    APB_ERR_NCCL = 6        /* reserved for the collective path */
} apb_status;

enum { APB_DTYPE_F32 = 0, APB_DTYPE_F16 = 1 };

/* apb_gemv* flags.  APB_FLAG_PDL launches with programmatic stream
 * serialisation: the kernel may start (and read planes / tables) while the
 * previous kernel in the stream is still running, and waits for it before
 * reading activations or writing outputs.  Only set it when the preceding
 * kernel does not write the planes or tables of this call. */
enum { APB_FLAG_PDL = 1 };
/* APB_FLAG_GLU: every problem's rows are interleaved (gate_i, up_i) pairs (rows
 * even) and the output has rows / 2 values per batch row,
 * y[m][i] = silu(gate_i . x_m) * (up_i . x_m), from the fp32 row sums, rounded
 * once to y_dtype (the Llama MLP's SiLU * up fused into the gate/up GEMV).
 * TMA kernel only (k 3..8, m_x <= 8, <= 16 problems); else APB_ERR_PARAM. */
enum { APB_FLAG_GLU = 2 };

/* Host-path plumbing: async copy on a stream (kind 0 H2D, 1 D2H, 2 D2D) and a
 * stream synchronisation (for bindings without their own CUDA runtime). */
int apb_memcpy_async(void* dst, const void* src, int64_t bytes, int kind, void* stream);
int apb_stream_sync(void* stream);

/* Library version (major*10000 + minor*100 + patch) and status strings. */
int apb_version(void);
const char* apb_status_string(int status);

/* bitplane.py:72-73 pad_columns. */
int64_t apb_pad_columns(int64_t cols);

/* bitplane.py:76-100 pack_bitplanes (+ bitplane.py:126-130 permute_layout when
 * permuted != 0), in one pass.  codes: uint8 [rows][ld_codes]; planes must hold
 * n_max*rows*padded_cols/8 bytes.  If d_code_or is not NULL it receives (OR=)
 * the bitwise OR of every code so the caller can raise CodeRangeError
 * (bitplane.py:88-91) with one 4-byte read; it must be zeroed by the caller. */
int apb_pack(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ld_codes, int n_max,
             int permuted, uint8_t* planes, uint32_t* d_code_or, void* stream);

/* bitplane.py:121-136 permute_layout (inverse=0) / inverse_permute_layout (1).
 * in and out must not alias. */
int apb_permute(const uint8_t* in, uint8_t* out, int n_planes, int64_t rows,
                int64_t padded_cols, int inverse, void* stream);

/* bitplane.py:103-118 unpack_codes: k-bit prefix codes from planes[0..k-1]
 * only -> uint8 [rows][ld_codes] (cols valid columns per row). */
int apb_unpack(const uint8_t* planes, int n_max, int64_t rows, int64_t cols,
               int64_t padded_cols, int permuted, int k, uint8_t* codes, int64_t ld_codes,
               void* stream);

/* engine.py:75-92 transpose_any_width (k in 2..8) over n word groups:
 * plane_words uint32 [k][n] (MSB plane first) -> out uint32 [B][n],
 * B = 2 (k<=2), 4 (k<=4) or 8.  engine.py:48-72 bit_transpose is k = B with
 * the plane order reversed. */
int apb_transpose_words(const uint32_t* plane_words, int k, int64_t n, uint32_t* out,
                        void* stream);

/* engine.py:284-309 gemv and engine.py:312-341 gemm (quantized path).
 * Reads ONLY planes[0..k-1] (permuted layout) and the k-bit table lut
 * (uint16 fp16 [rows][1<<k]).
 *   x      : fp16 [m_x][ldx] activations.  With x_split = 1 the m_x rows are
 *            (hi, lo) pairs of an fp32 activation (x = hi + lo) and the output
 *            has m_x/2 rows: y[m] = W.(x_hi[m]) + W.(x_lo[m]).  x_split = 2
 *            ("scaled pairs", apb_split_x_scaled): the pairs hold x * s_m with
 *            s_m a power of two, and m_x/2 floats 1/s_m follow the rows in the
 *            same buffer (element offset m_x * ldx): y[m] = (W.hi + W.lo) / s_m,
 *            so fp32 activations of any magnitude keep ~22 significant bits.
 *   y      : [m_out][ldy] of y_dtype (APB_DTYPE_F32 or APB_DTYPE_F16).
 * Accumulation is fp32 in a fixed order; results are bit-reproducible for
 * identical inputs and independent of planes k..n_max-1 (test_engine.py:165-176). */
int apb_gemv(const uint8_t* planes, int n_max, int64_t rows, int64_t cols, int64_t padded_cols,
             int k, const uint16_t* lut, const uint16_t* x, int m_x, int64_t ldx, int x_split,
             void* y, int y_dtype, int64_t ldy, int flags, void* stream);

/* Grouped form of apb_gemv: n_problems independent layers (same k, m_x,
 * x_split, y_dtype) in ONE launch, e.g. the seven linears of a decoder block.
 * Arrays of per-problem pointers/shapes live in HOST memory. */
int apb_gemv_grouped(int n_problems, const uint8_t* const* planes, const int* n_max,
                     const int64_t* rows, const int64_t* cols, const int64_t* padded_cols, int k,
                     const uint16_t* const* lut, const uint16_t* const* x, int m_x,
                     const int64_t* ldx, int x_split, void* const* y, int y_dtype,
                     const int64_t* ldy, int flags, void* stream);

/* Caller-owned launch plan for repeated calls with the same layers / shapes:
 * apb_gemv_plan_create validates and prepares everything of an
 * apb_gemv_grouped call except the activation / output pointers (tensor maps,
 * partition, launch shape) and returns an opaque heap object (NULL when the
 * call is not served by the TMA kernel, e.g. m_x > 8: use apb_gemv_grouped).
 * apb_gemv_plan_launch launches it with new x / y pointers (NULL: keep the
 * previous ones; same shapes, x 16-byte aligned).  A plan is not thread-safe;
 * destroy it with apb_gemv_plan_destroy. */
void* apb_gemv_plan_create(int n_problems, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
                           const int64_t* cols, const int64_t* padded_cols, int k, const uint16_t* const* lut,
                           const uint16_t* const* x, int m_x, const int64_t* ldx, int x_split, void* const* y,
                           int y_dtype, const int64_t* ldy, int flags);
int apb_gemv_plan_launch(void* plan, const uint16_t* const* x, void* const* y, void* stream);
void apb_gemv_plan_destroy(void* plan);

/* engine.py:312-341 small-batch GEMM (SURVEY 8(b) name): apb_gemv over m
 * activation rows X [m][ldx] -> Y [m][ldy]. */
int apb_gemm_small(const uint8_t* planes, int n_max, int64_t rows, int64_t cols, int64_t padded_cols, int k,
                   const uint16_t* lut, int m, const uint16_t* X, int64_t ldx, void* Y, int y_dtype, int64_t ldy,
                   void* stream);

/* engine.py:357-362 dequantize, from the top-k planes: w [rows][ldw] of
 * w_dtype (fp16 is exact: the values ARE fp16 table entries). */
int apb_dequant(const uint8_t* planes, int n_max, int64_t rows, int64_t cols,
                int64_t padded_cols, int permuted, int k, const uint16_t* lut, void* w,
                int w_dtype, int64_t ldw, void* stream);

/* Dense path activation split (engine.py:343-354 at fp32 accuracy on tensor
 * cores): out rows [0, m) = hi = fp16(x * s_r), rows [m, 2m) = lo =
 * fp16(x * s_r - hi), inv_scale[r] = 1 / s_r with s_r the power of two that
 * puts row r's max |x| in [2^14, 2^15).  Y = (hi.W^T + lo.W^T) * inv_scale. */
int apb_split_hilo(const float* x, int64_t m, int64_t cols, int64_t ldx, uint16_t* out, int64_t ld,
                   float* inv_scale, void* stream);

/* Dense path as ONE Blackwell kernel (engine.py:343-354: dequantize + fp32
 * GEMM).  apb_dense_prep_x writes the activations in the
 * kernel's K order (within each 1024-column tile, 64-column block v holds
 * bitplane lane words 2v, 2v+1: element 32h + 8p + b = column 256p + 16v + 8h + b),
 * xp [mx][padded_cols] fp16 with zeros past cols: fp16 x -> mx = m rows; fp32 x
 * -> mx = 2m rows, (hi, lo) = (fp16(x*s), fp16(x*s - hi)) at rows (2i, 2i+1)
 * with s an exact power of two per row and inv[i] = 1/s.
 * apb_gemm_dense_tc: y [m_out][ldy] fp32 = dequant_k(W) . x^T with the top-k
 * planes + fp16 table decoded straight into the tcgen05.mma A operand in shared
 * memory (no dense weight tensor), x tiles by TMA, fp32 accumulation in tensor
 * memory; pairs = 1: m_out = mx / 2 and y = (hi-product + lo-product) * inv. */
int apb_dense_prep_x(const void* x, int x_dtype, int64_t m, int64_t cols, int64_t ldx, uint16_t* xp,
                     int64_t padded_cols, float* inv, void* stream);
int apb_gemm_dense_tc(const uint8_t* planes, int n_max, int64_t rows, int64_t cols, int64_t padded_cols,
                      int k, const uint16_t* lut, const uint16_t* xp, int64_t mx, int pairs,
                      const float* inv, float* y, int64_t ldy, float* ws, int64_t ws_bytes, void* stream);
/* Workspace bytes apb_gemm_dense_tc uses for split-K on this device (0: none):
 * when the output tiles cannot cover the SMs (small batch), K is split into
 * 2..8 chunks whose fp32 partial tiles are summed in fixed order by a second
 * kernel (deterministic).  ws = NULL / too small -> a single pass. */
int64_t apb_gemm_dense_tc_workspace(int64_t rows, int64_t padded_cols, int64_t mx);

/* Helper for the fp32-activation path: x fp32 [m][ldx_in] -> fp16 pairs
 * out [2m][ldx_out] with out[2i] = fp16(x[i]), out[2i+1] = fp16(x[i]-out[2i]).
 * Columns cols..ldx_out-1 are zero-filled.  With round_only = 1 it writes
 * m rows fp16(x[i]) only (activations_fp16, engine.py:276-277). */
int apb_split_x(const float* x, int m, int64_t cols, int64_t ldx_in, uint16_t* out,
                int64_t ldx_out, int round_only, void* stream);

/* x_split = 2 operand (engine.py:270-281 for fp32 activations): out [2m][ldx_out]
 * = (hi, lo) pairs of x * s_r (s_r: the power of two putting row r's max |x| in
 * [2^14, 2^15); hi = fp16(x*s_r), lo = fp16(x*s_r - hi), columns >= cols zero),
 * followed by m floats 1/s_r at element offset 2m * ldx_out (ldx_out even). */
int apb_split_x_scaled(const float* x, int m, int64_t cols, int64_t ldx_in, uint16_t* out,
                       int64_t ldx_out, void* stream);

/* Fused glue of a decoder block around the GEMVs (decode-step measurement,
 * BASELINE config C5; outside the reference's hot path).  Device pointers,
 * fp16 = uint16 bit patterns, one token wide.
 *   apb_rms_residual: resid (f32) += add (f16, may be NULL); out = rmsnorm(resid) * w
 *   apb_rope_cache  : q_out = rope(q); k_cache[h][.] = rope(k); v_cache[h][.] = v
 *                     (cache pointers at the new position, head stride in elements)
 *   apb_silu_mul    : out = silu(gate) * up */
int apb_rms_residual(float* resid, const uint16_t* add, const uint16_t* w, uint16_t* out, int64_t n, float eps,
                     void* stream);
int apb_rope_cache(const uint16_t* q, const uint16_t* k, const uint16_t* v, const float* cosv, const float* sinv,
                   uint16_t* q_out, uint16_t* k_cache, uint16_t* v_cache, int heads, int head_dim,
                   int64_t cache_head_stride, void* stream);
int apb_silu_mul(const uint16_t* gate, const uint16_t* up, uint16_t* out, int64_t n, void* stream);
/* decode-step ends: resid = float(embed[*token]) and out = fp16(rmsnorm(resid) * w);
 * argmax of an fp16 vector (first index on ties) into *out. */
int apb_embed_rms(const uint16_t* embed, const int64_t* token, int64_t n, float* resid, const uint16_t* w,
                  uint16_t* out, float eps, void* stream);
int apb_argmax_f16(const uint16_t* x, int64_t n, int64_t* out, void* stream);

/* Single-query decode attention with RoPE and KV-cache append fused in
 * (head_dim 128).  q, k, v: this token's projections (heads x head_dim fp16);
 * k_cache / v_cache: row 0 of head 0, heads `cache_head_stride` elements apart;
 * rows 0..pos-1 hold the past, the rotated k and v of this token are written to
 * row pos, and out[h] = softmax(scale * rot(q_h) . K_h[0..pos]) V_h[0..pos]
 * (fp16, heads x head_dim).  workspace: >= apb_attention_decode_workspace(
 * heads, head_dim, pos + 1) bytes, zero-filled once before first use (the
 * kernel leaves it reusable).  next_k_cache / next_v_cache (NULL or both set,
 * same geometry): the next block's cache, whose rows 0..pos are prefetched into
 * L2 for its own attention call.  Launched with programmatic stream
 * serialisation like the GEMVs. */
int64_t apb_attention_decode_workspace(int heads, int head_dim, int64_t max_keys);
int apb_attention_decode(const uint16_t* q, const uint16_t* k, const uint16_t* v, const float* cosv,
                         const float* sinv, uint16_t* k_cache, uint16_t* v_cache, int heads, int head_dim,
                         int64_t cache_head_stride, int pos, float scale, void* workspace,
                         int64_t workspace_bytes, uint16_t* out, const uint16_t* next_k_cache,
                         const uint16_t* next_v_cache, void* stream);

/* ---- RMSNorm folded into the GEMV epilogues (decode step) ----
 * rmsnorm(r) . w = s * (r . w) with the scalar s = rsqrt(mean(r^2) + eps), so
 * W (rmsnorm(r) . w) = s * (W (r . w)):
 *   mode 1 (producer, e.g. the o / down projection; m_x = 1, one problem, fp16
 *     y): resid[i] += (W x)[i] (fp32), y[i] = fp16(resid[i] * norm_w[i]) -- the
 *     next GEMV's activation -- and partials[cta] = this CTA's sum of resid^2
 *     (partials: zero-filled once, n_partials >= the launch's grid -- 320
 *     covers every grid on a 148-SM B200 -- else APB_ERR_PARAM);
 *   mode 2 (consumer, e.g. q/k/v or gate/up): every row sum is multiplied by
 *     s = rsqrt(sum(partials[0..min(n_partials, 320))) / norm_size + eps)
 *     (summed in a fixed order: deterministic) before the GLU epilogue / the
 *     store.
 * TMA kernel only (k 3..8). */
typedef struct {
    int mode;               /* 0 none, 1 producer, 2 consumer */
    float* resid;           /* mode 1: [rows] fp32 residual stream */
    const uint16_t* norm_w; /* mode 1: [rows] fp16 RMSNorm weight */
    float* partials;        /* mode 1: written; mode 2: read */
    int n_partials;
    int norm_size;          /* mode 2: hidden size */
    float eps;              /* mode 2 */
} apb_norm_epilogue;
int apb_gemv_grouped_norm(int n_problems, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
                          const int64_t* cols, const int64_t* padded_cols, int k, const uint16_t* const* lut,
                          const uint16_t* const* x, int m_x, const int64_t* ldx, void* const* y, int y_dtype,
                          const int64_t* ldy, const apb_norm_epilogue* norm, int flags, void* stream);

/* ---- row-sharded GEMV with the all-gather fused in ----
 * apb_gemv_grouped_peers: apb_gemv_grouped over this rank's row slab (y[i] =
 * this rank's rows inside its full output) that also stores every y value at
 * the same place of each peer's output -- y_peers[i * n_peers + j] is problem
 * i's y pointer as mapped from peer j (CUDA IPC / NVLink P2P), n_peers <= 7
 * other ranks -- and, per CTA, adds the number of values it wrote to every
 * rank's arrival counter (peer_flags[0..n_peers-1] the peers', then
 * peer_flags[n_peers] this rank's own) with release semantics at system scope.
 * k 3..8, m_x <= 8, <= 16 problems, <= 64K columns.
 * apb_peer_wait: on the stream, wait until *arrivals has grown by per_step
 * (the full output's values) since the previous wait (*expected tracks the
 * target in device memory: graph-replayable); gives up after spin_limit polls
 * and sets *status = 1.
 * apb_peer_alloc / open / close / free: cudaMalloc'd (zeroed) region + its
 * IPC handle (apb_peer_handle_bytes() bytes), and the peer-side mapping. */
int apb_gemv_grouped_peers(int n_problems, const uint8_t* const* planes, const int* n_max, const int64_t* rows,
                           const int64_t* cols, const int64_t* padded_cols, int k, const uint16_t* const* lut,
                           const uint16_t* const* x, int m_x, const int64_t* ldx, int x_split, void* const* y,
                           int y_dtype, const int64_t* ldy, int n_peers, void* const* y_peers,
                           uint32_t* const* peer_flags, int flags, void* stream);
/* SURVEY 8(b) name of the single-layer form: this rank's row slab
 * [row_offset, row_offset + rows) of a [m_x][ldy] output written into every
 * rank's output y_ranks[r] (as mapped here) + the arrival counters flag_ranks[r]. */
int apb_gemv_allgather(const uint8_t* planes, int n_max, int64_t rows, int64_t cols, int64_t padded_cols, int k,
                       const uint16_t* lut, const uint16_t* x, int m_x, int64_t ldx, int rank, int world,
                       void* const* y_ranks, int64_t row_offset, int y_dtype, int64_t ldy,
                       uint32_t* const* flag_ranks, int flags, void* stream);
int apb_peer_wait(const uint32_t* arrivals, uint32_t* expected, uint32_t per_step, int* status,
                  long long spin_limit, void* stream);
int apb_peer_alloc(int64_t bytes, void** ptr, void* handle);
int apb_peer_open(const void* handle, void** ptr);
int apb_peer_close(void* ptr);
int apb_peer_free(void* ptr);
int apb_peer_handle_bytes(void);

/* ---- offline quantizer (reference quantizer.py:370-435, clustering.py:89-302) ----
 * Sensitivity-weighted exact 1-D k-means seed (2^n_min clusters per row, by
 * dynamic programming) and one exact weighted 2-means split per extra bit up to
 * n_max; bit-exact with the reference's float64 arithmetic.  All pointers are
 * device memory:
 *   weights, sens : [rows][n] float64 (sens already coerced: finite, >= 0, every
 *                   row sum > 0 -- quantizer.py:195-212)
 *   order         : [rows][n] int64, the STABLE ascending argsort of each row
 *   codes         : [rows][n] uint8 parent (n_max-bit) codes
 *   tables        : the fp16 centroid tables for k = n_min..n_max concatenated,
 *                   [rows][2^k] each
 *   sse           : [n_max-n_min+1][rows] float64 weighted SSE per bit-width
 *   level_codes   : NULL or [n_max-n_min+1][rows][n] uint8 codes at every k
 *   workspace     : >= apb_quant_workspace(rows, n, n_min, n_max) bytes,
 *                   16-byte aligned */
int64_t apb_quant_workspace(int rows, int n, int n_min, int n_max);
int apb_quant_build(const double* weights, const double* sens, const int64_t* order, int rows, int n, int n_min,
                    int n_max, uint8_t* codes, uint16_t* tables, double* sse, uint8_t* level_codes,
                    void* workspace, int64_t workspace_bytes, void* stream);
/* continue_upscale (quantizer.py:438-512): extend stored k0-bit codes (codes_in,
 * [rows][n]) with fp16 table table_k0 ([rows][2^k0]) to new_n_max bits by
 * splitting; codes / tables (k0+1..new_n_max concatenated) / sse
 * ([new_n_max-k0][rows]) as in apb_quant_build; *bad |= 1 when some row's codes
 * are not value-contiguous (the caller raises).  Workspace:
 * apb_quant_workspace(rows, n, 2, new_n_max).
 * apb_quant_sse_levels: np.sum(sens * (w - table_k[codes >> shift])**2, axis=1)
 * in original column order (the record of the levels <= k0). */
int apb_quant_continue(const double* weights, const double* sens, const int64_t* order, const uint8_t* codes_in,
                       const uint16_t* table_k0, int rows, int n, int k0, int new_n_max, uint8_t* codes,
                       uint16_t* tables, double* sse, int* bad, void* workspace, int64_t workspace_bytes,
                       void* stream);
/* cluster_rows / quantize_seed / kmeans_1d_weighted (clustering.py:204-227,
 * quantizer.py:122-157, 281-307) for any cluster count 1 <= k <= 4096: per
 * row the exact weighted k-means bounds over the sorted order ([rows][k+1],
 * trailing empty intervals of low-distinct rows end at n), float64 centroids
 * ([rows][k], an empty interval copies the previous column) and, if codes is
 * not NULL, each element's interval index in original order ([rows][n]).
 * sens must be coerced by the caller; order is the stable argsort. */
/* upscale (quantizer.py:310-367), one bit more for each row: value-contiguous
 * codes (in each row's sorted order) go through the split kernels with the
 * float64 centroids `parents` [rows][2^k0] (workspace:
 * apb_quant_workspace(rows, n, 2, k0 + 1); *bad |= 1 if some row is not
 * contiguous); other codes through apb_quant_upscale_general (gorder = stable
 * sort by (code, value), scratch >= rows * (2n + 3(n + 2^k0 + 1)) doubles).
 * Outputs: codes [rows][n] uint8 and float64 centroids [rows][2^(k0+1)]. */
int apb_quant_upscale(const double* weights, const double* sens, const int64_t* order, const uint8_t* codes_in,
                      const double* parents, int rows, int n, int k0, uint8_t* codes, double* means, int* bad,
                      void* workspace, int64_t workspace_bytes, void* stream);
int apb_quant_upscale_general(const double* weights, const double* sens, const int64_t* gorder,
                              const uint8_t* codes_in, const double* parents, int rows, int n, int k0,
                              uint8_t* codes, double* means, double* scratch, void* stream);
/* split_boundaries (clustering.py:252-302): rows of sorted values sv with
 * weights sw ([rows][n], identity = 0..n-1 per row as int64), interval bounds
 * [rows][2^log2m + 1] -> the 2-means split of every interval
 * out [rows][2^(log2m+1) + 1] (prefix sums recomputed like _prefix_sums).
 * Workspace: apb_quant_workspace(rows, n, 2, log2m + 1). */
int apb_quant_split(const double* sv, const double* sw, const int64_t* identity, int rows, int n, int log2m,
                    const int* bounds, int* out, void* workspace, int64_t workspace_bytes, void* stream);
int64_t apb_quant_cluster_workspace(int rows, int n, int k);
int apb_quant_cluster(const double* weights, const double* sens, const int64_t* order, int rows, int n, int k,
                      int* bounds, double* means, int* codes, void* workspace, int64_t workspace_bytes,
                      void* stream);
int apb_quant_sse_levels(const double* weights, const double* sens, const uint8_t* codes, int shift,
                         const uint16_t* table_k, int k, int rows, int n, double* sse, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ANYPREC_B200_H */
