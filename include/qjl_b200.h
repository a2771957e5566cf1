/*
 * qjl_b200.h -- C ABI of the B200-native (sm_100a) QJL decode-time key path.
 *
 * Plain C: raw device pointers, sizes, and a cudaStream_t passed as void*.
 * Every entry point returns an int status (0 = OK, < 0 = error; see
 * qjl_status_string / qjl_last_error).  The library allocates no persistent
 * device memory: caches, sketches, outputs and workspaces are owned by the
 * caller (PyTorch tensors in the Python host layer).  Calls are stream
 * ordered; readers pass the prefix length `n`, which gives the reference's
 * "consistent prefix" semantics (kvcache.py:189-196).
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   qjl_detect_outliers  <- detect_outliers            pkg/src/qjl/kvcache.py:104-123
 *   qjl_build_sketch     <- KeyCacheState.create/__init__ sketch split
 *                                                       pkg/src/qjl/kvcache.py:198-267
 *   qjl_prefill_profile  <- detect_outliers + KeyCacheState.create, fused
 *   qjl_quantize_keys    <- KeyCacheState.append -> quantize_key (x2 sides)
 *                                                       pkg/src/qjl/kvcache.py:293-306,
 *                                                       pkg/src/qjl/estimator.py:110-124
 *   qjl_sketch_query     <- sketch_query               pkg/src/qjl/estimator.py:127-132
 *   qjl_scores           <- KeyCacheState.estimate_logits -> _side_logits ->
 *                           packed_sign_dot_batch       pkg/src/qjl/kvcache.py:311-329,
 *                                                       pkg/src/qjl/estimator.py:149-170
 *   qjl_softmax_f64      <- softmax / estimate_scores  pkg/src/qjl/kvcache.py:38-44, :331-337
 *   qjl_decode           <- quantized_decode (scores + softmax + weights @ values)
 *                                                       pkg/src/qjl/attention.py:56-71
 *   qjl_quantize_values  <- quantize_value             pkg/src/qjl/kvcache.py:140-161
 *   qjl_decode_step      <- append + quantize_value + quantized_decode, one step
 *                                                       kvcache.py:293-306, attention.py:56-71
 *   qjl_orthogonalize    <- orthogonalize (batched)   pkg/src/qjl/sketch.py:82-103
 *   qjl_qjlc_export      <- write_cache record loop    pkg/src/qjl/kvcache.py:389-437
 *   qjl_qjlc_import      <- read_cache record loop     pkg/src/qjl/kvcache.py:440-520
 *
 * Data layout in HBM (unit = one (batch, kv-head) pair; rows padded to 128-token tiles):
 *   key cache   bits_in  u8  [row][m_in/8]    LSB-first sign bits; byte-identical to the
 *                                            reference's LE u64 words when m % 64 == 0
 *               bits_out u8  [row][m_out/8]
 *               norm_in  f16 [row]            ||k_inlier||_2
 *               norm_out f16 [row]            ||k_outlier||_2
 *   value cache P2T (tensor-core path): 2-bit codes, group 32, d = 128, fp16 zero/scale
 *               codes u8 [tile][4096]: byte (d/4)*128 + (t%128)/4*4 + t%4 holds dims
 *               4(d/4)..+3 of token t at bits 2(d%4)..+1 (one u32 = 4 tokens x 4 dims)
 *               zero f16 [row][d/32], scale f16 [row][d/32]
 *   value cache U8 (reference format): 1 byte per code, any bits 1..8, any group dividing
 *               d, fp32 zero/scale per (token, group) -- rows layout only.
 *   Row addressing (tile_stride, both cache structs):
 *     tile_stride == 0  rows layout: every array is [units][capacity][row bytes];
 *     tile_stride  > 0  tile-major records: row r of unit u of every array lives at
 *                       array + (u * capacity/128 + r/128) * tile_stride + (r%128) * row bytes
 *                       (P2T codes: + the in-tile offset above).  capacity % 128 == 0.
 *   The tensor-core decode streams one contiguous record per (unit, 128-token tile):
 *     [bits_in 128*m_in/8][bits_out 128*m_out/8][norm_in 256][norm_out 256 if m_out]
 *     [codes 4096][zero 1024][scale 1024]            (qjl_tile_record, QJL_REC_*)
 *   so a P2T value cache must be the tail of the same records as its key cache.
 *   sketch      s_full [units or 1][m_in+m_out][d]: rows 0..m_in-1 hold S_in at the
 *               inlier columns (zeros at outlier columns), rows m_in.. hold S_out at
 *               the outlier columns -- one zero-padded K=d GEMM per unit.
 */
#ifndef QJL_B200_H
#define QJL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QJL_ABI_VERSION 3

#if defined(__GNUC__)
#define QJL_API __attribute__((visibility("default")))
#else
#define QJL_API
#endif

enum {
  QJL_OK = 0,
  QJL_ERR_ARG = -1,          /* shape / parameter error  -> Python ValueError   */
  QJL_ERR_UNSUPPORTED = -2,  /* valid but unsupported configuration             */
  QJL_ERR_CUDA = -3,         /* CUDA runtime / launch error -> RuntimeError     */
  QJL_ERR_WORKSPACE = -4,    /* workspace too small                             */
  QJL_ERR_EMPTY = -5         /* empty cache (kvcache.py:324-325)                */
};

enum { QJL_F32 = 0, QJL_F16 = 1, QJL_BF16 = 2, QJL_F64 = 3 };
enum { QJL_VLAYOUT_U8 = 0, QJL_VLAYOUT_P2T = 2 };
/* qjl_tile_record field indices */
enum { QJL_REC_BITS_IN = 0, QJL_REC_BITS_OUT, QJL_REC_NORM_IN, QJL_REC_NORM_OUT, QJL_REC_CODES,
       QJL_REC_ZERO, QJL_REC_SCALE, QJL_REC_FIELDS };
/* qjl_decode / qjl_decode_step / qjl_scores flags */
enum {
  /* The previous kernel on `stream` is a qjl_decode / qjl_decode_step / qjl_scores of this
   * library, and every input of this call (cache rows, q, k_new, v_new, sketch) was
   * written before that launch: the query-sketch kernel may then read its inputs while the
   * previous decode drains (programmatic dependent launch).  Without it every read waits
   * for the stream.  (qjl_scores: tensor-core path only; the generic path ignores it.) */
  QJL_DECODE_CHAINED = 1,
  /* Fixed 512-token segments per unit, merged in segment order: a unit's output bits depend
   * only on that unit (a unit-sharded decode equals the unsharded one bit for bit).  The
   * default schedule splits the flattened (unit, tile) space evenly over the CTAs, so a
   * unit's partial sums follow the launch's total size (equal within rounding). */
  QJL_DECODE_DETERMINISTIC = 2
};

typedef struct qjl_key_cache {
  uint8_t* bits_in;
  uint8_t* bits_out;   /* NULL when m_out == 0 */
  uint16_t* norm_in;
  uint16_t* norm_out;  /* NULL when m_out == 0 */
  int64_t capacity;
  int32_t units, d, m_in, m_out;
  int64_t tile_stride;   /* 0: rows layout; > 0: tile-major records of this many bytes */
} qjl_key_cache_t;

typedef struct qjl_value_cache {
  void* codes;
  void* zero;
  void* scale;
  int64_t capacity;
  int32_t units, d, bits, group, layout;
  int32_t pad_;
  int64_t tile_stride;   /* P2T: the key cache's record bytes; U8: 0 */
} qjl_value_cache_t;

typedef struct qjl_sketch {
  const void* s_full;   /* [units or 1][m_in + m_out][d] */
  int32_t dtype;        /* QJL_F64 / QJL_F32 / QJL_BF16 / QJL_F16 */
  int32_t pad_;
  int64_t unit_stride;  /* elements between consecutive units; 0 = shared */
} qjl_sketch_t;

QJL_API int qjl_abi_version(void);
QJL_API const char* qjl_status_string(int status);
/* Detail message of the last failing call on this host thread. */
QJL_API const char* qjl_last_error(void);
/* SM count / compute capability of the current device. */
QJL_API int qjl_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* Outlier profile per unit: top-h channels by mean |k| over n0 prompt rows,
 * fp64 accumulation, ties -> lower index, channels sorted ascending.
 * keys: [units][n0][d] (rows contiguous, unit stride in elements).
 * channels: int32 [units][h]; magnitudes: f64 [units][d] (may be NULL). */
QJL_API int qjl_detect_outliers(const void* keys, int dtype, int units, int64_t n0, int d,
                        int64_t unit_stride, int h, int32_t* channels,
                        double* magnitudes, void* ws, size_t ws_bytes, void* stream);
/* Device workspace (bytes) qjl_detect_outliers / qjl_prefill_profile use for `units`
 * prompts of n0 keys of dimension d: fp64 per-block channel partials (0: none needed).
 * ws == NULL makes the call allocate it stream-ordered (cudaMallocAsync) itself. */
QJL_API size_t qjl_detect_workspace(int units, int64_t n0, int d);

/* Build per-unit zero-padded sketches from device fp64 S_in [m_in][d-h] and
 * S_out [m_out][h] (either may be NULL when its side is empty) and channels
 * [units][h].  Output s_full [units][m_in+m_out][d] in `dtype` (RN rounding). */
QJL_API int qjl_build_sketch(const double* s_in, const double* s_out, int m_in, int m_out,
                     int d, int h, const int32_t* channels, int units, int dtype,
                     void* s_full, void* stream);

/* Fused prefill profile: detect_outliers + per-unit S_full build in
 * one pass over the prompt -- per-block channel partials, then CTAs per unit sum them
 * in a fixed order, rank, write channels / magnitudes and scatter S_in / S_out into
 * the unit's zero-padded S_full from the ranks they hold.  s_in [m_in][d-h] and
 * s_out [m_out][h] are given in the operand dtype `sketch_dtype` (rounded once, as
 * qjl_build_sketch rounds them).  Same outputs, bit for bit, as qjl_detect_outliers
 * followed by qjl_build_sketch (kvcache.py:104-123, :198-267). */
QJL_API int qjl_prefill_profile(const void* keys, int dtype, int units, int64_t n0, int d,
                                int64_t unit_stride, int h, const void* s_in, const void* s_out,
                                int m_in, int m_out, int sketch_dtype, int32_t* channels,
                                double* magnitudes, void* s_full, void* ws, size_t ws_bytes,
                                void* stream);

/* K1: append n keys per unit at rows [row_offset, row_offset + n).
 * keys: [units][n][d] with `key_unit_stride` elements between units (0: every unit
 * quantizes the same n keys, e.g. one key set under many per-unit sketches).
 * channels: [units][h] outlier channels (for the norm split), may be NULL if h == 0. */
QJL_API int qjl_quantize_keys(const void* keys, int dtype, int64_t n, int64_t key_unit_stride,
                      const qjl_sketch_t* sketch, const int32_t* channels, int h,
                      const qjl_key_cache_t* cache, int64_t row_offset, void* stream);

/* S_full @ q per unit and query head (fp64 accumulation): q [units][G][d] ->
 * sq [units][G][m_in+m_out] in sq_dtype (QJL_F32 or QJL_F64). */
QJL_API int qjl_sketch_query(const void* q, int q_dtype, int units, int G, int d,
                     const qjl_sketch_t* sketch, int m_total, int sq_dtype, void* sq, void* stream);

/* Canonical tile record (see the layout above): byte offsets of the QJL_REC_* fields
 * within one 128-token record (-1 for absent fields: no outlier side, or no values when
 * values == 0) and the record size in bytes, or -1 for an unsupported shape.
 * values != 0 appends the P2T value fields (d == 128). */
QJL_API int64_t qjl_tile_record(int d, int m_in, int m_out, int values, int64_t* offsets);

/* Which kernels a call would run: 1 when qjl_decode (values != NULL) / qjl_scores
 * (values == NULL) takes the tensor-core path for this cache and head count, 0 when the
 * generic kernels run (or, for P2T values, when the call would be rejected), < 0 on bad args. */
QJL_API int qjl_tensor_core_path(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int G);

/* K2: logits [units][G][n] (f32) of G query heads per unit over the first n keys.
 * Tile-major caches with m_in/32 in {8, 16}, m_out/32 in {0, 2, 4}, d == 128 and G <= 4
 * run the tensor-core score kernel; every other shape runs the generic kernel.
 * flags: QJL_DECODE_CHAINED (ABI 3; other bits are rejected). */
QJL_API size_t qjl_scores_workspace(int units, int G, int m_total);
QJL_API int qjl_scores(const qjl_key_cache_t* cache, int64_t n, const void* q, int q_dtype, int G,
               const qjl_sketch_t* sketch, float* logits, void* workspace,
               size_t workspace_bytes, unsigned flags, void* stream);

/* packed_sign_dot_batch: out f64 [G][n] = 2 * sum_{set bits of row i} values[g] - sum(values[g])
 * for n packed rows of m bits (row_bytes apart, m % 32 == 0), values f64 [G][m]. */
QJL_API int qjl_sign_dot_batch(const uint8_t* bits, int64_t n, int m, int64_t row_bytes,
                               const double* values, int G, double* out, void* stream);

/* Row softmax in fp64 of logits * inv_temperature: [rows][n] -> weights f64. */
QJL_API int qjl_softmax_f64(const float* logits, int64_t rows, int64_t n, double inv_temperature,
                    double* weights, void* stream);

/* K2+K3 fused decode: out [units][G][d] f32 = softmax(logits * inv_temperature) @ V.
 * lse (optional, may be NULL): [units][G] f32 log-sum-exp of the scaled logits.
 * logits (optional, may be NULL): [units][G][n] f32, the scaled logits the softmax consumed
 * (what `estimate_scores` normalizes, kvcache.py:331-337).
 * P2T caches (tile-major records) run the tensor-core decode (G <= 4); U8 caches run the
 * generic decode.  flags: QJL_DECODE_*. */
QJL_API size_t qjl_decode_workspace(const qjl_key_cache_t* cache, const qjl_value_cache_t* values,
                            int64_t n, int G);
QJL_API int qjl_decode(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int64_t n,
               const void* q, int q_dtype, int G, const qjl_sketch_t* sketch,
               float inv_temperature, float* out, float* lse, float* logits, void* workspace,
               size_t workspace_bytes, unsigned flags, void* stream);

/* One generation step (Algorithm 1 of the paper): append the new token of
 * every unit -- k_new / v_new [units][d] in q_dtype -- at row n (K1 + value quantizer
 * arithmetic, fused into the query-sketch kernel), then decode over rows [0, n + 1).
 * channels [units][h] is the outlier profile.  P2T caches only (QJL_ERR_UNSUPPORTED
 * otherwise: callers then append and decode separately).  Workspace:
 * qjl_decode_workspace(cache, values, n + 1, G). */
QJL_API int qjl_decode_step(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int64_t n,
                            const void* q, int q_dtype, int G, const qjl_sketch_t* sketch,
                            const int32_t* channels, int h, const void* k_new, const void* v_new,
                            float inv_temperature, float* out, float* lse, float* logits, void* workspace,
                            size_t workspace_bytes, unsigned flags, void* stream);

/* Benchmark hook: time the dominant kernel of the P2T decode as it runs in a decode loop.
 * Runs the query-sketch kernel once, then `reps` back-to-back decode kernels chained with
 * programmatic dependent launch (each one re-reads the whole cache and rewrites out/lse),
 * bracketed by CUDA events on `stream`; *ms = mean kernel time.  Same arguments as
 * qjl_decode otherwise (flags: QJL_DECODE_DETERMINISTIC selects the schedule timed). */
QJL_API int qjl_bench_decode_kernel(const qjl_key_cache_t* cache, const qjl_value_cache_t* values,
                                    int64_t n, const void* q, int q_dtype, int G,
                                    const qjl_sketch_t* sketch, float inv_temperature, float* out,
                                    float* lse, void* workspace, size_t workspace_bytes, unsigned flags,
                                    int reps, float* ms, void* stream);

/* Benchmark timing hook: while enabled, every qjl_quantize_keys call is bracketed by CUDA
 * events recorded on its launch stream.  qjl_timing_read synchronizes on them and returns the
 * summed kernel time (ms) and the number of bracketed launches (reset != 0 clears the record). */
QJL_API int qjl_timing_enable(int on);
QJL_API int qjl_timing_read(double* total_ms, int* launches, int reset);

/* Value quantizer: v [units][n][d] -> value cache rows [row_offset, row_offset + n). */
QJL_API int qjl_quantize_values(const void* v, int dtype, int64_t n, int64_t unit_stride,
                        const qjl_value_cache_t* values, int64_t row_offset, void* stream);

/* orthogonalize (sketch.py:82-103) for a batch of sketches: gaussian / out [batch][m][d]
 * fp64.  Rows are taken in blocks of <= d; each block is replaced by the sign-corrected
 * thin QR factor of its transpose (positive diag R), rows rescaled to norm sqrt(d).
 * Used by the statistical suites.  d * min(m, d) * 8 <= 200 KB. */
QJL_API int qjl_orthogonalize(const double* gaussian, int batch, int m, int d, double* out,
                              void* stream);

/* QJLC cache files (write_cache / read_cache, pkg/src/qjl/kvcache.py:368-520).
 * One record per token, little-endian, in append order (kvcache.py:430-436, :472):
 *   [inlier sign words 8*ceil(m_in_file/64) B][inlier norm f16]
 *   [outlier sign words 8*ceil(m_out_file/64) B][outlier norm f16]
 *   [d value codes, 1 B each][zero f32][scale f32]
 * m_in_file / m_out_file are the logical widths of the file header; the key cache's
 * (32-bit padded) widths must fit inside the file's words, and bits past the logical
 * width are written / loaded as zero.  An empty side (width 0) writes a 0.0 norm
 * (EMPTY_KEY, estimator.py:95).  Rows-layout caches only (tile_stride == 0); the value cache
 * must use the U8 layout with group == d
 * (the only value format the file holds).  records: [units][unit_stride] bytes, unit u's
 * n records at u * unit_stride.  The header, outlier channels and magnitudes of each file
 * are host data (paper_2406_03482_b200/qjlc.py). */
QJL_API int64_t qjl_qjlc_record_bytes(int d, int m_in_file, int m_out_file);
/* Rows [row_offset, row_offset + n) of every unit -> records.  n == 0 -> QJL_ERR_EMPTY
 * ("refusing to serialize an empty cache", kvcache.py:407-408). */
QJL_API int qjl_qjlc_export(const qjl_key_cache_t* keys, const qjl_value_cache_t* values,
                            int m_in_file, int m_out_file, int64_t row_offset, int64_t n,
                            uint8_t* records, int64_t unit_stride, void* stream);
/* records -> rows [row_offset, row_offset + n) of every unit; values may be NULL (keys only). */
QJL_API int qjl_qjlc_import(const uint8_t* records, int64_t unit_stride, int64_t n, int m_in_file,
                            int m_out_file, const qjl_key_cache_t* keys,
                            const qjl_value_cache_t* values, int64_t row_offset, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QJL_B200_H */
