// C ABI entry points (include/qjl_b200.h): argument validation mirroring the
// reference's ValueError conditions, then stream-ordered launches.
#include <stdarg.h>
#include <stdio.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace qjl {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: CUDA error %d (%s)", what, (int)e, cudaGetErrorString(e));
  return QJL_ERR_CUDA;
}

int device_sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = sms;
  return sms;
}

static std::mutex g_tmu;
static bool g_timing = false;
static std::vector<cudaEvent_t> g_ev;   // pairs (start, stop)
static size_t g_ev_used = 0;

static cudaEvent_t next_event() {
  if (g_ev_used == g_ev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_ev.push_back(e);
  }
  return g_ev[g_ev_used++];
}

void timing_begin(cudaStream_t st) {
  if (!g_timing) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  if (g_ev_used % 2) return;  // unbalanced: ignore
  cudaEventRecord(next_event(), st);
}

bool timing_enabled() { return g_timing; }

void timing_end(cudaStream_t st) {
  if (!g_timing) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  if (g_ev_used % 2 == 0) return;
  cudaEventRecord(next_event(), st);
}

static bool valid_dtype(int dt) { return dt == QJL_F32 || dt == QJL_F16 || dt == QJL_BF16 || dt == QJL_F64; }

static int check_key_cache(const qjl_key_cache_t* kc) {
  QJL_CHECK_ARG(kc != nullptr, "key cache descriptor is NULL");
  QJL_CHECK_ARG(kc->units >= 1, "units must be >= 1 (got %d)", kc->units);
  QJL_CHECK_ARG(kc->d >= 1 && kc->d <= 1024, "head dim d must be in [1, 1024] (got %d)", kc->d);
  QJL_CHECK_ARG(kc->m_in >= 0 && kc->m_out >= 0 && kc->m_in + kc->m_out >= 1,
                "sketch sizes must be non-negative with m_in + m_out >= 1");
  if (kc->m_in % 32 || kc->m_out % 32) {
    set_error("device path packs sketch bits in 32-bit words: m_in=%d, m_out=%d must be multiples of 32",
              kc->m_in, kc->m_out);
    return QJL_ERR_UNSUPPORTED;
  }
  if (kc->m_in + kc->m_out > 1024) {
    set_error("m_in + m_out = %d exceeds 1024", kc->m_in + kc->m_out);
    return QJL_ERR_UNSUPPORTED;
  }
  QJL_CHECK_ARG(kc->m_in == 0 || (kc->bits_in && kc->norm_in), "bits_in/norm_in must be set when m_in > 0");
  QJL_CHECK_ARG(kc->m_out == 0 || (kc->bits_out && kc->norm_out), "bits_out/norm_out must be set when m_out > 0");
  QJL_CHECK_ARG(kc->capacity >= 0, "capacity must be >= 0");
  QJL_CHECK_ARG(kc->tile_stride >= 0, "tile stride must be >= 0");
  if (kc->tile_stride > 0) {
    // tile-major caches are canonical records (keys only, or keys + P2T values)
    QJL_CHECK_ARG(kc->capacity % 128 == 0, "tile-major caches hold whole 128-row tiles (capacity %lld)",
                  (long long)kc->capacity);
    const TileRecord rk = tile_record(kc->d, kc->m_in, kc->m_out, false);
    const TileRecord rv = tile_record(kc->d, kc->m_in, kc->m_out, true);
    QJL_CHECK_ARG(kc->tile_stride == rk.bytes || (kc->d == 128 && kc->tile_stride == rv.bytes),
                  "tile stride %lld is not a record size of this shape (%lld keys only, %lld with values)",
                  (long long)kc->tile_stride, (long long)rk.bytes, (long long)rv.bytes);
    const uint8_t* b = kc->bits_in;
    QJL_CHECK_ARG((const uint8_t*)kc->norm_in == b + rk.off[QJL_REC_NORM_IN] &&
                      (kc->m_out == 0 || (kc->bits_out == b + rk.off[QJL_REC_BITS_OUT] &&
                                          (const uint8_t*)kc->norm_out == b + rk.off[QJL_REC_NORM_OUT])),
                  "key arrays of a tile-major cache must sit at their record offsets (qjl_tile_record)");
  }
  return QJL_OK;
}

// value caches: P2T lives in the key cache's tile records; U8 is rows layout
static int check_value_cache(const qjl_value_cache_t* vc, int d, int units) {
  QJL_CHECK_ARG(vc != nullptr, "value cache descriptor is NULL");
  QJL_CHECK_ARG(vc->codes && vc->zero && vc->scale, "value cache pointers must be set");
  QJL_CHECK_ARG(vc->d == d, "value dim %d != key dim %d", vc->d, d);
  QJL_CHECK_ARG(vc->units == units, "value units %d != key units %d", vc->units, units);
  QJL_CHECK_ARG(vc->bits >= 1 && vc->bits <= 8, "value bit width must be in [1, 8], got %d", vc->bits);
  QJL_CHECK_ARG(vc->group >= 1 && d % vc->group == 0, "value group %d must divide d=%d", vc->group, d);
  if (vc->layout == QJL_VLAYOUT_P2T) {
    if (!(d == 128 && vc->bits == 2 && vc->group == 32)) {
      set_error("the P2T value layout is 2-bit, group 32, d = 128 (got d=%d bits=%d group=%d)", d, vc->bits,
                vc->group);
      return QJL_ERR_UNSUPPORTED;
    }
    QJL_CHECK_ARG(vc->tile_stride > 0 && vc->capacity % 128 == 0,
                  "P2T values live in tile-major records (tile_stride > 0, capacity %% 128 == 0)");
  } else {
    QJL_CHECK_ARG(vc->layout == QJL_VLAYOUT_U8, "unknown value layout %d", vc->layout);
    QJL_CHECK_ARG(vc->tile_stride == 0, "U8 value caches use the rows layout (tile_stride 0)");
  }
  if (d > 128) {
    set_error("decode supports head dim <= 128 (got %d)", d);
    return QJL_ERR_UNSUPPORTED;
  }
  return QJL_OK;
}

static int check_sketch(const qjl_sketch_t* sk) {
  QJL_CHECK_ARG(sk != nullptr && sk->s_full != nullptr, "sketch is NULL");
  QJL_CHECK_ARG(valid_dtype(sk->dtype), "bad sketch dtype %d", sk->dtype);
  QJL_CHECK_ARG(sk->unit_stride >= 0, "sketch unit stride must be >= 0");
  return QJL_OK;
}

}  // namespace qjl

using namespace qjl;

#define QJL_TRY(expr)              \
  do {                             \
    int rc_ = (expr);              \
    if (rc_ != QJL_OK) return rc_; \
  } while (0)

extern "C" {

int qjl_abi_version(void) { return QJL_ABI_VERSION; }

const char* qjl_status_string(int status) {
  switch (status) {
    case QJL_OK: return "ok";
    case QJL_ERR_ARG: return "invalid argument";
    case QJL_ERR_UNSUPPORTED: return "unsupported configuration";
    case QJL_ERR_CUDA: return "CUDA error";
    case QJL_ERR_WORKSPACE: return "workspace too small";
    case QJL_ERR_EMPTY: return "cache is empty";
  }
  return "unknown status";
}

const char* qjl_last_error(void) { return g_err; }

int qjl_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing = on != 0;
  return QJL_OK;
}

int qjl_timing_read(double* total_ms, int* launches, int reset) {
  std::lock_guard<std::mutex> lk(g_tmu);
  double tot = 0.0;
  int cnt = 0;
  for (size_t i = 0; i + 1 < g_ev_used; i += 2) {
    cudaError_t e = cudaEventSynchronize(g_ev[i + 1]);
    if (e != cudaSuccess) return cuda_status(e, "timing_read");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_ev[i], g_ev[i + 1]);
    tot += ms;
    ++cnt;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = cnt;
  if (reset) g_ev_used = 0;
  return QJL_OK;
}

int qjl_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (sm_count) *sm_count = device_sm_count();
  if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  return QJL_OK;
}

size_t qjl_detect_workspace(int units, int64_t n0, int d) {
  if (units < 1 || n0 < 1 || d < 1) return 0;
  return detect_workspace(units, n0, d);
}

int qjl_detect_outliers(const void* keys, int dtype, int units, int64_t n0, int d,
                        int64_t unit_stride, int h, int32_t* channels, double* magnitudes,
                        void* ws, size_t ws_bytes, void* stream) {
  QJL_CHECK_ARG(keys != nullptr, "keys is NULL");
  QJL_CHECK_ARG(valid_dtype(dtype), "bad key dtype %d", dtype);
  QJL_CHECK_ARG(units >= 1, "units must be >= 1");
  QJL_CHECK_ARG(n0 >= 1, "prompt keys must be a non-empty n x d matrix");
  QJL_CHECK_ARG(d >= 1 && d <= 1024, "d must be in [1, 1024]");
  QJL_CHECK_ARG(h >= 0 && h <= d, "outlier count must be in [0, %d], got %d", d, h);
  QJL_CHECK_ARG(h == 0 || channels != nullptr, "channels output is NULL");
  QJL_CHECK_ARG(unit_stride >= n0 * d, "unit stride %lld < n0*d", (long long)unit_stride);
  return launch_detect_outliers(keys, dtype, units, n0, d, unit_stride, h, channels, magnitudes, ws,
                                ws_bytes, (cudaStream_t)stream);
}

int qjl_build_sketch(const double* s_in, const double* s_out, int m_in, int m_out, int d, int h,
                     const int32_t* channels, int units, int dtype, void* s_full, void* stream) {
  QJL_CHECK_ARG(s_full != nullptr, "s_full is NULL");
  QJL_CHECK_ARG(valid_dtype(dtype), "bad sketch dtype %d", dtype);
  QJL_CHECK_ARG(d >= 1 && d <= 1024 && h >= 0 && h <= d, "bad d/h");
  QJL_CHECK_ARG(units >= 1, "units must be >= 1");
  QJL_CHECK_ARG((s_in == nullptr) == (m_in == 0) && (m_in == 0) == (d - h == 0),
                "inlier sketch must be present exactly when d - h > 0");
  QJL_CHECK_ARG((s_out == nullptr) == (m_out == 0) && (m_out == 0) == (h == 0),
                "outlier sketch must be present exactly when h > 0");
  QJL_CHECK_ARG(h == 0 || channels != nullptr, "channels is NULL");
  if (h > 0 && d - h > 0 && (int64_t)m_out * (d - h) < (int64_t)m_in * h) {
    set_error("outlier bit rate below inlier bit rate: m_out/h = %d/%d < m_in/(d-h) = %d/%d", m_out, h,
              m_in, d - h);
    return QJL_ERR_ARG;  // kvcache.py:219-226
  }
  return launch_build_sketch(s_in, s_out, m_in, m_out, d, h, channels, units, dtype, s_full,
                             (cudaStream_t)stream);
}

int qjl_prefill_profile(const void* keys, int dtype, int units, int64_t n0, int d, int64_t unit_stride, int h,
                        const void* s_in, const void* s_out, int m_in, int m_out, int sketch_dtype,
                        int32_t* channels, double* magnitudes, void* s_full, void* ws, size_t ws_bytes,
                        void* stream) {
  QJL_CHECK_ARG(keys != nullptr, "keys is NULL");
  QJL_CHECK_ARG(valid_dtype(dtype), "bad key dtype %d", dtype);
  QJL_CHECK_ARG(units >= 1, "units must be >= 1");
  QJL_CHECK_ARG(n0 >= 1, "prompt keys must be a non-empty n x d matrix");
  QJL_CHECK_ARG(d >= 1 && d <= 1024, "d must be in [1, 1024]");
  QJL_CHECK_ARG(h >= 0 && h <= d, "outlier count must be in [0, %d], got %d", d, h);
  QJL_CHECK_ARG(h == 0 || channels != nullptr, "channels output is NULL");
  QJL_CHECK_ARG(unit_stride >= n0 * d, "unit stride %lld < n0*d", (long long)unit_stride);
  QJL_CHECK_ARG(s_full != nullptr, "s_full is NULL");
  QJL_CHECK_ARG(valid_dtype(sketch_dtype), "bad sketch dtype %d", sketch_dtype);
  QJL_CHECK_ARG((s_in == nullptr) == (m_in == 0) && (m_in == 0) == (d - h == 0),
                "inlier sketch must be present exactly when d - h > 0");
  QJL_CHECK_ARG((s_out == nullptr) == (m_out == 0) && (m_out == 0) == (h == 0),
                "outlier sketch must be present exactly when h > 0");
  if (h > 0 && d - h > 0 && (int64_t)m_out * (d - h) < (int64_t)m_in * h) {
    set_error("outlier bit rate below inlier bit rate: m_out/h = %d/%d < m_in/(d-h) = %d/%d", m_out, h,
              m_in, d - h);
    return QJL_ERR_ARG;  // kvcache.py:219-226
  }
  return launch_prefill_profile(keys, dtype, units, n0, d, unit_stride, h, s_in, s_out, m_in, m_out,
                                sketch_dtype, channels, magnitudes, s_full, ws, ws_bytes, (cudaStream_t)stream);
}

int qjl_quantize_keys(const void* keys, int dtype, int64_t n, int64_t key_unit_stride,
                      const qjl_sketch_t* sketch, const int32_t* channels, int h,
                      const qjl_key_cache_t* cache, int64_t row_offset, void* stream) {
  QJL_TRY(check_key_cache(cache));
  QJL_TRY(check_sketch(sketch));
  QJL_CHECK_ARG(keys != nullptr, "keys is NULL");
  QJL_CHECK_ARG(valid_dtype(dtype), "bad key dtype %d", dtype);
  QJL_CHECK_ARG(n >= 0 && row_offset >= 0 && row_offset + n <= cache->capacity,
                "rows [%lld, %lld) exceed capacity %lld", (long long)row_offset,
                (long long)(row_offset + n), (long long)cache->capacity);
  QJL_CHECK_ARG(h >= 0 && h <= cache->d && (h == 0 || channels), "bad outlier channels");
  QJL_CHECK_ARG((h > 0) == (cache->m_out > 0), "outlier sketch must be present exactly when h > 0");
  QJL_CHECK_ARG(key_unit_stride == 0 || key_unit_stride >= n * cache->d, "key unit stride too small");
  if (n == 0) return QJL_OK;
  int rc = launch_quantize_keys_tc(keys, dtype, n, key_unit_stride, *sketch, channels, h, *cache,
                                   row_offset, (cudaStream_t)stream);
  if (rc != QJL_ERR_UNSUPPORTED) return rc;
  return launch_quantize_keys_simt(keys, dtype, n, key_unit_stride, *sketch, channels, h, *cache,
                                   row_offset, (cudaStream_t)stream);
}

int qjl_sketch_query(const void* q, int q_dtype, int units, int G, int d, const qjl_sketch_t* sketch,
                     int m_total, int sq_dtype, void* sq, void* stream) {
  QJL_TRY(check_sketch(sketch));
  QJL_CHECK_ARG(q && sq, "NULL pointer");
  QJL_CHECK_ARG(valid_dtype(q_dtype), "bad query dtype %d", q_dtype);
  QJL_CHECK_ARG(sq_dtype == QJL_F32 || sq_dtype == QJL_F64, "sketched queries are f32 or f64");
  QJL_CHECK_ARG(units >= 1 && G >= 1 && d >= 1 && d <= 1024 && m_total >= 1, "bad shape");
  if (sq_dtype == QJL_F64)
    return launch_sketch_query_f64(q, q_dtype, units, G, d, *sketch, m_total, (double*)sq, (cudaStream_t)stream);
  return launch_sketch_query(q, q_dtype, units, G, d, *sketch, m_total, m_total, (float*)sq, nullptr,
                             (cudaStream_t)stream);
}

size_t qjl_scores_workspace(int units, int G, int m_total) {
  // generic: Sq + side sums; tensor-core: B images + constants + counters (<= this bound)
  const size_t a = (size_t)units * G * (m_total + 2) * sizeof(float);
  const size_t b = (size_t)units * (5 * 2048 + 64 + 8) + 1024;
  return a > b ? a : b;
}

int qjl_scores(const qjl_key_cache_t* cache, int64_t n, const void* q, int q_dtype, int G,
               const qjl_sketch_t* sketch, float* logits, void* workspace, size_t workspace_bytes,
               unsigned flags, void* stream) {
  QJL_TRY(check_key_cache(cache));
  QJL_CHECK_ARG((flags & ~(unsigned)QJL_DECODE_CHAINED) == 0, "qjl_scores flags: QJL_DECODE_CHAINED only (got %u)", flags);
  QJL_TRY(check_sketch(sketch));
  QJL_CHECK_ARG(q && logits, "NULL pointer");
  QJL_CHECK_ARG(valid_dtype(q_dtype), "bad query dtype %d", q_dtype);
  QJL_CHECK_ARG(G >= 1, "G must be >= 1");
  if (n <= 0) {
    set_error("cache is empty; append at least one key first");
    return QJL_ERR_EMPTY;
  }
  QJL_CHECK_ARG(n <= cache->capacity, "n exceeds capacity");
  const int m_total = cache->m_in + cache->m_out;
  if (workspace_bytes < qjl_scores_workspace(cache->units, G, m_total) || !workspace) {
    set_error("scores workspace needs %zu bytes", qjl_scores_workspace(cache->units, G, m_total));
    return QJL_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (cache->tile_stride > 0 && tile_path_supported(*cache, nullptr, G))
    return launch_scores_tile(*cache, n, q, q_dtype, G, *sketch, logits, workspace, workspace_bytes, flags, st);
  float* sq = (float*)workspace;
  float* sums = sq + (size_t)cache->units * G * m_total;
  QJL_TRY(launch_sketch_query(q, q_dtype, cache->units, G, cache->d, *sketch, cache->m_in, m_total,
                              sq, sums, st));
  return launch_scores_simt(*cache, n, G, sq, sums, logits, st);
}

int qjl_sign_dot_batch(const uint8_t* bits, int64_t n, int m, int64_t row_bytes,
                       const double* values, int G, double* out, void* stream) {
  QJL_CHECK_ARG(bits && values && out, "NULL pointer");
  QJL_CHECK_ARG(n >= 1 && G >= 1 && m >= 1, "bad shape");
  if (m % 32 || row_bytes % 4 || row_bytes * 8 < m) {
    set_error("sign_dot_batch needs m %% 32 == 0 and 4-byte aligned rows (m=%d, row_bytes=%lld)", m,
              (long long)row_bytes);
    return QJL_ERR_UNSUPPORTED;
  }
  if ((size_t)G * (m + 1) * 8 > 200 * 1024) {
    set_error("sign_dot_batch: G*m too large");
    return QJL_ERR_UNSUPPORTED;
  }
  return launch_sign_dot_batch(bits, n, m, row_bytes, values, G, out, (cudaStream_t)stream);
}

int qjl_softmax_f64(const float* logits, int64_t rows, int64_t n, double inv_temperature,
                    double* weights, void* stream) {
  QJL_CHECK_ARG(logits && weights, "NULL pointer");
  QJL_CHECK_ARG(rows >= 1 && n >= 1, "bad shape");
  QJL_CHECK_ARG(inv_temperature > 0, "temperature must be positive");
  return launch_softmax_f64(logits, rows, n, inv_temperature, weights, (cudaStream_t)stream);
}

size_t qjl_decode_workspace(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int64_t n,
                            int G) {
  if (!cache || !values || n <= 0 || G <= 0) return 0;
  if (values->layout == QJL_VLAYOUT_P2T) return decode_tile_workspace(*cache, n, G, false);
  return decode_simt_workspace(cache->units, n, G, values->d, cache->m_in + cache->m_out);
}

// shared argument checks of the decode entry points; *tile = the tensor-core path applies
static int check_decode(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int64_t n, const void* q,
                        int q_dtype, int G, const qjl_sketch_t* sketch, float inv_temperature, const float* out) {
  QJL_TRY(check_key_cache(cache));
  QJL_TRY(check_value_cache(values, cache->d, cache->units));
  QJL_TRY(check_sketch(sketch));
  QJL_CHECK_ARG(q && out, "NULL pointer");
  QJL_CHECK_ARG(valid_dtype(q_dtype), "bad query dtype %d", q_dtype);
  QJL_CHECK_ARG(G >= 1, "G must be >= 1");
  QJL_CHECK_ARG(inv_temperature > 0.f, "temperature must be positive");
  if (n <= 0) {
    set_error("cache is empty");
    return QJL_ERR_EMPTY;
  }
  QJL_CHECK_ARG(n <= cache->capacity && n <= values->capacity, "n exceeds capacity");
  if (values->layout == QJL_VLAYOUT_P2T) {
    if (!tile_path_supported(*cache, values, G)) {
      set_error("P2T decode runs on the tensor-core path: d = 128, G <= 4, m_in/32 in {8, 16}, m_out/32 in "
                "{0, 2, 4}, values in the keys' tile records (got d=%d G=%d m_in=%d m_out=%d)",
                cache->d, G, cache->m_in, cache->m_out);
      return QJL_ERR_UNSUPPORTED;
    }
  } else {
    QJL_CHECK_ARG(cache->tile_stride == 0, "U8 caches use the rows layout");
  }
  return QJL_OK;
}

int qjl_decode(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int64_t n, const void* q,
               int q_dtype, int G, const qjl_sketch_t* sketch, float inv_temperature, float* out,
               float* lse, float* logits, void* workspace, size_t workspace_bytes, unsigned flags, void* stream) {
  QJL_TRY(check_decode(cache, values, n, q, q_dtype, G, sketch, inv_temperature, out));
  const size_t need = qjl_decode_workspace(cache, values, n, G);
  if (!workspace || workspace_bytes < need) {
    set_error("decode workspace needs %zu bytes (got %zu)", need, workspace_bytes);
    return QJL_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (values->layout == QJL_VLAYOUT_P2T)
    return launch_decode_tile(*cache, n, q, q_dtype, G, *sketch, inv_temperature, out, lse, logits, workspace,
                              workspace_bytes, flags, st);
  const int m_total = cache->m_in + cache->m_out;
  float* sq = (float*)workspace;
  float* sums = sq + (size_t)cache->units * G * m_total;
  float* part = sums + (size_t)cache->units * G * 2;
  QJL_TRY(launch_sketch_query(q, q_dtype, cache->units, G, cache->d, *sketch, cache->m_in, m_total,
                              sq, sums, st));
  return launch_decode_simt(*cache, *values, n, G, sq, sums, inv_temperature, out, lse, logits, part, st);
}

int qjl_bench_decode_kernel(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int64_t n,
                            const void* q, int q_dtype, int G, const qjl_sketch_t* sketch, float inv_temperature,
                            float* out, float* lse, void* workspace, size_t workspace_bytes, unsigned flags,
                            int reps, float* ms, void* stream) {
  QJL_TRY(check_decode(cache, values, n, q, q_dtype, G, sketch, inv_temperature, out));
  QJL_CHECK_ARG(values->layout == QJL_VLAYOUT_P2T, "the benchmark hook times the tensor-core decode (P2T)");
  QJL_CHECK_ARG(reps >= 1 && ms, "reps must be >= 1 and ms set");
  const size_t need = qjl_decode_workspace(cache, values, n, G);
  if (!workspace || workspace_bytes < need) {
    set_error("decode workspace needs %zu bytes (got %zu)", need, workspace_bytes);
    return QJL_ERR_WORKSPACE;
  }
  return bench_decode_tile(*cache, n, q, q_dtype, G, *sketch, inv_temperature, out, lse, workspace,
                           workspace_bytes, flags, reps, ms, (cudaStream_t)stream);
}

int qjl_tensor_core_path(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int G) {
  QJL_TRY(check_key_cache(cache));
  if (values) QJL_TRY(check_value_cache(values, cache->d, cache->units));
  if (G < 1) return QJL_ERR_ARG;
  if (values && values->layout != QJL_VLAYOUT_P2T) return 0;
  if (!values && cache->tile_stride == 0) return 0;
  return tile_path_supported(*cache, values, G) ? 1 : 0;
}

int64_t qjl_tile_record(int d, int m_in, int m_out, int values, int64_t* offsets) {
  if (d < 1 || m_in < 0 || m_out < 0 || m_in % 32 || m_out % 32) return -1;
  if (values && d != 128) return -1;
  const TileRecord r = tile_record(d, m_in, m_out, values != 0);
  if (offsets)
    for (int i = 0; i < QJL_REC_FIELDS; ++i) offsets[i] = r.off[i];
  return r.bytes;
}

int qjl_quantize_values(const void* v, int dtype, int64_t n, int64_t unit_stride,
                        const qjl_value_cache_t* values, int64_t row_offset, void* stream) {
  QJL_CHECK_ARG(v != nullptr, "values is NULL");
  QJL_CHECK_ARG(valid_dtype(dtype), "bad value dtype %d", dtype);
  QJL_TRY(check_value_cache(values, values ? values->d : 0, values ? values->units : 0));
  QJL_CHECK_ARG(n >= 0 && row_offset >= 0 && row_offset + n <= values->capacity,
                "rows exceed value capacity");
  QJL_CHECK_ARG(unit_stride >= n * values->d, "value unit stride too small");
  if (n == 0) return QJL_OK;
  return launch_quantize_values(v, dtype, n, unit_stride, *values, row_offset, (cudaStream_t)stream);
}

int64_t qjl_qjlc_record_bytes(int d, int m_in, int m_out) {
  if (d < 1 || m_in < 0 || m_out < 0) return -1;
  return qjlc_record_bytes(d, m_in, m_out);
}

// shared checks of the QJLC record entry points: the key cache's padded widths must
// fit inside the file's whole u64 words, values in the reference's own format
static int check_qjlc(const qjl_key_cache_t* kc, const qjl_value_cache_t* vc, int mfi, int mfo,
                      int64_t row_offset, int64_t n, const void* records, int64_t ustride) {
  QJL_TRY(check_key_cache(kc));
  QJL_CHECK_ARG(records != nullptr, "records buffer is NULL");
  if (kc->tile_stride != 0) {
    set_error("QJLC records move rows-layout caches (the file's value format is U8)");
    return QJL_ERR_UNSUPPORTED;
  }
  QJL_CHECK_ARG(mfi >= 0 && mfi <= kc->m_in && (mfi > 0) == (kc->m_in > 0),
                "file inlier width %d does not fit the cache's %d bits", mfi, kc->m_in);
  QJL_CHECK_ARG(mfo >= 0 && mfo <= kc->m_out && (mfo > 0) == (kc->m_out > 0),
                "file outlier width %d does not fit the cache's %d bits", mfo, kc->m_out);
  if (kc->m_in > 64 * ((mfi + 63) / 64) || kc->m_out > 64 * ((mfo + 63) / 64)) {
    set_error("cache rows (%d/%d bits) are wider than the file's sign words (%d/%d bits)", kc->m_in,
              kc->m_out, mfi, mfo);
    return QJL_ERR_UNSUPPORTED;
  }
  QJL_CHECK_ARG(n >= 0 && row_offset >= 0 && row_offset + n <= kc->capacity, "rows exceed key capacity");
  QJL_CHECK_ARG(ustride >= n * qjlc_record_bytes(kc->d, mfi, mfo), "record unit stride too small");
  if (vc) {
    QJL_CHECK_ARG(vc->codes && vc->zero && vc->scale, "value cache pointers must be set");
    QJL_CHECK_ARG(vc->d == kc->d && vc->units == kc->units, "value cache shape does not match the keys");
    QJL_CHECK_ARG(vc->bits >= 1 && vc->bits <= 8, "value bit width must be in [1, 8], got %d", vc->bits);
    QJL_CHECK_ARG(row_offset + n <= vc->capacity, "rows exceed value capacity");
    if (vc->layout != QJL_VLAYOUT_U8 || vc->group != vc->d) {
      set_error("QJLC files hold one byte per code and one f32 zero/scale per token: the value cache "
                "must use the U8 layout with group == d (got layout %d, group %d)", vc->layout, vc->group);
      return QJL_ERR_UNSUPPORTED;
    }
  }
  return QJL_OK;
}

int qjl_qjlc_export(const qjl_key_cache_t* keys, const qjl_value_cache_t* values, int m_in_file,
                    int m_out_file, int64_t row_offset, int64_t n, uint8_t* records, int64_t unit_stride,
                    void* stream) {
  QJL_CHECK_ARG(values != nullptr, "a QJLC record carries value codes: values is NULL");
  QJL_TRY(check_qjlc(keys, values, m_in_file, m_out_file, row_offset, n, records, unit_stride));
  if (n == 0) {
    set_error("refusing to serialize an empty cache");
    return QJL_ERR_EMPTY;
  }
  return launch_qjlc_export(*keys, *values, m_in_file, m_out_file, row_offset, n, records, unit_stride,
                            (cudaStream_t)stream);
}

int qjl_qjlc_import(const uint8_t* records, int64_t unit_stride, int64_t n, int m_in_file, int m_out_file,
                    const qjl_key_cache_t* keys, const qjl_value_cache_t* values, int64_t row_offset,
                    void* stream) {
  QJL_TRY(check_qjlc(keys, values, m_in_file, m_out_file, row_offset, n, records, unit_stride));
  if (n == 0) return QJL_OK;
  return launch_qjlc_import(records, unit_stride, m_in_file, m_out_file, n, *keys, values, row_offset,
                            (cudaStream_t)stream);
}

int qjl_orthogonalize(const double* gaussian, int batch, int m, int d, double* out, void* stream) {
  QJL_CHECK_ARG(gaussian != nullptr && out != nullptr, "sketch pointers must be set");
  QJL_CHECK_ARG(batch >= 1, "batch must be >= 1");
  QJL_CHECK_ARG(m >= 1 && d >= 1, "sketch dimensions must be positive, got m=%d, d=%d", m, d);
  const int k = d < m ? d : m;
  if ((size_t)k * d * sizeof(double) > 200 * 1024 || k > 256) {
    set_error("orthogonalize stages a d x min(m, d) fp64 block in shared memory: d=%d is too large", d);
    return QJL_ERR_UNSUPPORTED;
  }
  return launch_orthogonalize(gaussian, batch, m, d, out, (cudaStream_t)stream);
}

int qjl_decode_step(const qjl_key_cache_t* cache, const qjl_value_cache_t* values, int64_t n, const void* q,
                    int q_dtype, int G, const qjl_sketch_t* sketch, const int32_t* channels, int h,
                    const void* k_new, const void* v_new, float inv_temperature, float* out, float* lse,
                    float* logits, void* workspace, size_t workspace_bytes, unsigned flags, void* stream) {
  QJL_TRY(check_key_cache(cache));
  QJL_TRY(check_value_cache(values, cache->d, cache->units));
  QJL_TRY(check_sketch(sketch));
  QJL_CHECK_ARG(q && out && k_new && v_new, "NULL pointer");
  QJL_CHECK_ARG(valid_dtype(q_dtype) && q_dtype != QJL_F64, "bad query dtype %d", q_dtype);
  QJL_CHECK_ARG(G >= 1, "G must be >= 1");
  QJL_CHECK_ARG(inv_temperature > 0.f, "temperature must be positive");
  QJL_CHECK_ARG(h >= 0 && h <= cache->d && (h == 0 || channels != nullptr), "bad outlier channels");
  QJL_CHECK_ARG((h > 0) == (cache->m_out > 0), "outlier sketch must be present exactly when h > 0");
  QJL_CHECK_ARG(n >= 0 && n + 1 <= cache->capacity && n + 1 <= values->capacity, "n + 1 exceeds capacity");
  if (values->layout != QJL_VLAYOUT_P2T || !tile_path_supported(*cache, values, G)) {
    set_error("decode_step runs on the tensor-core path (P2T tile records, supported sketch widths); "
              "append + decode instead");
    return QJL_ERR_UNSUPPORTED;
  }
  const size_t need = qjl_decode_workspace(cache, values, n + 1, G);
  if (!workspace || workspace_bytes < need) {
    set_error("decode workspace needs %zu bytes (got %zu)", need, workspace_bytes);
    return QJL_ERR_WORKSPACE;
  }
  return launch_decode_step_tile(*cache, *values, n, q, q_dtype, G, *sketch, channels, h, k_new, v_new,
                                 inv_temperature, out, lse, logits, workspace, workspace_bytes, flags,
                                 (cudaStream_t)stream);
}

}  // extern "C"
