// Prefill-side kernels: outlier profile, per-unit sketch build, generic (SIMT)
// key quantizer, value quantizer.  The tcgen05 tensor-core key quantizer for
// bf16/fp16 keys lives in k_quant_tc.cu; this file's quantizer handles every
// dtype with fp64 accumulation (fp32 keys, odd shapes, single-key shims).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace qjl {

// ---------------------------------------------------------------------------
// detect_outliers (kvcache.py:104-123): mean |k| per channel in fp64, top-h by
// (magnitude desc, index asc), emitted sorted ascending.  One CTA per unit:
// deterministic summation order, no atomics.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(1024) k_detect_outliers(const T* __restrict__ keys, int64_t n0,
                                                          int d, int64_t unit_stride, int h,
                                                          int32_t* __restrict__ channels,
                                                          double* __restrict__ magnitudes) {
  extern __shared__ double sm_mag[];  // [rows_par][d] partials, then [d] means
  const int u = blockIdx.x;
  const T* K = keys + (int64_t)u * unit_stride;
  const int rows_par = blockDim.x / d;  // blockDim.x is a multiple of d
  const int c = threadIdx.x % d, rp = threadIdx.x / d;
  double acc = 0.0;
  if (rp < rows_par) {
    for (int64_t r = rp; r < n0; r += rows_par) acc += fabs(to_f64(K[r * d + c]));
    sm_mag[rp * d + c] = acc;
  }
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < d)
    for (int i = 0; i < rows_par; ++i) s += sm_mag[i * d + threadIdx.x];
  __syncthreads();
  if (threadIdx.x < d) sm_mag[threadIdx.x] = s / (double)n0;
  __syncthreads();
  __shared__ int sel[1024];
  if (threadIdx.x < d) {
    const double mc = sm_mag[threadIdx.x];
    int rank = 0;
    for (int j = 0; j < d; ++j) {
      const double mj = sm_mag[j];
      rank += (mj > mc) || (mj == mc && j < (int)threadIdx.x);
    }
    sel[threadIdx.x] = rank < h;
    if (magnitudes) magnitudes[(int64_t)u * d + threadIdx.x] = mc;
  }
  __syncthreads();
  if (threadIdx.x < d && sel[threadIdx.x]) {
    int pos = 0;
    for (int j = 0; j < (int)threadIdx.x; ++j) pos += sel[j];
    channels[(int64_t)u * h + pos] = threadIdx.x;
  }
}

// Two-phase form for large prompts: (1) CTAs over (row block, unit) accumulate |k| per
// channel in fp64 over 256 rows with 16-byte loads; (2) one CTA per unit adds the
// block partials in a fixed order, then ranks.  |bf16| / |fp16| sums are exact in
// fp64 at these lengths, so the result does not depend on the split.
constexpr int kDetRows = 256;
constexpr int kDetBulkD = 128;     // 16-bit keys with d <= this: bulk-copied row blocks (<= 64 KB)

// |x| as fp64 without the F2F conversion pipe: for a normal 16-bit float the fp64 bit
// pattern is the magnitude bits shifted into place plus an exponent rebias (exact);
// zero and subnormal inputs (rare) take the converting path.
__device__ __forceinline__ double abs_f64_bits(__nv_bfloat16 x) {
  const uint32_t b = __bfloat16_as_ushort(x) & 0x7FFFu;
  if ((b & 0x7F80u) == 0u) return fabs((double)__bfloat162float(x));
  return __hiloint2double((int)((b << 13) + ((1023u - 127u) << 20)), 0);
}
__device__ __forceinline__ double abs_f64_bits(__half x) {
  const uint32_t b = __half_as_ushort(x) & 0x7FFFu;
  if ((b & 0x7C00u) == 0u) return fabs((double)__half2float(x));
  return __hiloint2double((int)((b << 10) + ((1023u - 15u) << 20)), 0);
}
__device__ __forceinline__ double abs_f64_bits(float x) { return fabs((double)x); }
__device__ __forceinline__ double abs_f64_bits(double x) { return fabs(x); }

// |x| of the 8 16-bit floats of one 16-byte vector, added to acc as fp64 values scaled by
// 2^-kDetShift: the magnitude bits are shifted into the high word of an fp64 whose low word
// is 0 and NO exponent rebias is added.  A normal 1.M x 2^(E - bias16) becomes
// 1.M x 2^(E - 1023), a subnormal 0.M x 2^(1 - bias16) becomes the fp64 subnormal
// 0.M x 2^-1022, and zero stays zero: every input, subnormals included, lands on the same
// power-of-two scaling, exactly, with two integer ops and no conversion unit.  The sums
// equal the unscaled ones times 2^-kDetShift bit for bit (the scaled values are exact, and
// sums that fall below 2^-1022 are exact multiples of 2^-1074); callers multiply back.
template <typename T> struct DetScaled;
template <> struct DetScaled<__nv_bfloat16> {
  static constexpr int kShift = 1023 - 127;                      // 2^-896
  static __device__ __forceinline__ int lo(uint32_t w) { return (int)((w << 13) & 0x0FFFE000u); }
  static __device__ __forceinline__ int hi(uint32_t w) { return (int)((w >> 3) & 0x0FFFE000u); }
};
template <> struct DetScaled<__half> {
  static constexpr int kShift = 1023 - 15;                       // 2^-1008
  static __device__ __forceinline__ int lo(uint32_t w) { return (int)((w << 10) & 0x01FFFC00u); }
  static __device__ __forceinline__ int hi(uint32_t w) { return (int)((w >> 6) & 0x01FFFC00u); }
};
template <typename T>
__device__ __forceinline__ void add_abs_scaled(const uint4& raw, double* acc) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    acc[2 * k] += __hiloint2double(DetScaled<T>::lo(w[k]), 0);
    acc[2 * k + 1] += __hiloint2double(DetScaled<T>::hi(w[k]), 0);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_detect_partial(const T* __restrict__ keys, int64_t n0, int d,
                                                        int64_t unit_stride, double* __restrict__ part) {
  constexpr int EPV = 16 / (int)sizeof(T);
  const bool bulk = sizeof(T) == 2 && d <= kDetBulkD;   // the block's rows arrive by one bulk copy
  extern __shared__ __align__(16) double sm_part[];   // [rows_par][d]; 16-bit keys: first the rows
  __shared__ __align__(8) uint64_t bar;
  // the finish kernel may launch now: it stages its sketch rows while this grid drains, and
  // waits (griddepcontrol.wait) for the partials
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int u = blockIdx.y, blk = blockIdx.x;
  const int tpr = d / EPV;                        // threads per row
  const int rows_par = blockDim.x / tpr;
  const int cg = threadIdx.x % tpr, rs = threadIdx.x / tpr;
  const T* K = keys + (int64_t)u * unit_stride;
  const int64_t r0 = (int64_t)blk * kDetRows, r_end = min(r0 + kDetRows, n0);
  double acc[EPV];
#pragma unroll
  for (int e = 0; e < EPV; ++e) acc[e] = 0.0;
  if (bulk) {
    // the 256 rows (contiguous, 64 KB at d = 128) land in shared memory with no registers
    // held per load: 3 CTAs per SM keep ~190 KB in flight, which a register-staged loop
    // (the per-element subnormal test serialises its loads) does not reach
    const uint32_t b = ptx::smem_u32(&bar), dst = ptx::smem_u32(sm_part);
    if (threadIdx.x == 0) {
      ptx::mbar_init(b, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)((r_end - r0) * d * (int64_t)sizeof(T));
      ptx::mbar_expect_tx(b, bytes);
      ptx::bulk_g2s(dst, K + r0 * d, bytes, b);
    }
    ptx::mbar_wait(b, 0);
    const T* rows = reinterpret_cast<const T*>(sm_part);
    if (rs < rows_par) {
      for (int64_t r = rs; r < r_end - r0; r += rows_par) {
        const uint4 raw = *reinterpret_cast<const uint4*>(rows + r * d + cg * EPV);
        if constexpr (sizeof(T) == 2) add_abs_scaled<T>(raw, acc);
      }
    }
    if constexpr (sizeof(T) == 2) {
      const double unscale = ldexp(1.0, DetScaled<T>::kShift);   // exact
#pragma unroll
      for (int e = 0; e < EPV; ++e) acc[e] *= unscale;
    }
    __syncthreads();                              // the rows are consumed; sm_part is reused
  } else if (rs < rows_par) {
#pragma unroll 4
    for (int64_t r = r0 + rs; r < r_end; r += rows_par) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(K + r * d + cg * EPV));
      const T* v = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int e = 0; e < EPV; ++e) acc[e] += abs_f64_bits(v[e]);
    }
  }
  if (rs < rows_par) {
#pragma unroll
    for (int e = 0; e < EPV; ++e) sm_part[rs * d + cg * EPV + e] = acc[e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double t = 0.0;
    for (int i = 0; i < rows_par; ++i) t += sm_part[i * d + c];
    part[((int64_t)u * gridDim.x + blk) * d + c] = t;
  }
}

// dynamic shared memory of k_detect_partial: the per-row-slot partials, and for 16-bit keys
// the block's rows
static size_t det_partial_smem(int d, size_t es, int rows_par) {
  const size_t a = (size_t)rows_par * d * sizeof(double);
  const size_t b = es == 2 && d <= kDetBulkD ? (size_t)kDetRows * d * es : 0;
  return a > b ? a : b;
}

// Channel means from the block partials with all 1024 threads: P = 1024 / d chunks of
// blocks per channel, each summed in block order with 8 loads in flight, then the P chunk
// sums added in chunk order -- a fixed order, shared by every kernel that finishes the
// detection, so they agree bit for bit.  mag: [d] means out; red: [1024] scratch.
__device__ __forceinline__ void channel_means(const double* __restrict__ part, int u, int nblk, int d,
                                              int64_t n0, double* mag, double* red) {
  const int P = max(1, (int)blockDim.x / d);
  const int c = threadIdx.x % d, k = threadIdx.x / d;
  if (k < P) {
    const int b0 = (int)((int64_t)k * nblk / P), b1 = (int)((int64_t)(k + 1) * nblk / P);
    const double* p = part + (int64_t)u * nblk * d + c;
    double s = 0.0;
    int b = b0;
    for (; b + 8 <= b1; b += 8) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(p + (int64_t)(b + j) * d);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[j];
    }
    for (; b < b1; ++b) s += __ldcg(p + (int64_t)b * d);
    red[k * d + c] = s;
  }
  __syncthreads();
  if (threadIdx.x < d) {
    double s = 0.0;
    for (int j = 0; j < P; ++j) s += red[j * d + threadIdx.x];
    mag[threadIdx.x] = s / (double)n0;
  }
  __syncthreads();
}

// rank of channel c by (magnitude desc, index asc), counted by P threads per channel
__device__ __forceinline__ void channel_ranks(const double* mag, int d, int* rank) {
  const int P = max(1, (int)blockDim.x / d);
  const int c = threadIdx.x % d, k = threadIdx.x / d;
  if (threadIdx.x < d) rank[threadIdx.x] = 0;
  __syncthreads();
  if (k < P) {
    const double mc = mag[c];
    const int j0 = (int)((int64_t)k * d / P), j1 = (int)((int64_t)(k + 1) * d / P);
    int r = 0;
    for (int j = j0; j < j1; ++j) {
      const double mj = mag[j];
      r += (mj > mc) || (mj == mc && j < c);
    }
    if (r) atomicAdd(&rank[c], r);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024) k_detect_finish(const double* __restrict__ part, int nblk, int64_t n0,
                                                        int d, int h, int32_t* __restrict__ channels,
                                                        double* __restrict__ magnitudes) {
  __shared__ double mag[1024];
  __shared__ double red[1024];
  __shared__ int rank[1024];
  __shared__ int sel[1024];
  const int u = blockIdx.x;
  channel_means(part, u, nblk, d, n0, mag, red);
  channel_ranks(mag, d, rank);
  if (threadIdx.x < d) {
    sel[threadIdx.x] = rank[threadIdx.x] < h;
    if (magnitudes) magnitudes[(int64_t)u * d + threadIdx.x] = mag[threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x < d && sel[threadIdx.x]) {
    int pos = 0;
    for (int j = 0; j < (int)threadIdx.x; ++j) pos += sel[j];
    channels[(int64_t)u * h + pos] = threadIdx.x;
  }
}

// Workspace of the two-phase detection: fp64 per-block channel partials.
size_t detect_workspace(int units, int64_t n0, int d) {
  if (n0 < 2 * kDetRows || d > 1024) return 0;
  const int64_t nblk = (n0 + kDetRows - 1) / kDetRows;
  return (size_t)units * nblk * d * sizeof(double);
}

// The partials buffer: the caller's workspace, or (ws == NULL) a stream-ordered allocation
static int detect_part(void* ws, size_t ws_bytes, size_t need, cudaStream_t st, double** part, bool* owned) {
  *owned = false;
  if (ws != nullptr) {
    if (ws_bytes < need) {
      set_error("detection workspace needs %zu bytes, got %zu", need, ws_bytes);
      return QJL_ERR_WORKSPACE;
    }
    *part = (double*)ws;
    return QJL_OK;
  }
  cudaError_t e = cudaMallocAsync((void**)part, need, st);
  if (e != cudaSuccess) return cuda_status(e, "detection workspace");
  *owned = true;
  return QJL_OK;
}

int launch_detect_outliers(const void* keys, int dtype, int units, int64_t n0, int d,
                           int64_t unit_stride, int h, int32_t* channels, double* mags, void* ws,
                           size_t ws_bytes, cudaStream_t st) {
  const size_t es = dtype_size(dtype);
  const bool two_phase = n0 >= 2 * kDetRows && d <= 1024 && (d * es) % 16 == 0 && (unit_stride * es) % 16 == 0 &&
                         ((uintptr_t)keys % 16) == 0 && 256 % (int)(d * es / 16) == 0;
  if (two_phase) {
    const int nblk = (int)((n0 + kDetRows - 1) / kDetRows);
    double* part = nullptr;
    bool owned = false;
    const int rc = detect_part(ws, ws_bytes, (size_t)units * nblk * d * sizeof(double), st, &part, &owned);
    if (rc != QJL_OK) return rc;
    const int tpr = (int)(d * es / 16), rows_par = 256 / tpr;
    const size_t smem = det_partial_smem(d, es, rows_par);
    dim3 grid(nblk, units);
    switch (dtype) {
#define QJL_DETP(DT)                                                                             \
  case DT: {                                                                                     \
    auto kern = k_detect_partial<Elem<DT>::T>;                                                   \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kern<<<grid, 256, smem, st>>>((const Elem<DT>::T*)keys, n0, d, unit_stride, part);           \
    break;                                                                                       \
  }
      QJL_DETP(QJL_F32)
      QJL_DETP(QJL_F16)
      QJL_DETP(QJL_BF16)
      QJL_DETP(QJL_F64)
#undef QJL_DETP
      default:
        if (owned) cudaFreeAsync(part, st);
        return QJL_ERR_ARG;
    }
    k_detect_finish<<<units, 1024, 0, st>>>(part, nblk, n0, d, h, channels, mags);
    if (owned) cudaFreeAsync(part, st);
    QJL_LAUNCH_CHECK("detect_outliers");
    return QJL_OK;
  }
  const int rows_par = (1024 / d) > 0 ? 1024 / d : 1;
  const int threads = rows_par * d;
  const size_t smem = (size_t)rows_par * d * sizeof(double);
  switch (dtype) {
#define QJL_DET(DT)                                                                         \
  case DT: {                                                                                \
    auto kern = k_detect_outliers<Elem<DT>::T>;                                             \
    if (smem > 48 * 1024)                                                                   \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    kern<<<units, threads, smem, st>>>((const Elem<DT>::T*)keys, n0, d, unit_stride, h,     \
                                       channels, mags);                                     \
    break;                                                                                  \
  }
    QJL_DET(QJL_F32)
    QJL_DET(QJL_F16)
    QJL_DET(QJL_BF16)
    QJL_DET(QJL_F64)
#undef QJL_DET
    default: return QJL_ERR_ARG;
  }
  QJL_LAUNCH_CHECK("detect_outliers");
  return QJL_OK;
}

// ---------------------------------------------------------------------------
// Per-unit zero-padded sketch: rows [0, m_in) carry S_in at the
// inlier columns in ascending order, rows [m_in, m_in+m_out) carry S_out at the
// outlier columns; everything else is 0.  Rounded once to the operand dtype.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_build_sketch(const double* __restrict__ s_in, const double* __restrict__ s_out,
                               int m_in, int m_out, int d, int h,
                               const int32_t* __restrict__ channels, T* __restrict__ s_full) {
  __shared__ int rank_in[1024];
  __shared__ int rank_out[1024];
  const int u = blockIdx.y;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    int ro = -1, below = 0;
    for (int j = 0; j < h; ++j) {
      const int ch = channels[(int64_t)u * h + j];
      ro = (ch == c) ? j : ro;
      below += ch < c;
    }
    rank_out[c] = ro;
    rank_in[c] = ro >= 0 ? -1 : c - below;
  }
  __syncthreads();
  const int m_total = m_in + m_out;
  const int d_in = d - h;
  T* out = s_full + (int64_t)u * m_total * d;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < m_total * d;
       idx += gridDim.x * blockDim.x) {
    const int r = idx / d, c = idx % d;
    double v = 0.0;
    if (r < m_in) {
      if (rank_in[c] >= 0) v = s_in[(int64_t)r * d_in + rank_in[c]];
    } else if (rank_out[c] >= 0) {
      v = s_out[(int64_t)(r - m_in) * h + rank_out[c]];
    }
    out[idx] = from_f64<T>(v);
  }
}

int launch_build_sketch(const double* s_in, const double* s_out, int m_in, int m_out, int d,
                        int h, const int32_t* channels, int units, int dtype, void* s_full,
                        cudaStream_t st) {
  const int m_total = m_in + m_out;
  dim3 grid((m_total * d + 255) / 256 < 64 ? (m_total * d + 255) / 256 : 64, units);
  switch (dtype) {
#define QJL_BS(DT)                                                                      \
  case DT:                                                                              \
    k_build_sketch<Elem<DT>::T><<<grid, 256, 0, st>>>(s_in, s_out, m_in, m_out, d, h,   \
                                                      channels, (Elem<DT>::T*)s_full);  \
    break;
    QJL_BS(QJL_F32)
    QJL_BS(QJL_F16)
    QJL_BS(QJL_BF16)
    QJL_BS(QJL_F64)
#undef QJL_BS
    default: return QJL_ERR_ARG;
  }
  QJL_LAUNCH_CHECK("build_sketch");
  return QJL_OK;
}

// ---------------------------------------------------------------------------
// Fused prefill profile: the per-unit finish of the two-phase
// detection (fixed-order sum of the block partials, mean, rank, channels) builds the
// unit's zero-padded S_full in the same CTA, from the channel ranks it already holds
// in shared memory -- no channels round trip, no separate build launch.  Same bits
// as k_detect_finish followed by k_build_sketch.
// ---------------------------------------------------------------------------
template <typename TS>
__global__ void __launch_bounds__(1024, 1) k_detect_finish_build(
    const double* __restrict__ part, int nblk, int64_t n0, int d, int h, int32_t* __restrict__ channels,
    double* __restrict__ magnitudes, const TS* __restrict__ s_in, const TS* __restrict__ s_out,
    int m_in, int m_out, TS* __restrict__ s_full) {
  __shared__ double mag[1024];
  __shared__ double red[1024];
  __shared__ int rank[1024];
  __shared__ int src[1024];           // column c: inlier rank, or -1 - outlier rank
  __shared__ int below[1024];
  // grid (units, row slices): every CTA of a unit re-derives the ranking from the partials
  // (parallel, cheap) and builds its slice of S_full rows; slice 0 publishes channels and
  // magnitudes
  // K1 (launched next with programmatic serialization) may start its setup now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int u = blockIdx.x, c = threadIdx.x;
  const bool publish = blockIdx.y == 0;
#ifndef QJL_FB_ABLATE
#define QJL_FB_ABLATE 0      // perf experiments: 1 skip the build, 2 skip the ranking too
#endif
  const int m_total = m_in + m_out, d_in = d - h;
  const int r0 = (int)((int64_t)blockIdx.y * m_total / gridDim.y);
  const int r1 = (int)((int64_t)(blockIdx.y + 1) * m_total / gridDim.y);
  // S_in / S_out arrive in the operand dtype, so the build is a column scatter.  The
  // slice's source rows are staged in shared memory first (contiguous, vector loads all
  // in flight at once), then every thread assembles 16-byte chunks of output rows.
  extern __shared__ __align__(16) uint8_t s_dyn[];
  TS* s_rows = reinterpret_cast<TS*>(s_dyn);
  const int ia = r0, ib = min(r1, m_in), nin = max(0, ib - ia);
  const int oa = max(r0, m_in) - m_in, ob = r1 - m_in, nout = max(0, ob - oa);
  // contiguous 16 B aligned spans go through one bulk copy (TMA engine, mbarrier
  // completion); anything else is copied element-wise
  __shared__ __align__(8) uint64_t stage_bar;
  auto bulk_ok = [&](const TS* src, int64_t n_el, TS* dst) {
    return ((uintptr_t)src & 15) == 0 && ((n_el * (int64_t)sizeof(TS)) & 15) == 0 && ((uintptr_t)dst & 15) == 0 &&
           n_el * (int64_t)sizeof(TS) < (1 << 20);
  };
  TS* s_out_rows = s_rows + (((int64_t)nin * d_in * sizeof(TS) + 15) / 16 * 16) / sizeof(TS);
  const TS* src_a = s_in + (int64_t)ia * d_in;
  const TS* src_b = s_out + (int64_t)oa * h;
  const int64_t na = (int64_t)nin * d_in, nb = (int64_t)nout * h;
  const bool bulk_a = !(QJL_FB_ABLATE & 4) && nin && bulk_ok(src_a, na, s_rows),
             bulk_b = !(QJL_FB_ABLATE & 4) && nout && bulk_ok(src_b, nb, s_out_rows);
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&stage_bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t bytes = (uint32_t)((bulk_a ? na : 0) + (bulk_b ? nb : 0)) * sizeof(TS);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    if (bulk_a)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(s_rows)),
                   "l"(src_a), "r"((uint32_t)(na * sizeof(TS))), "r"(bar)
                   : "memory");
    if (bulk_b)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(s_out_rows)),
                   "l"(src_b), "r"((uint32_t)(nb * sizeof(TS))), "r"(bar)
                   : "memory");
  }
  if (nin && !bulk_a && !(QJL_FB_ABLATE & 4))
    for (int64_t i = threadIdx.x; i < na; i += blockDim.x) s_rows[i] = src_a[i];
  if (nout && !bulk_b && !(QJL_FB_ABLATE & 4))
    for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) s_out_rows[i] = src_b[i];
  // PDL: the staging above reads only the sketches (inputs of the call); the partials come
  // from k_detect_partial, launched just before with programmatic serialization
  asm volatile("griddepcontrol.wait;" ::: "memory");
  channel_means(part, u, nblk, d, n0, mag, red);
  if (QJL_FB_ABLATE & 2) return;
  channel_ranks(mag, d, rank);
  // outlier flags as one bit per channel (warp ballots) -> prefix counts by popc
  const bool is_out = c < d && rank[c] < h;
  const unsigned bal = __ballot_sync(0xffffffffu, is_out);
  if ((c & 31) == 0 && c < d) below[c >> 5] = (int)bal;
  if (c < d && magnitudes && publish) magnitudes[(int64_t)u * d + c] = mag[c];
  __syncthreads();
  if (c < d) {
    // ascending position among the outliers / among the inliers (kvcache.py:90-101)
    int nb = __popc((unsigned)below[c >> 5] & ((1u << (c & 31)) - 1u));
    for (int w = 0; w < (c >> 5); ++w) nb += __popc((unsigned)below[w]);
    if (is_out && publish) channels[(int64_t)u * h + nb] = c;
    src[c] = is_out ? -1 - nb : c - nb;
  }
  __syncthreads();
  __syncthreads();                     // barrier init visible; element-wise copies done
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(bar)
      : "memory");
  TS* out = s_full + (int64_t)u * m_total * d;
  const TS zero = from_f64<TS>(0.0);
  constexpr int V = 16 / (int)sizeof(TS);          // columns per 16-byte store
  const int cpr = (d + V - 1) / V;
  if (d % V == 0 && blockDim.x % cpr == 0) {
    // every thread keeps the same V columns for all its rows: source columns in registers
    const int c0 = (threadIdx.x % cpr) * V;
    int ci[V], co[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int sc = src[c0 + j];
      ci[j] = sc >= 0 ? sc : -1;
      co[j] = sc < 0 ? -1 - sc : -1;
    }
    const int rstep = blockDim.x / cpr;
    for (int r = r0 + threadIdx.x / cpr; r < r1; r += rstep) {
      TS o[V];
      if (r < m_in) {
        const TS* row = s_rows + (r - ia) * d_in;
#pragma unroll
        for (int j = 0; j < V; ++j) o[j] = ci[j] >= 0 ? row[ci[j]] : zero;
      } else {
        const TS* row = s_out_rows + (r - m_in - oa) * h;
#pragma unroll
        for (int j = 0; j < V; ++j) o[j] = co[j] >= 0 ? row[co[j]] : zero;
      }
      if (!(QJL_FB_ABLATE & 8) || r < 0)
        *reinterpret_cast<uint4*>(out + (int64_t)r * d + c0) = *reinterpret_cast<const uint4*>(o);
    }
    return;
  }
  for (int t = threadIdx.x; t < (r1 - r0) * cpr; t += blockDim.x) {
    const int r = r0 + t / cpr, c0 = (t % cpr) * V;
    TS o[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c = c0 + j;
      const int sc = c < d ? src[c] : 0;
      TS v = zero;
      if (r < m_in) {
        if (sc >= 0) v = s_rows[(r - ia) * d_in + sc];
      } else if (sc < 0) {
        v = s_out_rows[(r - m_in - oa) * h + (-1 - sc)];
      }
      o[j] = v;
    }
    TS* dst = out + (int64_t)r * d + c0;
    if (d % V == 0) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(o);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j)
        if (c0 + j < d) dst[j] = o[j];
    }
  }
}

// S_full from operand-dtype S_in / S_out and given channels (fallback of the fused path)
template <typename TS>
__global__ void k_scatter_sketch(const TS* __restrict__ s_in, const TS* __restrict__ s_out, int m_in, int m_out,
                                 int d, int h, const int32_t* __restrict__ channels, TS* __restrict__ s_full) {
  __shared__ int src[1024];
  const int u = blockIdx.y;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    int ro = -1, below = 0;
    for (int j = 0; j < h; ++j) {
      const int ch = channels[(int64_t)u * h + j];
      ro = (ch == c) ? j : ro;
      below += ch < c;
    }
    src[c] = ro >= 0 ? -1 - ro : c - below;
  }
  __syncthreads();
  const int m_total = m_in + m_out, d_in = d - h;
  TS* out = s_full + (int64_t)u * m_total * d;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < m_total * d; idx += gridDim.x * blockDim.x) {
    const int r = idx / d, c = idx % d, sc = src[c];
    TS v = from_f64<TS>(0.0);
    if (r < m_in) {
      if (sc >= 0) v = s_in[(int64_t)r * d_in + sc];
    } else if (sc < 0) {
      v = s_out[(int64_t)(r - m_in) * h + (-1 - sc)];
    }
    out[idx] = v;
  }
}

static int launch_scatter_sketch(const void* s_in, const void* s_out, int m_in, int m_out, int d, int h,
                                 const int32_t* channels, int units, int dtype, void* s_full, cudaStream_t st) {
  const int m_total = m_in + m_out;
  dim3 grid((m_total * d + 255) / 256 < 64 ? (m_total * d + 255) / 256 : 64, units);
  switch (dtype) {
#define QJL_SS(DT)                                                                                 \
  case DT:                                                                                         \
    k_scatter_sketch<Elem<DT>::T><<<grid, 256, 0, st>>>((const Elem<DT>::T*)s_in,                  \
                                                        (const Elem<DT>::T*)s_out, m_in, m_out, d, \
                                                        h, channels, (Elem<DT>::T*)s_full);        \
    break;
    QJL_SS(QJL_F32)
    QJL_SS(QJL_F16)
    QJL_SS(QJL_BF16)
    QJL_SS(QJL_F64)
#undef QJL_SS
    default: return QJL_ERR_ARG;
  }
  QJL_LAUNCH_CHECK("scatter_sketch");
  return QJL_OK;
}

int launch_prefill_profile(const void* keys, int dtype, int units, int64_t n0, int d, int64_t unit_stride,
                           int h, const void* s_in, const void* s_out, int m_in, int m_out,
                           int sketch_dtype, int32_t* channels, double* mags, void* s_full, void* ws,
                           size_t ws_bytes, cudaStream_t st) {
  const size_t es = dtype_size(dtype);
  const bool two_phase = n0 >= 2 * kDetRows && d <= 1024 && (d * es) % 16 == 0 && (unit_stride * es) % 16 == 0 &&
                         ((uintptr_t)keys % 16) == 0 && 256 % (int)(d * es / 16) == 0 && h > 0;
  if (!two_phase) {
    int rc = h > 0 ? launch_detect_outliers(keys, dtype, units, n0, d, unit_stride, h, channels, mags, ws,
                                            ws_bytes, st)
                   : QJL_OK;
    if (rc != QJL_OK) return rc;
    return launch_scatter_sketch(s_in, s_out, m_in, m_out, d, h, channels, units, sketch_dtype, s_full, st);
  }
  const int nblk = (int)((n0 + kDetRows - 1) / kDetRows);
  double* part = nullptr;
  bool owned = false;
  const int prc = detect_part(ws, ws_bytes, (size_t)units * nblk * d * sizeof(double), st, &part, &owned);
  if (prc != QJL_OK) return prc;
  const int tpr = (int)(d * es / 16), rows_par = 256 / tpr;
  const size_t smem = det_partial_smem(d, es, rows_par);
  dim3 grid(nblk, units);
  switch (dtype) {
#define QJL_PPP(DT)                                                                                  \
  case DT: {                                                                                         \
    auto kern = k_detect_partial<Elem<DT>::T>;                                                       \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kern<<<grid, 256, smem, st>>>((const Elem<DT>::T*)keys, n0, d, unit_stride, part);               \
    break;                                                                                           \
  }
    QJL_PPP(QJL_F32)
    QJL_PPP(QJL_F16)
    QJL_PPP(QJL_BF16)
    QJL_PPP(QJL_F64)
#undef QJL_PPP
    default:
      if (owned) cudaFreeAsync(part, st);
      return QJL_ERR_ARG;
  }
  // row slices: about one wave of 1024-thread CTAs (1 per SM) over all units, and few
  // enough source rows per slice to stage them in <= 160 KB of shared memory
  const size_t ts = dtype_size(sketch_dtype);
  const size_t row_bytes = (size_t)std::max(d - h, h) * ts;          // widest source row
  const int m_total = m_in + m_out;
  // d <= 256: 256-thread CTAs (one thread per channel), 3 resident per SM (28 KB of static
  // ranking arrays + the staged rows each), so a unit's rows are built by ~3 x SMs / units
  // CTAs in one wave (C4: 3 slices of 192 rows per unit; one 1024-thread CTA per unit left
  // 20 SMs idle and ran the latency-bound ranking and the 123 KB staging serially per SM)
  const int fb_threads = d <= 256 ? 256 : 1024;
  int slices = std::max(1, device_sm_count() * (fb_threads == 256 ? 3 : 1) / units);
  const int max_rows = std::max(1, (int)((160 * 1024 - 64) / row_bytes) - 1);
  slices = std::max(slices, (m_total + max_rows - 1) / max_rows);
  slices = std::min(slices, m_total);
  const size_t smem_fb = ((size_t)(m_total + slices - 1) / slices + 1) * row_bytes + 64;
  cudaLaunchAttribute fattr[1];
  fattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  fattr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t fcfg = {};
  fcfg.gridDim = dim3(units, slices);
  fcfg.blockDim = dim3(fb_threads);
  fcfg.dynamicSmemBytes = smem_fb;
  fcfg.stream = st;
  fcfg.attrs = fattr;
  fcfg.numAttrs = 1;
  cudaError_t fb_err = cudaSuccess;
  switch (sketch_dtype) {
#define QJL_PPF(DT)                                                                                     \
  case DT:                                                                                              \
    cudaFuncSetAttribute(k_detect_finish_build<Elem<DT>::T>,                                            \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fb);                    \
    fb_err = cudaLaunchKernelEx(&fcfg, k_detect_finish_build<Elem<DT>::T>, (const double*)part, nblk, n0, d, h, \
                                channels, mags, (const Elem<DT>::T*)s_in, (const Elem<DT>::T*)s_out, m_in,   \
                                m_out, (Elem<DT>::T*)s_full);                                                \
    break;
    QJL_PPF(QJL_F32)
    QJL_PPF(QJL_F16)
    QJL_PPF(QJL_BF16)
    QJL_PPF(QJL_F64)
#undef QJL_PPF
    default:
      if (owned) cudaFreeAsync(part, st);
      return QJL_ERR_ARG;
  }
  if (fb_err != cudaSuccess) {
    if (owned) cudaFreeAsync(part, st);
    return cuda_status(fb_err, "prefill_profile");
  }
  if (owned) cudaFreeAsync(part, st);
  QJL_LAUNCH_CHECK("prefill_profile");
  return QJL_OK;
}

// ---------------------------------------------------------------------------
// Generic key quantizer (estimator.py:110-124 batched, kvcache.py:293-306):
// projections in fp64 (exact products, fp64 sums), sign test `p >= 0` (ties and
// -0.0 -> 1, NaN -> 0), bits packed with warp ballots: lane j of a warp owns
// sketch row 32w+j, so the ballot word IS the LSB-first u32 of those 32 rows.
// Norms ||k_in||, ||k_out|| in fp64, rounded once to fp16.
// CTA = 128 threads x TOK tokens; thread t owns sketch rows t + 128 i (i < RPT).  S is
// staged through smem kQCk columns at a time as [kQCk][m_total + 1] (conflict-free row
// reads and staging stores), the tokens as [d][TOK] so one 16-byte broadcast load feeds
// 2 tokens x RPT rows of FMAs.  The fp64 FMA chain per (row, token) runs over c in increasing order.
// ---------------------------------------------------------------------------
constexpr int kQCk = 16;
#ifndef QJL_QK_PRE
#define QJL_QK_PRE 1
#endif

template <typename TK, typename TS, int RPT, int TOK, int kQThreads>
__global__ void __launch_bounds__(kQThreads) k_quantize_keys_simt(
    const TK* __restrict__ keys, int64_t n, int64_t key_unit_stride, const TS* __restrict__ s_full,
    int64_t s_unit_stride, int d, int m_in, int m_out, const int32_t* __restrict__ channels, int h,
    qjl_key_cache_t kc, int64_t row_offset) {
  extern __shared__ double sm[];
  constexpr int kQTok = TOK;
  const int m_total = m_in + m_out;
  double* sk = sm;                         // [d][kQTok]
  double* ss = sm + kQTok * d;             // [kQCk][m_total + 1] (padded: conflict-free staging)
  const int msp = m_total + 1;
  __shared__ unsigned char is_out[1024];
  const int u = blockIdx.y;
  const int64_t t0 = (int64_t)blockIdx.x * kQTok;
  const TK* K = keys + (int64_t)u * key_unit_stride;
  const TS* S = s_full + (int64_t)u * s_unit_stride;

  for (int c = threadIdx.x; c < d; c += blockDim.x) is_out[c] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < h; j += blockDim.x) is_out[channels[(int64_t)u * h + j]] = 1;
  for (int i = threadIdx.x; i < kQTok * d; i += blockDim.x) {
    const int tt = i / d, c = i % d;                 // coalesced key reads, transposed store
    sk[c * kQTok + tt] = (t0 + tt < n) ? to_f64(K[(t0 + tt) * d + c]) : 0.0;
  }

  double acc[RPT][kQTok];
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int t = 0; t < kQTok; ++t) acc[i][t] = 0.0;

  // S chunks: the next chunk's values are loaded into registers while the current one is
  // multiplied (element e of the thread: i = threadIdx.x + 128 e, row i / kQCk, col i % kQCk)
  constexpr bool kPre = QJL_QK_PRE && RPT <= 2;       // register budget: prefetch for m <= 256 only
  constexpr int PF = kPre ? RPT * kQCk : 1;
  double pf[PF];
  auto load_chunk = [&](int c0) {
    if (!kPre) return;
#pragma unroll
    for (int e = 0; e < PF; ++e) {
      const int i = threadIdx.x + e * kQThreads, r = i / kQCk, cc = i % kQCk;
      pf[e] = (r < m_total && c0 + cc < d) ? to_f64(S[(int64_t)r * d + c0 + cc]) : 0.0;
    }
  };
  load_chunk(0);
  for (int c0 = 0; c0 < d; c0 += kQCk) {
    __syncthreads();                                  // the previous chunk's reads of ss are done
    if constexpr (kPre) {
#pragma unroll
      for (int e = 0; e < PF; ++e) {
        const int i = threadIdx.x + e * kQThreads, r = i / kQCk, cc = i % kQCk;
        if (r < m_total) ss[cc * msp + r] = pf[e];
      }
    } else {
      for (int i = threadIdx.x; i < m_total * kQCk; i += blockDim.x) {
        const int r = i / kQCk, cc = i % kQCk;
        ss[cc * msp + r] = (c0 + cc < d) ? to_f64(S[(int64_t)r * d + c0 + cc]) : 0.0;
      }
    }
    __syncthreads();
    if (c0 + kQCk < d) load_chunk(c0 + kQCk);         // in flight during this chunk's FMAs
    const int ncc = min(kQCk, d - c0);
    for (int cc = 0; cc < ncc; ++cc) {
      double sv[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = threadIdx.x + i * kQThreads;
        sv[i] = r < m_total ? ss[cc * msp + r] : 0.0;
      }
      const double2* kv2 = reinterpret_cast<const double2*>(sk + (c0 + cc) * kQTok);
#pragma unroll
      for (int t2 = 0; t2 < kQTok / 2; ++t2) {
        const double2 kv = kv2[t2];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          acc[i][2 * t2] = fma(sv[i], kv.x, acc[i][2 * t2]);
          acc[i][2 * t2 + 1] = fma(sv[i], kv.y, acc[i][2 * t2 + 1]);
        }
      }
    }
  }

  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r0 = (threadIdx.x & ~31) + i * kQThreads;  // warp-uniform first row
    if (r0 >= m_total) continue;
#pragma unroll
    for (int t = 0; t < kQTok; ++t) {
      const unsigned word = __ballot_sync(0xffffffffu, acc[i][t] >= 0.0);
      const int64_t row = row_offset + t0 + t;
      if (lane == 0 && t0 + t < n) {
        if (r0 < m_in) {
          reinterpret_cast<uint32_t*>(kc.bits_in + row_off(u, row, m_in / 8, kc.capacity, kc.tile_stride))[r0 / 32] = word;
        } else {
          reinterpret_cast<uint32_t*>(kc.bits_out + row_off(u, row, m_out / 8, kc.capacity, kc.tile_stride))[(r0 - m_in) / 32] =
              word;
        }
      }
    }
  }

  // norms: one warp per token
  const int warp = threadIdx.x >> 5;
  for (int t = warp; t < kQTok; t += kQThreads / 32) {
    if (t0 + t >= n) continue;
    double s_in = 0.0, s_out = 0.0;
    for (int c = lane; c < d; c += 32) {
      const double v = sk[c * kQTok + t];
      if (is_out[c]) s_out = fma(v, v, s_out); else s_in = fma(v, v, s_in);
    }
    s_in = warp_sum_f64(s_in);
    s_out = warp_sum_f64(s_out);
    if (lane == 0) {
      const int64_t no = row_off(u, row_offset + t0 + t, 2, kc.capacity, kc.tile_stride);
      *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(kc.norm_in) + no) = f16_canon(f64_to_f16_bits(sqrt(s_in)));
      if (m_out > 0)
        *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(kc.norm_out) + no) = f16_canon(f64_to_f16_bits(sqrt(s_out)));
    }
  }
}

template <typename TK, typename TS>
static int launch_qk_simt_2(const void* keys, int64_t n, int64_t kus, const void* s, int64_t sus,
                            int d, int m_in, int m_out, const int32_t* ch, int h,
                            const qjl_key_cache_t& kc, int64_t row_offset, cudaStream_t st) {
  const int m_total = m_in + m_out;
  const int nt = m_total <= 256 ? 128 : 256;          // CTA threads: <= 4 sketch rows per thread
  const int rpt = (m_total + nt - 1) / nt;
  const int tok = rpt <= 4 ? 16 : 8;                  // acc[RPT][TOK] in registers
#define QJL_QK(R, TT, NT)                                                                  \
  if (nt == NT && rpt == R && tok == TT) {                                                 \
    auto kern = k_quantize_keys_simt<TK, TS, R, TT, NT>;                                   \
    const size_t smem = ((size_t)TT * d + (size_t)(m_total + 1) * kQCk) * sizeof(double);  \
    dim3 grid((unsigned)((n + TT - 1) / TT), kc.units);                                    \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    timing_begin(st);                                                                      \
    kern<<<grid, NT, smem, st>>>((const TK*)keys, n, kus, (const TS*)s, sus, d,            \
                                 m_in, m_out, ch, h, kc, row_offset);                      \
    timing_end(st);                                                                        \
    QJL_LAUNCH_CHECK("quantize_keys_simt");                                                \
    return QJL_OK;                                                                         \
  }
  QJL_QK(1, 16, 128)
  QJL_QK(2, 16, 128)
  QJL_QK(2, 16, 256)
  QJL_QK(3, 16, 256)
  QJL_QK(4, 16, 256)
#undef QJL_QK
  set_error("quantize_keys: m_in + m_out = %d exceeds 1024", m_total);
  return QJL_ERR_UNSUPPORTED;
}

template <typename TK>
static int launch_qk_simt_1(const void* keys, int64_t n, int64_t kus, const qjl_sketch_t& sk,
                            int d, int m_in, int m_out, const int32_t* ch, int h,
                            const qjl_key_cache_t& kc, int64_t row_offset, cudaStream_t st) {
  switch (sk.dtype) {
    case QJL_F64: return launch_qk_simt_2<TK, double>(keys, n, kus, sk.s_full, sk.unit_stride, d, m_in, m_out, ch, h, kc, row_offset, st);
    case QJL_F32: return launch_qk_simt_2<TK, float>(keys, n, kus, sk.s_full, sk.unit_stride, d, m_in, m_out, ch, h, kc, row_offset, st);
    case QJL_F16: return launch_qk_simt_2<TK, __half>(keys, n, kus, sk.s_full, sk.unit_stride, d, m_in, m_out, ch, h, kc, row_offset, st);
    case QJL_BF16: return launch_qk_simt_2<TK, __nv_bfloat16>(keys, n, kus, sk.s_full, sk.unit_stride, d, m_in, m_out, ch, h, kc, row_offset, st);
  }
  return QJL_ERR_ARG;
}

int launch_quantize_keys_simt(const void* keys, int dtype, int64_t n, int64_t kus,
                              const qjl_sketch_t& sk, const int32_t* ch, int h,
                              const qjl_key_cache_t& kc, int64_t row_offset, cudaStream_t st) {
  const int d = kc.d, m_in = kc.m_in, m_out = kc.m_out;
  switch (dtype) {
    case QJL_F32: return launch_qk_simt_1<float>(keys, n, kus, sk, d, m_in, m_out, ch, h, kc, row_offset, st);
    case QJL_F64: return launch_qk_simt_1<double>(keys, n, kus, sk, d, m_in, m_out, ch, h, kc, row_offset, st);
    case QJL_F16: return launch_qk_simt_1<__half>(keys, n, kus, sk, d, m_in, m_out, ch, h, kc, row_offset, st);
    case QJL_BF16: return launch_qk_simt_1<__nv_bfloat16>(keys, n, kus, sk, d, m_in, m_out, ch, h, kc, row_offset, st);
  }
  return QJL_ERR_ARG;
}

// ---------------------------------------------------------------------------
// Value quantizer (kvcache.py:140-161) per group: zero = min, scale =
// (max - min)/(2^b - 1), codes = clip(rint((v - zero)/scale)) -- all in fp64 so
// codes match the reference bit for bit (IEEE div + rint are exact-rounded);
// constant group -> scale 0, codes 0.  Constants stored fp16 (P2T) or f32 (U8).
// One warp per token; lane l owns dims l + 32*i.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_quantize_values(const T* __restrict__ v, int64_t n,
                                                         int64_t unit_stride,
                                                         qjl_value_cache_t vc, int64_t row_offset) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.y;
  const int64_t t = (int64_t)blockIdx.x * 8 + warp;
  const int d = vc.d, G = d / vc.group, gs = vc.group;
  const int levels = (1 << vc.bits) - 1;
  const bool valid = t < n;
  const T* V = v + (int64_t)u * unit_stride + (valid ? t : 0) * d;
  const int64_t r = row_offset + t;
  const int64_t row = (int64_t)u * vc.capacity + r;   // U8 (rows layout) row index
  const bool p2 = vc.layout == QJL_VLAYOUT_P2T;
  for (int g = 0; g < G; ++g) {
    // group g spans dims [g*gs, (g+1)*gs); lanes stride over it
    double mn = INFINITY, mx = -INFINITY;
    for (int i = lane; i < gs; i += 32) {
      const double x = to_f64(V[g * gs + i]);
      mn = fmin(mn, x);
      mx = fmax(mx, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const double zero = mn;
    const double spread = mx - mn;
    const double scale = spread == 0.0 ? 0.0 : spread / (double)levels;
    for (int i = lane; i < gs; i += 32) {
      const int dim = g * gs + i;
      int code = 0;
      if (spread != 0.0) {
        double q = rint((to_f64(V[dim]) - zero) / scale);
        q = fmin(fmax(q, 0.0), (double)levels);
        code = (int)q;
      }
      if (!p2) {
        if (valid) reinterpret_cast<uint8_t*>(vc.codes)[row * d + dim] = (uint8_t)code;
      } else {
        // P2T: dims 4a..4a+3 share a byte (slot = dim & 3); OR the four lanes together
        uint32_t b = (uint32_t)code << (2 * (lane & 3));
        b |= __shfl_xor_sync(0xffffffffu, b, 1);
        b |= __shfl_xor_sync(0xffffffffu, b, 2);
        if (valid && (lane & 3) == 0)
          reinterpret_cast<uint8_t*>(vc.codes)[tile_off(u, r, 4096, vc.capacity, vc.tile_stride) + p2t_byte(r, dim)] =
              (uint8_t)b;
      }
    }
    if (valid && lane == 0) {
      if (!p2) {
        reinterpret_cast<float*>(vc.zero)[row * G + g] = (float)zero;
        reinterpret_cast<float*>(vc.scale)[row * G + g] = (float)scale;
      } else {
        const int64_t o = row_off(u, r, 2 * G, vc.capacity, vc.tile_stride) + 2 * g;
        *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(vc.zero) + o) = f64_to_f16_bits(zero);
        *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(vc.scale) + o) = f64_to_f16_bits(scale);
      }
    }
  }
}

// P2T fast path (2-bit, group 32, d = 128): one thread per (4-token block, group).  The
// screen runs in fp32; codes whose quotient lies within 1e-3 of a rounding boundary
// are recomputed exactly as the reference does, in fp64 (kvcache.py:151-159:
// rint((v - zero) / ((max - min) / 3))), so codes match the reference bit for bit.
template <typename T>
__global__ void __launch_bounds__(256) k_quantize_values_p2t(const T* __restrict__ v, int64_t n,
                                                             int64_t unit_stride, qjl_value_cache_t vc,
                                                             int64_t row_offset) {
  constexpr int EPV = 16 / (int)sizeof(T);
  const int u = blockIdx.y;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int g = (int)(idx & 3);
  const int64_t t0 = (idx >> 2) * 4;                    // first token of this thread's block
  if (t0 >= n) return;
  const T* V = v + (int64_t)u * unit_stride;
  uint8_t* codes = reinterpret_cast<uint8_t*>(vc.codes);
  uint8_t* zo = reinterpret_cast<uint8_t*>(vc.zero);
  uint8_t* so = reinterpret_cast<uint8_t*>(vc.scale);
  uint32_t cw[4][8];                                    // [token][byte a = 4-dim slot group] (bits of one byte)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t t = t0 + i;
#pragma unroll
    for (int a = 0; a < 8; ++a) cw[i][a] = 0u;
    if (t >= n) continue;
    float x[32];
    const T* src = V + t * 128 + 32 * g;
#pragma unroll
    for (int k = 0; k < 32 / EPV; ++k) {
      const uint4 raw = *reinterpret_cast<const uint4*>(src + k * EPV);
      const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int j = 0; j < EPV; ++j) x[k * EPV + j] = to_f32(e[j]);
    }
    float mn = x[0], mx = x[0];
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      mn = fminf(mn, x[k]);
      mx = fmaxf(mx, x[k]);
    }
    const double mn64 = (double)mn, mx64 = (double)mx;   // inputs are exact in fp32
    const double spread = mx64 - mn64;
    const double scale = spread == 0.0 ? 0.0 : spread / 3.0;
    const int64_t co = row_off(u, row_offset + t, 8, vc.capacity, vc.tile_stride) + 2 * g;
    *reinterpret_cast<uint16_t*>(zo + co) = f64_to_f16_bits(mn64);
    *reinterpret_cast<uint16_t*>(so + co) = f64_to_f16_bits(scale);
    if (spread != 0.0) {
      const float inv = 3.0f / (float)spread;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float q = (x[k] - mn) * inv;
        float r = rintf(q);
        if (fabsf(q - floorf(q) - 0.5f) < 1e-3f)        // near a tie: exact fp64 quotient
          r = (float)rint(((double)x[k] - mn64) / scale);
        const uint32_t c = (uint32_t)fminf(fmaxf(r, 0.f), 3.f);
        cw[i][k >> 2] |= c << (2 * (k & 3));
      }
    }
  }
  // dims 32g + 4a' .. + 3 of token t form byte (8g + a') of the P2T tile layout
  const int64_t r0 = row_offset + t0;
  if ((r0 & 3) == 0 && t0 + 4 <= n) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const uint32_t w = cw[0][a] | (cw[1][a] << 8) | (cw[2][a] << 16) | (cw[3][a] << 24);
      const int64_t byte = tile_off(u, r0, 4096, vc.capacity, vc.tile_stride) + p2t_byte(r0, 32 * g + 4 * a);
      *reinterpret_cast<uint32_t*>(codes + byte) = w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (t0 + i >= n) break;
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        codes[tile_off(u, r0 + i, 4096, vc.capacity, vc.tile_stride) + p2t_byte(r0 + i, 32 * g + 4 * a)] =
            (uint8_t)cw[i][a];
      }
    }
  }
}

int launch_quantize_values(const void* v, int dtype, int64_t n, int64_t unit_stride,
                           const qjl_value_cache_t& vc, int64_t row_offset, cudaStream_t st) {
  const size_t es = dtype_size(dtype);
  if (vc.layout == QJL_VLAYOUT_P2T && dtype != QJL_F64 && ((uintptr_t)v % 16) == 0 &&
      (unit_stride * es) % 16 == 0) {
    const int64_t threads = ((n + 3) / 4) * 4;
    dim3 grid((unsigned)((threads + 255) / 256), vc.units);
    switch (dtype) {
      case QJL_F32:
        k_quantize_values_p2t<float><<<grid, 256, 0, st>>>((const float*)v, n, unit_stride, vc, row_offset);
        break;
      case QJL_F16:
        k_quantize_values_p2t<__half><<<grid, 256, 0, st>>>((const __half*)v, n, unit_stride, vc, row_offset);
        break;
      case QJL_BF16:
        k_quantize_values_p2t<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)v, n, unit_stride, vc,
                                                                   row_offset);
        break;
    }
    QJL_LAUNCH_CHECK("quantize_values_p2t");
    return QJL_OK;
  }
  dim3 grid((unsigned)((n + 7) / 8), vc.units);
  switch (dtype) {
#define QJL_QV(DT)                                                                          \
  case DT:                                                                                  \
    k_quantize_values<Elem<DT>::T><<<grid, 256, 0, st>>>((const Elem<DT>::T*)v, n,          \
                                                         unit_stride, vc, row_offset);      \
    break;
    QJL_QV(QJL_F32)
    QJL_QV(QJL_F16)
    QJL_QV(QJL_BF16)
    QJL_QV(QJL_F64)
#undef QJL_QV
    default: return QJL_ERR_ARG;
  }
  QJL_LAUNCH_CHECK("quantize_values");
  return QJL_OK;
}

}  // namespace qjl
