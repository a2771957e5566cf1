// Query sketch, generic score estimator, fp64 softmax.
#include "common.cuh"
#include "kernels.h"

namespace qjl {

// ---------------------------------------------------------------------------
// sketch_query (estimator.py:127-132): sq[u][g][r] = S_full[u][r] . q[u][g] in
// fp64, stored f32.  One CTA per (unit, query head).  Also returns, in
// `sums` (f32 [units][G][2]), the per-side totals sum_j Sq_j used by the
// 2*sum_set - sum_all identity (estimator.py:164-169).
// ---------------------------------------------------------------------------
template <typename TQ, typename TS, typename TO>
__global__ void __launch_bounds__(256) k_sketch_query(const TQ* __restrict__ q, int G, int d,
                                                      const TS* __restrict__ s_full,
                                                      int64_t s_unit_stride, int m_in, int m_total,
                                                      TO* __restrict__ sq,
                                                      float* __restrict__ sums) {
  extern __shared__ double qs[];  // [d] then [8] warp partials x 2
  const int ug = blockIdx.x;
  const int u = ug / G;
  const TQ* Q = q + (int64_t)ug * d;
  const TS* S = s_full + (int64_t)u * s_unit_stride;
  for (int c = threadIdx.x; c < d; c += blockDim.x) qs[c] = to_f64(Q[c]);
  __syncthreads();
  double part_in = 0.0, part_out = 0.0;
  for (int r = threadIdx.x; r < m_total; r += blockDim.x) {
    const TS* row = S + (int64_t)r * d;
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc = fma(to_f64(row[c]), qs[c], acc);
    sq[(int64_t)ug * m_total + r] = (TO)acc;
    if (r < m_in) part_in += (double)(float)acc; else part_out += (double)(float)acc;
  }
  if (sums) {
    double* red = qs + d;
    part_in = warp_sum_f64(part_in);
    part_out = warp_sum_f64(part_out);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { red[w] = part_in; red[8 + w] = part_out; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a += red[i]; b += red[8 + i]; }
      sums[(int64_t)ug * 2 + 0] = (float)a;
      sums[(int64_t)ug * 2 + 1] = (float)b;
    }
  }
}

template <typename TQ, typename TO>
static int launch_sq_1(const void* q, int units, int G, int d, const qjl_sketch_t& sk, int m_in,
                       int m_total, TO* sq, float* sums, cudaStream_t st) {
  const size_t smem = (d + 16) * sizeof(double);
  switch (sk.dtype) {
#define QJL_SQ(DT)                                                                           \
  case DT:                                                                                   \
    k_sketch_query<TQ, Elem<DT>::T, TO><<<units * G, 256, smem, st>>>(                       \
        (const TQ*)q, G, d, (const Elem<DT>::T*)sk.s_full, sk.unit_stride, m_in, m_total,    \
        sq, sums);                                                                           \
    break;
    QJL_SQ(QJL_F32)
    QJL_SQ(QJL_F16)
    QJL_SQ(QJL_BF16)
    QJL_SQ(QJL_F64)
#undef QJL_SQ
    default: return QJL_ERR_ARG;
  }
  QJL_LAUNCH_CHECK("sketch_query");
  return QJL_OK;
}

template <typename TO>
static int launch_sq_o(const void* q, int q_dtype, int units, int G, int d, const qjl_sketch_t& sk, int m_in,
                       int m_total, TO* sq, float* sums, cudaStream_t st) {
  switch (q_dtype) {
    case QJL_F32: return launch_sq_1<float, TO>(q, units, G, d, sk, m_in, m_total, sq, sums, st);
    case QJL_F16: return launch_sq_1<__half, TO>(q, units, G, d, sk, m_in, m_total, sq, sums, st);
    case QJL_BF16: return launch_sq_1<__nv_bfloat16, TO>(q, units, G, d, sk, m_in, m_total, sq, sums, st);
    case QJL_F64: return launch_sq_1<double, TO>(q, units, G, d, sk, m_in, m_total, sq, sums, st);
  }
  return QJL_ERR_ARG;
}

int launch_sketch_query(const void* q, int q_dtype, int units, int G, int d,
                        const qjl_sketch_t& sk, int m_in, int m_total, float* sq, float* sums,
                        cudaStream_t st) {
  return launch_sq_o<float>(q, q_dtype, units, G, d, sk, m_in, m_total, sq, sums, st);
}

int launch_sketch_query_f64(const void* q, int q_dtype, int units, int G, int d, const qjl_sketch_t& sk,
                            int m_total, double* sq, cudaStream_t st) {
  return launch_sq_o<double>(q, q_dtype, units, G, d, sk, m_total, m_total, sq, nullptr, st);
}

// ---------------------------------------------------------------------------
// Generic score estimator (kvcache.py:311-329 + estimator.py:149-170), one
// thread per cached token; the unit's query sketches sit in smem and every
// thread walks its own packed bits (smem reads are warp-broadcasts).
//   logit = sqrt(pi/2)/m_in  * nu_in  * (2*sum_{set} Sq_in  - sum Sq_in)
//         + sqrt(pi/2)/m_out * nu_out * (2*sum_{set} Sq_out - sum Sq_out)
// ---------------------------------------------------------------------------
template <int GMAX>
__device__ __forceinline__ void set_sums(const uint8_t* __restrict__ bits, int m,
                                         const float* __restrict__ sq_sm, int m_total, int G,
                                         float* acc) {
  const uint32_t* w32 = reinterpret_cast<const uint32_t*>(bits);
  for (int w = 0; w < m / 32; ++w) {
    const uint32_t word = w32[w];
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const uint32_t mask = 0u - ((word >> j) & 1u);
#pragma unroll
      for (int g = 0; g < GMAX; ++g)
        if (g < G) acc[g] += __uint_as_float(mask & __float_as_uint(sq_sm[g * m_total + 32 * w + j]));
    }
  }
}

template <int GMAX>
__global__ void __launch_bounds__(128) k_scores_simt(qjl_key_cache_t kc, int64_t n, int G,
                                                     const float* __restrict__ sq,
                                                     const float* __restrict__ sums,
                                                     float* __restrict__ logits) {
  extern __shared__ float sqs[];  // [G][m_total] + [G][2]
  const int u = blockIdx.y;
  const int m_in = kc.m_in, m_out = kc.m_out, m_total = m_in + m_out;
  for (int i = threadIdx.x; i < G * m_total; i += blockDim.x) sqs[i] = sq[(int64_t)u * G * m_total + i];
  for (int i = threadIdx.x; i < 2 * G; i += blockDim.x) sqs[G * m_total + i] = sums[(int64_t)u * G * 2 + i];
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  float a_in[GMAX], a_out[GMAX];
#pragma unroll
  for (int g = 0; g < GMAX; ++g) { a_in[g] = 0.f; a_out[g] = 0.f; }
  set_sums<GMAX>(kc.bits_in + row_off(u, t, m_in / 8, kc.capacity, kc.tile_stride), m_in, sqs, m_total, G, a_in);
  if (m_out > 0)
    set_sums<GMAX>(kc.bits_out + row_off(u, t, m_out / 8, kc.capacity, kc.tile_stride), m_out, sqs + m_in, m_total,
                   G, a_out);
  const int64_t no = row_off(u, t, 2, kc.capacity, kc.tile_stride);
  const float nu_in = f16_bits_to_f32(*reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(kc.norm_in) + no));
  const float nu_out =
      m_out > 0 ? f16_bits_to_f32(*reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(kc.norm_out) + no))
                : 0.f;
  const float c_in = m_in > 0 ? kEstimatorScale / (float)m_in : 0.f;
  const float c_out = m_out > 0 ? kEstimatorScale / (float)m_out : 0.f;
#pragma unroll
  for (int g = 0; g < GMAX; ++g) {
    if (g >= G) break;
    const float* sm2 = sqs + G * m_total + 2 * g;
    float lg = c_in * nu_in * (2.f * a_in[g] - sm2[0]);
    if (m_out > 0) lg += c_out * nu_out * (2.f * a_out[g] - sm2[1]);
    logits[((int64_t)u * G + g) * n + t] = lg;
  }
}

int launch_scores_simt(const qjl_key_cache_t& kc, int64_t n, int G, const float* sq,
                       const float* sums, float* logits, cudaStream_t st) {
  const int m_total = kc.m_in + kc.m_out;
  const size_t smem = ((size_t)G * m_total + 2 * G) * sizeof(float);
  dim3 grid((unsigned)((n + 127) / 128), kc.units);
#define QJL_SC(GM)                                                                              \
  if (G <= GM) {                                                                                \
    cudaFuncSetAttribute(k_scores_simt<GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                         (int)smem);                                                            \
    k_scores_simt<GM><<<grid, 128, smem, st>>>(kc, n, G, sq, sums, logits);                     \
    QJL_LAUNCH_CHECK("scores_simt");                                                            \
    return QJL_OK;                                                                              \
  }
  QJL_SC(1)
  QJL_SC(2)
  QJL_SC(4)
  QJL_SC(8)
  QJL_SC(16)
#undef QJL_SC
  set_error("scores: at most 16 query heads per unit (got %d)", G);
  return QJL_ERR_UNSUPPORTED;
}

// ---------------------------------------------------------------------------
// softmax in fp64 (kvcache.py:38-44) of logits * inv_T; one CTA per row.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_softmax_f64(const float* __restrict__ logits, int64_t n,
                                                     double inv_t, double* __restrict__ w) {
  __shared__ double red[8];
  const float* L = logits + (int64_t)blockIdx.x * n;
  double* W = w + (int64_t)blockIdx.x * n;
  double mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, (double)L[i] * inv_t);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmax(mx, red[i]);
  __syncthreads();
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double e = exp((double)L[i] * inv_t - mx);
    W[i] = e;
    s += e;
  }
  s = warp_sum_f64(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double tot = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += red[i];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) W[i] = W[i] / tot;
}

int launch_softmax_f64(const float* logits, int64_t rows, int64_t n, double inv_t, double* w,
                       cudaStream_t st) {
  k_softmax_f64<<<(unsigned)rows, 256, 0, st>>>(logits, n, inv_t, w);
  QJL_LAUNCH_CHECK("softmax_f64");
  return QJL_OK;
}

}  // namespace qjl

namespace qjl {
// ---------------------------------------------------------------------------
// packed_sign_dot_batch (estimator.py:149-170) on device, fp64 accumulation
// like the reference: out[g][i] = 2 * sum_{set bits of row i} values[g] - sum(values[g]).
// One thread per row; values staged in smem (broadcast reads).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_sign_dot_batch(const uint8_t* __restrict__ bits, int64_t n,
                                                        int m, int64_t row_bytes,
                                                        const double* __restrict__ values, int G,
                                                        double* __restrict__ out) {
  extern __shared__ double vs[];  // [G][m] + [G] totals
  for (int i = threadIdx.x; i < G * m; i += blockDim.x) vs[i] = values[i];
  __syncthreads();
  if (threadIdx.x < G) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s += vs[threadIdx.x * m + j];
    vs[G * m + threadIdx.x] = s;
  }
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t* w32 = reinterpret_cast<const uint32_t*>(bits + r * row_bytes);
  for (int g = 0; g < G; ++g) {
    double acc = 0.0;
    for (int w = 0; w < m / 32; ++w) {
      const uint32_t word = w32[w];
      for (int j = 0; j < 32; ++j)
        if ((word >> j) & 1u) acc += vs[g * m + 32 * w + j];
    }
    out[(int64_t)g * n + r] = 2.0 * acc - vs[G * m + g];
  }
}

int launch_sign_dot_batch(const uint8_t* bits, int64_t n, int m, int64_t row_bytes,
                          const double* values, int G, double* out, cudaStream_t st) {
  const size_t smem = ((size_t)G * m + G) * sizeof(double);
  cudaFuncSetAttribute(k_sign_dot_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_sign_dot_batch<<<(unsigned)((n + 127) / 128), 128, smem, st>>>(bits, n, m, row_bytes, values, G, out);
  QJL_LAUNCH_CHECK("sign_dot_batch");
  return QJL_OK;
}
}  // namespace qjl
