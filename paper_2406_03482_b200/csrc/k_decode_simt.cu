// Generic fused decode (scores -> online softmax -> weights @ dequantized V) for the
// reference's own value format (U8 codes, fp32 zero/scale, any bit width and group),
// rows-layout caches, any G <= 8, any m % 32 == 0 -- the path behind the drop-in
// `quantized_decode` (attention.py:56-71) for shapes outside the tensor-core envelope.
// Flash-decoding split over tokens with an fp32 (m, l, acc) merge.
#include "common.cuh"
#include "kernels.h"

namespace qjl {

constexpr int kDTile = 128;  // tokens per tile == threads per CTA

template <int GMAX>
__device__ __forceinline__ void set_sums_dec(const uint8_t* __restrict__ bits, int m,
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

__device__ __forceinline__ float load_value(const qjl_value_cache_t& vc, int64_t row, int dim) {
  const int G = vc.d / vc.group;
  const int grp = dim / vc.group;
  const float z = reinterpret_cast<const float*>(vc.zero)[row * G + grp];
  const float s = reinterpret_cast<const float*>(vc.scale)[row * G + grp];
  const float c = (float)reinterpret_cast<const uint8_t*>(vc.codes)[row * vc.d + dim];
  return fmaf(c, s, z);
}

// ws layout per (unit, split, g): m, l, acc[d]
template <int GMAX>
__global__ void __launch_bounds__(kDTile) k_decode_simt(qjl_key_cache_t kc, qjl_value_cache_t vc,
                                                        int64_t n, int G, int64_t chunk,
                                                        const float* __restrict__ sq,
                                                        const float* __restrict__ sums, float inv_t,
                                                        float* __restrict__ logits, float* __restrict__ ws) {
  extern __shared__ float sm[];
  const int m_in = kc.m_in, m_out = kc.m_out, m_total = m_in + m_out, d = vc.d;
  float* sqs = sm;                              // [G][m_total]
  float* ssum = sqs + G * m_total;              // [G][2]
  float* p = ssum + 2 * G;                      // [G][kDTile]
  float* red = p + G * kDTile;                  // [G][4]
  const int u = blockIdx.y, split = blockIdx.x, nsplit = gridDim.x;
  for (int i = threadIdx.x; i < G * m_total; i += blockDim.x) sqs[i] = sq[(int64_t)u * G * m_total + i];
  for (int i = threadIdx.x; i < 2 * G; i += blockDim.x) ssum[i] = sums[(int64_t)u * G * 2 + i];
  const float c_in = m_in > 0 ? kEstimatorScale / (float)m_in : 0.f;
  const float c_out = m_out > 0 ? kEstimatorScale / (float)m_out : 0.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  float m_run[GMAX], l_part[GMAX], acc[GMAX];
#pragma unroll
  for (int g = 0; g < GMAX; ++g) { m_run[g] = -INFINITY; l_part[g] = 0.f; acc[g] = 0.f; }
  const int64_t t_begin = (int64_t)split * chunk;
  const int64_t t_end = t_begin + chunk < n ? t_begin + chunk : n;
  __syncthreads();

  for (int64_t t0 = t_begin; t0 < t_end; t0 += kDTile) {
    const int64_t t = t0 + threadIdx.x;
    const bool valid = t < t_end;
    float lg[GMAX];
#pragma unroll
    for (int g = 0; g < GMAX; ++g) lg[g] = -INFINITY;
    if (valid) {
      const int64_t row = (int64_t)u * kc.capacity + t;
      float a_in[GMAX], a_out[GMAX];
#pragma unroll
      for (int g = 0; g < GMAX; ++g) { a_in[g] = 0.f; a_out[g] = 0.f; }
      set_sums_dec<GMAX>(kc.bits_in + row * (m_in / 8), m_in, sqs, m_total, G, a_in);
      if (m_out > 0) set_sums_dec<GMAX>(kc.bits_out + row * (m_out / 8), m_out, sqs + m_in, m_total, G, a_out);
      const float nu_in = f16_bits_to_f32(kc.norm_in[row]);
      const float nu_out = m_out > 0 ? f16_bits_to_f32(kc.norm_out[row]) : 0.f;
#pragma unroll
      for (int g = 0; g < GMAX; ++g) {
        if (g < G) {
          float v = c_in * nu_in * (2.f * a_in[g] - ssum[2 * g]);
          if (m_out > 0) v += c_out * nu_out * (2.f * a_out[g] - ssum[2 * g + 1]);
          lg[g] = v * inv_t;
          if (logits) logits[((int64_t)u * G + g) * n + t] = lg[g];
        }
      }
    }
    // tile max per query head
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      if (g < G) {
        const float wm = warp_max(lg[g]);
        if (lane == 0) red[g * 4 + warp] = wm;
      }
    }
    __syncthreads();
    float alpha[GMAX];
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      alpha[g] = 1.f;
      if (g < G) {
        const float tm = fmaxf(fmaxf(red[g * 4], red[g * 4 + 1]), fmaxf(red[g * 4 + 2], red[g * 4 + 3]));
        const float m_new = fmaxf(m_run[g], tm);
        alpha[g] = (m_run[g] == -INFINITY) ? 0.f : expf(m_run[g] - m_new);
        m_run[g] = m_new;
        const float pv = valid ? expf(lg[g] - m_new) : 0.f;
        p[g * kDTile + threadIdx.x] = pv;
        l_part[g] = l_part[g] * alpha[g] + pv;
      }
    }
    __syncthreads();
    // PV: thread == output dim (d <= kDTile)
    if (threadIdx.x < d) {
#pragma unroll
      for (int g = 0; g < GMAX; ++g) acc[g] *= alpha[g];
      const int nt = (int)(t_end - t0 < kDTile ? t_end - t0 : kDTile);
      for (int j = 0; j < nt; ++j) {
        const float v = load_value(vc, (int64_t)u * vc.capacity + t0 + j, threadIdx.x);
#pragma unroll
        for (int g = 0; g < GMAX; ++g)
          if (g < G) acc[g] = fmaf(p[g * kDTile + j], v, acc[g]);
      }
    }
    __syncthreads();
  }
  // reduce l over the CTA
#pragma unroll
  for (int g = 0; g < GMAX; ++g) {
    if (g < G) {
      const float s = warp_sum(l_part[g]);
      if (lane == 0) red[g * 4 + warp] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int g = 0; g < GMAX; ++g) {
    if (g >= G) break;
    float* W = ws + (((int64_t)u * nsplit + split) * G + g) * (d + 2);
    if (threadIdx.x == 0) {
      W[0] = m_run[g];
      W[1] = red[g * 4] + red[g * 4 + 1] + red[g * 4 + 2] + red[g * 4 + 3];
    }
    if (threadIdx.x < d) W[2 + threadIdx.x] = acc[g];
  }
}

// Merge split partials: out = sum_s acc_s e^{m_s - M} / sum_s l_s e^{m_s - M}.
__global__ void k_decode_merge(const float* __restrict__ ws, int nsplit, int G, int d,
                               float* __restrict__ out, float* __restrict__ lse) {
  const int ug = blockIdx.x;
  const int u = ug / G, g = ug % G;
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, ws[(((int64_t)u * nsplit + s) * G + g) * (d + 2)]);
  float L = 0.f, a = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float* W = ws + (((int64_t)u * nsplit + s) * G + g) * (d + 2);
    if (W[0] == -INFINITY) continue;
    const float f = expf(W[0] - M);
    L += W[1] * f;
    if (threadIdx.x < d) a += W[2 + threadIdx.x] * f;
  }
  if (threadIdx.x < d) out[(int64_t)ug * d + threadIdx.x] = a / L;
  if (lse && threadIdx.x == 0) lse[ug] = M + logf(L);
}

void decode_simt_plan(int units, int64_t n, int* nsplit, int64_t* chunk) {
  const int target = 2 * device_sm_count();
  int s = (target + units - 1) / units;
  int64_t max_s = (n + kDTile - 1) / kDTile;
  if (s > max_s) s = (int)max_s;
  if (s < 1) s = 1;
  int64_t c = (n + s - 1) / s;
  c = (c + kDTile - 1) / kDTile * kDTile;
  *chunk = c;
  *nsplit = (int)((n + c - 1) / c);
}

size_t decode_simt_workspace(int units, int64_t n, int G, int d, int m_total) {
  int ns;
  int64_t ch;
  decode_simt_plan(units, n, &ns, &ch);
  return ((size_t)units * ns * G * (d + 2) + (size_t)units * G * (m_total + 2)) * sizeof(float);
}

int launch_decode_simt(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, int G,
                       const float* sq, const float* sums, float inv_t, float* out, float* lse,
                       float* logits, float* ws, cudaStream_t st) {
  int nsplit;
  int64_t chunk;
  decode_simt_plan(kc.units, n, &nsplit, &chunk);
  const int m_total = kc.m_in + kc.m_out;
  const size_t smem = ((size_t)G * m_total + 2 * G + (size_t)G * kDTile + 4 * G) * sizeof(float);
  dim3 grid(nsplit, kc.units);
#define QJL_DS(GM)                                                                          \
  if (G <= GM) {                                                                            \
    cudaFuncSetAttribute(k_decode_simt<GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                         (int)smem);                                                        \
    k_decode_simt<GM><<<grid, kDTile, smem, st>>>(kc, vc, n, G, chunk, sq, sums, inv_t, logits, ws); \
    QJL_LAUNCH_CHECK("decode_simt");                                                        \
    k_decode_merge<<<kc.units * G, 128, 0, st>>>(ws, nsplit, G, vc.d, out, lse);            \
    QJL_LAUNCH_CHECK("decode_merge");                                                       \
    return QJL_OK;                                                                          \
  }
  QJL_DS(1)
  QJL_DS(2)
  QJL_DS(4)
  QJL_DS(8)
#undef QJL_DS
  set_error("decode: at most 8 query heads per unit on the generic path (got %d)", G);
  return QJL_ERR_UNSUPPORTED;
}

}  // namespace qjl
