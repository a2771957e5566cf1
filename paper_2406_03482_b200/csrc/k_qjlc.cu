// QJLC cache records (write_cache / read_cache, pkg/src/qjl/kvcache.py:389-520) <->
// the device cache layout.  One record per token, little-endian, in append order
// (kvcache.py:430-436, :472):
//
//   [inlier sign words 8*ceil(m_in/64) B][inlier norm f16][outlier sign words
//    8*ceil(m_out/64) B][outlier norm f16][d codes, 1 B each][zero f32][scale f32]
//
// The sign bytes are the device bytes (LSB-first) plus zero padding to
// whole u64 words; norms are already f16 on the device (the reference's storage
// policy, kvcache.py:490); values must be in the reference's own format (U8 layout,
// one group per token, f32 zero/scale).  Pure byte movement, HBM-bound: each CTA
// stages T whole records in shared memory, so both the field-wise side (device
// arrays, contiguous across rows) and the record side move with coalesced vector
// accesses.
#include "common.cuh"
#include "kernels.h"

namespace qjl {
namespace {

struct Rec {
  int R;                      // record bytes
  int wib, wob;               // file bytes of the inlier / outlier sign words
  int mib, mob;               // device bytes per row (m_dev / 8)
  int mfi, mfo;               // logical widths in the file header
  int d;
  int o_ni, o_bo, o_no, o_c, o_z, o_s;
  uint32_t dv_wi, dv_ho, dv_wc;   // magic reciprocals: / (wib/4), / (wob/2), / (d/4)
};

// floor(i / D) for i < 2^16, D < 2^16 with M = floor(2^32 / D) + 1
__host__ __device__ __forceinline__ uint32_t magic_of(uint32_t D) {
  return (uint32_t)((((uint64_t)1) << 32) / D + 1);
}
__device__ __forceinline__ int qdiv(int i, uint32_t M) { return (int)__umulhi((uint32_t)i, M); }

// bits of a 32/16-bit file word at bit position `pos` that lie below the logical width
__device__ __forceinline__ uint32_t mask_bits(int valid, int width) {
  return valid >= width ? (width == 32 ? 0xFFFFFFFFu : 0xFFFFu) : (valid <= 0 ? 0u : ((1u << valid) - 1u));
}

template <bool AL>
__device__ __forceinline__ void st32(uint8_t* p, uint32_t v) {
  if (AL) {
    *reinterpret_cast<uint32_t*>(p) = v;
  } else {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
  }
}
template <bool AL>
__device__ __forceinline__ uint32_t ld32(const uint8_t* p) {
  if (AL) return *reinterpret_cast<const uint32_t*>(p);
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
template <bool AL>
__device__ __forceinline__ void st16(uint8_t* p, uint32_t v) {
  if (AL) {
    *reinterpret_cast<uint16_t*>(p) = (uint16_t)v;
  } else {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8);
  }
}
template <bool AL>
__device__ __forceinline__ uint32_t ld16(const uint8_t* p) {
  if (AL) return *reinterpret_cast<const uint16_t*>(p);
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8);
}

// contiguous span copy between shared memory and global memory (16 B vectors when the
// global side is 16 B aligned; the shared side is always 16 B aligned)
template <bool TO_GLOBAL>
__device__ __forceinline__ void span_copy(uint8_t* g, uint8_t* s, int L) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  int head = 0;
  if (((uintptr_t)g & 15) == 0) {
    const int nv = L >> 4;
    for (int i = tid; i < nv; i += nthr) {
      if (TO_GLOBAL)
        reinterpret_cast<uint4*>(g)[i] = reinterpret_cast<const uint4*>(s)[i];
      else
        reinterpret_cast<uint4*>(s)[i] = __ldg(reinterpret_cast<const uint4*>(g) + i);
    }
    head = nv << 4;
  } else if (((uintptr_t)g & 3) == 0) {
    const int nv = L >> 2;
    for (int i = tid; i < nv; i += nthr) {
      if (TO_GLOBAL)
        reinterpret_cast<uint32_t*>(g)[i] = reinterpret_cast<const uint32_t*>(s)[i];
      else
        reinterpret_cast<uint32_t*>(s)[i] = __ldg(reinterpret_cast<const uint32_t*>(g) + i);
    }
    head = nv << 2;
  }
  for (int i = head + tid; i < L; i += nthr) {
    if (TO_GLOBAL) g[i] = s[i];
    else s[i] = g[i];
  }
}

// AL: record size R is a multiple of 4 (d % 4 == 0), so every field except the
// outlier words / norm (offset 2 mod 4) is 4-byte aligned in shared memory.
template <bool AL>
__global__ void __launch_bounds__(256) k_qjlc_export(qjl_key_cache_t kc, qjl_value_cache_t vc, Rec F,
                                                     int64_t row0, int64_t n, uint8_t* __restrict__ out,
                                                     int64_t ustride, int T) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int u = blockIdx.y, tid = threadIdx.x, nthr = blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * T;
  const int nt = (int)(n - t0 < (int64_t)T ? n - t0 : (int64_t)T);
  const int64_t r0 = (int64_t)u * kc.capacity + row0 + t0;      // first key cache row
  const int64_t v0 = (int64_t)u * vc.capacity + row0 + t0;      // first value cache row
  // inlier sign words (device rows are contiguous: nt * mib bytes)
  if (F.wib) {
    const int fw = F.wib >> 2, dw = F.mib >> 2;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(kc.bits_in + r0 * F.mib);
    for (int i = tid; i < nt * fw; i += nthr) {
      const int t = qdiv(i, F.dv_wi), w = i - t * fw;
      uint32_t v = w < dw ? __ldg(src + t * dw + w) : 0u;
      v &= mask_bits(F.mfi - 32 * w, 32);
      st32<AL>(sm + t * F.R + 4 * w, v);
    }
  }
  // outlier sign words as 16-bit halves (record offset wib + 2)
  if (F.wob) {
    const int fh = F.wob >> 1, dh = F.mob >> 1;
    const uint16_t* src = reinterpret_cast<const uint16_t*>(kc.bits_out + r0 * F.mob);
    for (int i = tid; i < nt * fh; i += nthr) {
      const int t = qdiv(i, F.dv_ho), w = i - t * fh;
      uint32_t v = w < dh ? (uint32_t)__ldg(src + t * dh + w) : 0u;
      v &= mask_bits(F.mfo - 16 * w, 16);
      st16<AL>(sm + t * F.R + F.o_bo + 2 * w, v);
    }
  }
  // norms (0.0 for an empty side, EMPTY_KEY), zero / scale
  for (int t = tid; t < nt; t += nthr) {
    uint8_t* rec = sm + t * F.R;
    st16<AL>(rec + F.o_ni, F.mfi ? (uint32_t)kc.norm_in[r0 + t] : 0u);
    st16<AL>(rec + F.o_no, F.mfo ? (uint32_t)kc.norm_out[r0 + t] : 0u);
    st32<AL>(rec + F.o_z, __float_as_uint(reinterpret_cast<const float*>(vc.zero)[v0 + t]));
    st32<AL>(rec + F.o_s, __float_as_uint(reinterpret_cast<const float*>(vc.scale)[v0 + t]));
  }
  // value codes, one byte each
  const uint8_t* codes = reinterpret_cast<const uint8_t*>(vc.codes) + v0 * F.d;
  if (AL) {
    const int cw = F.d >> 2;
    for (int i = tid; i < nt * cw; i += nthr) {
      const int t = qdiv(i, F.dv_wc), w = i - t * cw;
      st32<true>(sm + t * F.R + F.o_c + 4 * w, __ldg(reinterpret_cast<const uint32_t*>(codes) + i));
    }
  } else {
    for (int i = tid; i < nt * F.d; i += nthr) {
      const int t = i / F.d, c = i - t * F.d;
      sm[t * F.R + F.o_c + c] = codes[i];
    }
  }
  __syncthreads();
  span_copy<true>(out + (int64_t)u * ustride + t0 * F.R, sm, nt * F.R);
}

template <bool AL>
__global__ void __launch_bounds__(256) k_qjlc_import(const uint8_t* __restrict__ in, int64_t ustride, Rec F,
                                                     int64_t n, qjl_key_cache_t kc, qjl_value_cache_t vc,
                                                     int has_values, int64_t row0, int T) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int u = blockIdx.y, tid = threadIdx.x, nthr = blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * T;
  const int nt = (int)(n - t0 < (int64_t)T ? n - t0 : (int64_t)T);
  const int64_t r0 = (int64_t)u * kc.capacity + row0 + t0;
  span_copy<false>(const_cast<uint8_t*>(in) + (int64_t)u * ustride + t0 * F.R, sm, nt * F.R);
  __syncthreads();
  if (F.mib) {
    const int dw = F.mib >> 2;
    uint32_t* dst = reinterpret_cast<uint32_t*>(kc.bits_in + r0 * F.mib);
    for (int i = tid; i < nt * dw; i += nthr) {
      const int t = i / dw, w = i - t * dw;     // dw is a power of two in practice
      // device words past the file's logical width are cleared (read_cache keeps only m bits)
      uint32_t v = 4 * w < F.wib ? ld32<AL>(sm + t * F.R + 4 * w) : 0u;
      dst[i] = v & mask_bits(F.mfi - 32 * w, 32);
    }
    for (int t = tid; t < nt; t += nthr) kc.norm_in[r0 + t] = (uint16_t)ld16<AL>(sm + t * F.R + F.o_ni);
  }
  if (F.mob) {
    const int dh = F.mob >> 1;
    uint16_t* dst = reinterpret_cast<uint16_t*>(kc.bits_out + r0 * F.mob);
    for (int i = tid; i < nt * dh; i += nthr) {
      const int t = i / dh, w = i - t * dh;
      uint32_t v = 2 * w < F.wob ? ld16<AL>(sm + t * F.R + F.o_bo + 2 * w) : 0u;
      dst[i] = (uint16_t)(v & mask_bits(F.mfo - 16 * w, 16));
    }
    for (int t = tid; t < nt; t += nthr) kc.norm_out[r0 + t] = (uint16_t)ld16<AL>(sm + t * F.R + F.o_no);
  }
  if (!has_values) return;
  const int64_t v0 = (int64_t)u * vc.capacity + row0 + t0;
  uint8_t* codes = reinterpret_cast<uint8_t*>(vc.codes) + v0 * F.d;
  if (AL) {
    const int cw = F.d >> 2;
    for (int i = tid; i < nt * cw; i += nthr) {
      const int t = qdiv(i, F.dv_wc), w = i - t * cw;
      reinterpret_cast<uint32_t*>(codes)[i] = ld32<true>(sm + t * F.R + F.o_c + 4 * w);
    }
  } else {
    for (int i = tid; i < nt * F.d; i += nthr) {
      const int t = i / F.d, c = i - t * F.d;
      codes[i] = sm[t * F.R + F.o_c + c];
    }
  }
  for (int t = tid; t < nt; t += nthr) {
    reinterpret_cast<float*>(vc.zero)[v0 + t] = __uint_as_float(ld32<AL>(sm + t * F.R + F.o_z));
    reinterpret_cast<float*>(vc.scale)[v0 + t] = __uint_as_float(ld32<AL>(sm + t * F.R + F.o_s));
  }
}

}  // namespace

int64_t qjlc_record_bytes(int d, int m_in_file, int m_out_file) {
  return 8LL * ((m_in_file + 63) / 64) + 2 + 8LL * ((m_out_file + 63) / 64) + 2 + d + 4 + 4;
}

static Rec make_rec(int d, int mfi, int mfo, int m_dev_in, int m_dev_out) {
  Rec F;
  F.d = d;
  F.mfi = mfi;
  F.mfo = mfo;
  F.wib = 8 * ((mfi + 63) / 64);
  F.wob = 8 * ((mfo + 63) / 64);
  F.mib = m_dev_in / 8;
  F.mob = m_dev_out / 8;
  F.o_ni = F.wib;
  F.o_bo = F.wib + 2;
  F.o_no = F.o_bo + F.wob;
  F.o_c = F.o_no + 2;
  F.o_z = F.o_c + d;
  F.o_s = F.o_z + 4;
  F.R = F.o_s + 4;
  F.dv_wi = F.wib ? magic_of(F.wib / 4) : 0;
  F.dv_ho = F.wob ? magic_of(F.wob / 2) : 0;
  F.dv_wc = magic_of(d / 4 > 0 ? d / 4 : 1);
  return F;
}

// tokens per CTA: whole records in <= 48 KB of shared memory, a multiple of 4 so the
// global span of every CTA but a unit's last starts 16 B aligned when ustride is
static int tokens_per_cta(int R) {
  int T = (48 * 1024 / R) & ~3;
  if (T > 128) T = 128;
  if (T < 4) T = 4;
  return T;
}

int launch_qjlc_export(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int mfi, int mfo,
                       int64_t row0, int64_t n, uint8_t* out, int64_t ustride, cudaStream_t st) {
  const Rec F = make_rec(kc.d, mfi, mfo, kc.m_in, kc.m_out);
  const int T = tokens_per_cta(F.R);
  const size_t smem = (size_t)T * F.R;
  dim3 grid((unsigned)((n + T - 1) / T), kc.units);
  if (F.R % 4 == 0) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_qjlc_export<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_qjlc_export<true><<<grid, 256, smem, st>>>(kc, vc, F, row0, n, out, ustride, T);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_qjlc_export<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_qjlc_export<false><<<grid, 256, smem, st>>>(kc, vc, F, row0, n, out, ustride, T);
  }
  QJL_LAUNCH_CHECK("qjlc_export");
  return QJL_OK;
}

int launch_qjlc_import(const uint8_t* in, int64_t ustride, int mfi, int mfo, int64_t n,
                       const qjl_key_cache_t& kc, const qjl_value_cache_t* vc, int64_t row0,
                       cudaStream_t st) {
  const Rec F = make_rec(kc.d, mfi, mfo, kc.m_in, kc.m_out);
  const int T = tokens_per_cta(F.R);
  const size_t smem = (size_t)T * F.R;
  dim3 grid((unsigned)((n + T - 1) / T), kc.units);
  qjl_value_cache_t v{};
  if (vc) v = *vc;
  if (F.R % 4 == 0) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_qjlc_import<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_qjlc_import<true><<<grid, 256, smem, st>>>(in, ustride, F, n, kc, v, vc != nullptr, row0, T);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_qjlc_import<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_qjlc_import<false><<<grid, 256, smem, st>>>(in, ustride, F, n, kc, v, vc != nullptr, row0, T);
  }
  QJL_LAUNCH_CHECK("qjlc_import");
  return QJL_OK;
}

}  // namespace qjl
