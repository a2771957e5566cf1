// Shared device/host helpers for the QJL B200 kernels (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qjl_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "qjl_b200 is written for sm_100a (B200) only"
#endif

namespace qjl {

constexpr float kEstimatorScale = 1.2533141373155002512f;  // sqrt(pi/2), estimator.py:27

// ---------------------------------------------------------------- host side
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
int device_sm_count();
// benchmark timing hook (api.cu): no-ops unless qjl_timing_enable(1)
void timing_begin(cudaStream_t st);
void timing_end(cudaStream_t st);
bool timing_enabled();

#define QJL_CHECK_ARG(cond, ...)        \
  do {                                  \
    if (!(cond)) {                      \
      ::qjl::set_error(__VA_ARGS__);    \
      return QJL_ERR_ARG;               \
    }                                   \
  } while (0)

#define QJL_LAUNCH_CHECK(what)                                            \
  do {                                                                    \
    cudaError_t e_ = cudaGetLastError();                                  \
    if (e_ != cudaSuccess) return ::qjl::cuda_status(e_, what);           \
  } while (0)

inline size_t dtype_size(int dt) {
  switch (dt) {
    case QJL_F32: return 4;
    case QJL_F16: return 2;
    case QJL_BF16: return 2;
    case QJL_F64: return 8;
  }
  return 0;
}

// -------------------------------------------------------------- device side
template <int DT>
struct Elem;
template <> struct Elem<QJL_F32> { using T = float; };
template <> struct Elem<QJL_F16> { using T = __half; };
template <> struct Elem<QJL_BF16> { using T = __nv_bfloat16; };
template <> struct Elem<QJL_F64> { using T = double; };

__device__ __forceinline__ double to_f64(float x) { return (double)x; }
__device__ __forceinline__ double to_f64(double x) { return x; }
__device__ __forceinline__ double to_f64(__half x) { return (double)__half2float(x); }
__device__ __forceinline__ double to_f64(__nv_bfloat16 x) { return (double)__bfloat162float(x); }
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(double x) { return (float)x; }
__device__ __forceinline__ float to_f32(__half x) { return __half2float(x); }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f64(double x);
template <> __device__ __forceinline__ double from_f64<double>(double x) { return x; }
template <> __device__ __forceinline__ float from_f64<float>(double x) { return (float)x; }
template <> __device__ __forceinline__ __half from_f64<__half>(double x) { return __double2half(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double x) {
  return __double2bfloat16(x);
}

__device__ __forceinline__ uint16_t f32_to_f16_bits(float x) {
  return __half_as_ushort(__float2half_rn(x));
}
__device__ __forceinline__ float f16_bits_to_f32(uint16_t b) {
  return __half2float(__ushort_as_half(b));
}
// fp64 -> fp16 with a single rounding (matches numpy float64 -> float16).
__device__ __forceinline__ uint16_t f64_to_f16_bits(double x) {
  return __half_as_ushort(__double2half(x));
}

// NaN as numpy's float16 NaN (0x7E00) whatever payload produced it (norms of NaN keys)
__device__ __forceinline__ uint16_t f16_canon(uint16_t v) {
  return ((v & 0x7C00u) == 0x7C00u && (v & 0x3FFu)) ? (uint16_t)0x7E00u : v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------- P2 value layout
// 2-bit codes, group 32, d = 128: 32 bytes per token, interleaved inside each
// 128-token tile so that one u32 word holds 4 tokens x 4 dims -- the A operand
// register of the PV IMMA (mma.m16n8k32 u8) after a single mask, `w & (3 << 2s)`
// per byte.  For row t of a unit and dim d:
//   tile = t >> 7, slice = (t >> 5) & 3 (the warp that consumes it),
//   j = t & 7 (k-block = tokens j, j+8, j+16, j+24 of the slice), i = (t >> 3) & 3 (byte),
//   MT = d >> 4 (m-tile), g = d & 7 (fragment row), r = (d >> 3) & 1, k = MT >> 1,
//   s = 2 * (MT & 1) + r (2-bit slot inside the byte)
//   word = tile * 1024 + slice * 256 + (g * 8 + (j ^ ((g & 1) << 2))) * 4 + k
// The j ^ 4 swizzle on odd rows makes the per-lane 16-byte loads bank-conflict free.
__host__ __device__ __forceinline__ void p2_pos(int64_t t, int d, int64_t* byte, int* shift) {
  const int64_t tile = t >> 7;
  const int slice = (int)(t >> 5) & 3, j = (int)t & 7, i = (int)(t >> 3) & 3;
  const int MT = d >> 4, g = d & 7, r = (d >> 3) & 1, k = MT >> 1, s = 2 * (MT & 1) + r;
  const int64_t word = tile * 1024 + slice * 256 + (g * 8 + (j ^ ((g & 1) << 2))) * 4 + k;
  *byte = word * 4 + i;
  *shift = 2 * s;
}

// P2T value-code layout (tcgen05 decode): one u32 word = 4 consecutive tokens (bytes)
// x 4 dims (2-bit slots), so one mask per word yields the u8 A-operand column of a
// TMEM-resident PV operand (row = dim, weight 4^(d % 4) folded out per row):
//   byte = tile * 4096 + (d >> 2) * 128 + ((t & 127) >> 2) * 4 + (t & 3), shift = 2 * (d & 3)
__host__ __device__ __forceinline__ void p2t_pos(int64_t t, int d, int64_t* byte, int* shift) {
  *byte = (t >> 7) * 4096 + (int64_t)(d >> 2) * 128 + ((t & 127) >> 2) * 4 + (t & 3);
  *shift = 2 * (d & 3);
}

}  // namespace qjl
