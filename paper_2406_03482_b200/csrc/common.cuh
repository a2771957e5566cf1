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
// 2-bit codes of a d=128 token live in 8 u32 words.  Word w holds the 16 dims
// {16*mt + w + 8*hh : mt in 0..7, hh in 0..1} at code slot p = 2*mt + hh (bits
// 2p..2p+1).  This is the A-fragment order of mma.m16n8k16 with one m-tile per
// 16 dims: lane-row g of every m-tile reads word g only.
__host__ __device__ __forceinline__ void p2_slot(int dim, int* word, int* slot) {
  int mt = dim >> 4, r = dim & 15;
  *word = r & 7;
  *slot = 2 * mt + (r >> 3);
}

}  // namespace qjl
