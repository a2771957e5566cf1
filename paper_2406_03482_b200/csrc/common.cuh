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

// ------------------------------------------------------------- row addressing
// Byte offset of row `row` of unit `u` in a cache array with `rb` bytes per row
// (qjl_b200.h, tile_stride): rows layout [units][capacity][rb] when ts == 0, else
// tile-major records -- unit u's 128-row tile j starts (u * capacity/128 + j) * ts in.
__host__ __device__ __forceinline__ int64_t row_off(int64_t u, int64_t row, int64_t rb, int64_t cap, int64_t ts) {
  return ts ? (u * (cap >> 7) + (row >> 7)) * ts + (row & 127) * rb : (u * cap + row) * rb;
}
// Byte offset of the 128-token tile holding row `row` of an array whose tiles are
// `tile_bytes` long in the rows layout (e.g. 4096 for P2T codes).
__host__ __device__ __forceinline__ int64_t tile_off(int64_t u, int64_t row, int64_t tile_bytes, int64_t cap,
                                                     int64_t ts) {
  return (u * (cap >> 7) + (row >> 7)) * (ts ? ts : tile_bytes);
}

// P2T value-code layout (tcgen05 decode): one u32 word = 4 consecutive tokens (bytes)
// x 4 dims (2-bit slots), so one mask per word yields the u8 A-operand column of a
// TMEM-resident PV operand (row = dim, weight 4^(d % 4) folded out per row).  Row
// dq = d / 4 of a tile holds 128 bytes = 8 chunks of 16 tokens; chunk j is stored at chunk
// position j ^ (dq % 4), so the rows of any 8 consecutive threads (two dim quads, one phase
// of a 128-bit shared load) sit in different bank groups.
// In-tile byte of (token t, dim d), and the bit shift of its 2-bit slot:
//   byte = dq * 128 + ((tw / 4) ^ (dq % 4)) * 16 + (tw % 4) * 4 + t % 4,  tw = (t % 128) / 4
//   shift = 2 * (d % 4)
__host__ __device__ __forceinline__ int p2t_byte(int64_t t, int d) {
  const int dq = d >> 2, tw = (int)((t & 127) >> 2);
  return dq * 128 + ((((tw >> 2) ^ (dq & 3))) << 4) + ((tw & 3) << 2) + (int)(t & 3);
}

// Canonical tile record (qjl_b200.h: qjl_tile_record): offsets of the QJL_REC_* fields.
struct TileRecord {
  int64_t off[QJL_REC_FIELDS];
  int64_t bytes;
};
__host__ __device__ inline TileRecord tile_record(int d, int m_in, int m_out, bool values) {
  TileRecord r;
  int64_t o = 0;
  r.off[QJL_REC_BITS_IN] = o;  o += 128 * (int64_t)(m_in / 8);
  r.off[QJL_REC_BITS_OUT] = m_out ? o : -1;  o += 128 * (int64_t)(m_out / 8);
  r.off[QJL_REC_NORM_IN] = o;  o += 256;
  r.off[QJL_REC_NORM_OUT] = m_out ? o : -1;  o += m_out ? 256 : 0;
  r.off[QJL_REC_CODES] = values ? o : -1;  o += values ? 128 * (int64_t)(d / 4) : 0;
  r.off[QJL_REC_ZERO] = values ? o : -1;  o += values ? 128 * 2 * (int64_t)(d / 32) : 0;
  r.off[QJL_REC_SCALE] = values ? o : -1;  o += values ? 128 * 2 * (int64_t)(d / 32) : 0;
  r.bytes = o;
  return r;
}

}  // namespace qjl
