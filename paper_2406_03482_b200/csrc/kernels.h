// Internal launch entry points (host side), implemented in k_*.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qjl_b200.h"

namespace qjl {

size_t detect_workspace(int units, int64_t n0, int d);
int launch_detect_outliers(const void* keys, int dtype, int units, int64_t n0, int d,
                           int64_t unit_stride, int h, int32_t* channels, double* mags, void* ws,
                           size_t ws_bytes, cudaStream_t st);
int launch_build_sketch(const double* s_in, const double* s_out, int m_in, int m_out, int d,
                        int h, const int32_t* channels, int units, int dtype, void* s_full,
                        cudaStream_t st);
// fused detect_outliers + per-unit S_full build (F2)
int launch_prefill_profile(const void* keys, int dtype, int units, int64_t n0, int d, int64_t unit_stride,
                           int h, const void* s_in, const void* s_out, int m_in, int m_out,
                           int sketch_dtype, int32_t* channels, double* mags, void* s_full, void* ws,
                           size_t ws_bytes, cudaStream_t st);
int launch_quantize_keys_simt(const void* keys, int dtype, int64_t n, int64_t kus,
                              const qjl_sketch_t& sk, const int32_t* ch, int h,
                              const qjl_key_cache_t& kc, int64_t row_offset, cudaStream_t st);
// tcgen05 + TMA tensor-core key quantizer (bf16/fp16 keys); returns
// QJL_ERR_UNSUPPORTED when the shape is outside its envelope (api.cu then runs the
// fp64 kernel, which is also the path for fp32/fp64 keys).
int launch_quantize_keys_tc(const void* keys, int dtype, int64_t n, int64_t kus,
                            const qjl_sketch_t& sk, const int32_t* ch, int h,
                            const qjl_key_cache_t& kc, int64_t row_offset, cudaStream_t st);
int launch_quantize_values(const void* v, int dtype, int64_t n, int64_t unit_stride,
                           const qjl_value_cache_t& vc, int64_t row_offset, cudaStream_t st);

int launch_sketch_query(const void* q, int q_dtype, int units, int G, int d,
                        const qjl_sketch_t& sk, int m_in, int m_total, float* sq, float* sums,
                        cudaStream_t st);
int launch_sketch_query_f64(const void* q, int q_dtype, int units, int G, int d, const qjl_sketch_t& sk,
                            int m_total, double* sq, cudaStream_t st);
int launch_scores_simt(const qjl_key_cache_t& kc, int64_t n, int G, const float* sq,
                       const float* sums, float* logits, cudaStream_t st);
int launch_sign_dot_batch(const uint8_t* bits, int64_t n, int m, int64_t row_bytes,
                          const double* values, int G, double* out, cudaStream_t st);
int launch_softmax_f64(const float* logits, int64_t rows, int64_t n, double inv_t, double* w,
                       cudaStream_t st);

size_t decode_simt_workspace(int units, int64_t n, int G, int d, int m_total);
int launch_decode_simt(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, int G,
                       const float* sq, const float* sums, float inv_t, float* out, float* lse,
                       float* logits, float* ws, cudaStream_t st);

// tcgen05 decode / scores on tile-major records (k_decode.cu).  vc == nullptr: keys only
// (the scores kernel; the record may or may not carry the value fields).
bool tile_path_supported(const qjl_key_cache_t& kc, const qjl_value_cache_t* vc, int G);
size_t decode_tile_workspace(const qjl_key_cache_t& kc, int64_t n, int G, bool scores);
int launch_decode_tile(const qjl_key_cache_t& kc, int64_t n, const void* q, int q_dtype, int G,
                       const qjl_sketch_t& sk, float inv_t, float* out, float* lse, float* logits, void* ws,
                       size_t ws_bytes, unsigned flags, cudaStream_t st);
// decode step with append: the new token (k_new, v_new [units][128], query dtype) is
// quantized into row n by the query-sketch kernel, then rows [0, n + 1) are decoded
int launch_decode_step_tile(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, const void* q,
                            int q_dtype, int G, const qjl_sketch_t& sk, const int32_t* channels, int h,
                            const void* k_new, const void* v_new, float inv_t, float* out, float* lse,
                            float* logits, void* ws, size_t ws_bytes, unsigned flags, cudaStream_t st);
int launch_scores_tile(const qjl_key_cache_t& kc, int64_t n, const void* q, int q_dtype, int G,
                       const qjl_sketch_t& sk, float* logits, void* ws, size_t ws_bytes, unsigned flags,
                       cudaStream_t st);
int bench_decode_tile(const qjl_key_cache_t& kc, int64_t n, const void* q, int q_dtype, int G, const qjl_sketch_t& sk,
                      float inv_t, float* out, float* lse, void* ws, size_t ws_bytes, unsigned flags, int reps,
                      float* ms, cudaStream_t st);

// batched block-wise sketch orthogonalization (k_orth.cu)
int launch_orthogonalize(const double* g, int batch, int m, int d, double* out, cudaStream_t st);

// QJLC cache records <-> device cache layout (k_qjlc.cu)
int64_t qjlc_record_bytes(int d, int m_in_file, int m_out_file);
int launch_qjlc_export(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int mfi, int mfo,
                       int64_t row0, int64_t n, uint8_t* out, int64_t ustride, cudaStream_t st);
int launch_qjlc_import(const uint8_t* in, int64_t ustride, int mfi, int mfo, int64_t n,
                       const qjl_key_cache_t& kc, const qjl_value_cache_t* vc, int64_t row0,
                       cudaStream_t st);

}  // namespace qjl
