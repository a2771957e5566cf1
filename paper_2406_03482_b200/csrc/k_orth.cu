// Device-side sketch orthogonalization (sketch.py:82-103) for batches of sketches --
// the statistical suites draw thousands of sketches per run.
//
// Per (sketch, block of <= d rows) one CTA: A = block^T (d x k, column-major in shared
// memory, fp64) is factored by Householder QR (LAPACK dgeqr2 / dlarfg conventions:
// beta = -sign(alpha) * ||x||, tau = (beta - alpha) / beta), Q is formed in place by
// backward accumulation (dorg2r), then every column j is multiplied by sign(R_jj)
// (0 -> +1) and by sqrt(d) and written as output row start + j.  Q * sign(diag R) is the
// unique thin QR factor with a positive diagonal, so the result equals numpy.linalg.qr's
// sign-corrected factor to rounding (~1e-15).
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace qjl {
namespace {

constexpr int kOrthThreads = 256;

// block-wide sum of one double per thread (all threads must call)
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__global__ void __launch_bounds__(kOrthThreads) k_orthogonalize(const double* __restrict__ g, int m, int d,
                                                                double* __restrict__ out) {
  extern __shared__ double A[];                  // [k][d]: column j = input row start + j
  __shared__ double red[kOrthThreads / 32];
  __shared__ double tau_s[256], rdiag[256];       // k <= 256 (api.cu bound)
  const int b = blockIdx.y;
  const int start = blockIdx.x * d;
  const int k = min(d, m - start);
  const double* G = g + ((int64_t)b * m + start) * d;
  for (int i = threadIdx.x; i < k * d; i += blockDim.x) A[i] = G[i];   // row-major block == A^T columns
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  // ---- Householder QR (dgeqr2): reflector j annihilates A(j+1:d, j)
  for (int j = 0; j < k; ++j) {
    double* col = A + (int64_t)j * d;
    double part = 0.0;
    for (int r = j + 1 + threadIdx.x; r < d; r += blockDim.x) part += col[r] * col[r];
    const double xnorm2 = block_sum(part, red);
    const double alpha = col[j];
    double tau = 0.0, beta = alpha;
    if (xnorm2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
      tau = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      for (int r = j + 1 + threadIdx.x; r < d; r += blockDim.x) col[r] *= scal;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tau_s[j] = tau;
      rdiag[j] = beta;
    }
    // apply H_j = I - tau v v^T (v_j = 1, v_r = col[r]) to columns j+1 .. k-1, a warp per column
    if (tau != 0.0) {
      for (int c = j + 1 + warp; c < k; c += nwarps) {
        double* cc = A + (int64_t)c * d;
        double w = (lane == 0) ? cc[j] : 0.0;
        for (int r = j + 1 + lane; r < d; r += 32) w += col[r] * cc[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        w *= tau;
        if (lane == 0) cc[j] -= w;
        for (int r = j + 1 + lane; r < d; r += 32) cc[r] -= w * col[r];
      }
    }
    __syncthreads();
  }
  // ---- form Q in place (dorg2r), last reflector first
  for (int i = k - 1; i >= 0; --i) {
    double* col = A + (int64_t)i * d;
    const double tau = tau_s[i];
    if (i < k - 1 && tau != 0.0) {
      for (int c = i + 1 + warp; c < k; c += nwarps) {
        double* cc = A + (int64_t)c * d;
        double w = (lane == 0) ? cc[i] : 0.0;   // v_i = 1
        for (int r = i + 1 + lane; r < d; r += 32) w += col[r] * cc[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        w *= tau;
        if (lane == 0) cc[i] -= w;
        for (int r = i + 1 + lane; r < d; r += 32) cc[r] -= w * col[r];
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < d; r += blockDim.x) {
      if (r > i) col[r] *= -tau;
      else if (r == i) col[r] = 1.0 - tau;
      else col[r] = 0.0;
    }
    __syncthreads();
  }
  // ---- sign correction and row scaling: output row start + j = Q[:, j] * sign(R_jj) * sqrt(d)
  const double scale = sqrt((double)d);
  double* O = out + ((int64_t)b * m + start) * d;
  for (int i = threadIdx.x; i < k * d; i += blockDim.x) {
    const int j = i / d;
    const double s = rdiag[j] < 0.0 ? -1.0 : 1.0;
    O[i] = A[i] * s * scale;
  }
}

}  // namespace

int launch_orthogonalize(const double* g, int batch, int m, int d, double* out, cudaStream_t st) {
  const int blocks = (m + d - 1) / d;
  const int k = d < m ? d : m;
  const size_t smem = (size_t)k * d * sizeof(double);
  cudaFuncSetAttribute(k_orthogonalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_orthogonalize<<<dim3(blocks, batch), kOrthThreads, smem, st>>>(g, m, d, out);
  QJL_LAUNCH_CHECK("orthogonalize");
  return QJL_OK;
}

}  // namespace qjl
