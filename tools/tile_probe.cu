// Memory-pipeline probe for the decode cache layout (C3 size: 16384 tiles x 11776 B).
// Compares the structure-of-arrays layout (7 bulk copies per 128-token tile, one per
// cache array) with tile-major records (one 11776-byte bulk copy per tile), for several
// ring depths and CTAs per SM.  Only thread 0 issues copies; consumers wait on the
// full barrier and release the stage through an empty barrier (4 warps arrive).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tile_probe tools/tile_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(b),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void expect_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

__constant__ int c_piece[7] = {4096, 1024, 256, 256, 4096, 1024, 1024};
constexpr int kRec = 11776;

// mode 0: SoA (7 arrays), mode 1: tile-major records.  Contiguous stream-K tile ranges.
__global__ void __launch_bounds__(128) k_probe(const uint8_t* buf, int64_t T, int mode, int stages,
                                               unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t s0 = smem_u32(sm);
  const uint32_t full = s0 + stages * kRec, empty = full + 8 * stages;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t r0 = (int64_t)blockIdx.x * T / gridDim.x, r1 = (int64_t)(blockIdx.x + 1) * T / gridDim.x;
  const int nt = (int)(r1 - r0);
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int i) {
    const int s = i % stages;
    if (i >= stages) mbar_wait(empty + 8 * s, ((i / stages) - 1) & 1);
    const int64_t t = r0 + i;
    const uint32_t fb = full + 8 * s, dst = s0 + s * kRec;
    expect_tx(fb, kRec);
    if (mode == 1) {
      bulk(dst, buf + t * kRec, kRec, fb, pol);
    } else {
      size_t base = 0;
      int off = 0;
#pragma unroll
      for (int p = 0; p < 7; ++p) {
        bulk(dst + off, buf + base + (size_t)t * c_piece[p], c_piece[p], fb, pol);
        base += (size_t)T * c_piece[p];
        off += c_piece[p];
      }
    }
  };
  if (tid == 0)
    for (int i = 0; i < stages - 1 && i < nt; ++i) issue(i);
  unsigned long long acc = 0;
  for (int i = 0; i < nt; ++i) {
    const int s = i % stages;
    if (tid == 0 && i + stages - 1 < nt) issue(i + stages - 1);
    mbar_wait(full + 8 * s, (i / stages) & 1);
    acc += sm[s * kRec + tid * 64];
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + 8 * s);
  }
  if (acc == 0xFFFFFFFFFFFFull) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int64_t T : {(int64_t)16384, (int64_t)131072}) {   // C3 (193 MB) and C5 B16x128k (1.54 GB)
    const size_t bytes = (size_t)T * kRec;
    uint8_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    for (int mode = 0; mode < 2; ++mode)
      for (int cps : {1, 2, 4})
        for (int stages : {3, 4, 6, 8, 12, 16}) {
          const size_t smem = (size_t)stages * kRec + 16 * stages;
          if (smem * cps > 220 * 1024 || smem > 227 * 1024) continue;
          cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          const int ctas = sms * cps;
          for (int w = 0; w < 2; ++w) k_probe<<<ctas, 128, smem>>>(buf, T, mode, stages, sink);
          const int reps = T > 20000 ? 5 : 20;
          cudaEventRecord(e0);
          for (int r = 0; r < reps; ++r) k_probe<<<ctas, 128, smem>>>(buf, T, mode, stages, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          printf("T=%6lld %-10s ctas/SM %d stages %2d: %8.1f us  %7.0f GB/s  (%s)\n", (long long)T,
                 mode ? "tile-major" : "7-arrays", cps, stages, ms * 1e3 / reps, (double)bytes * reps / (ms * 1e-3) / 1e9,
                 cudaGetErrorString(cudaGetLastError()));
        }
    cudaFree(buf);
  }
  return 0;
}
