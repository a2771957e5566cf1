// HBM streaming probe: CTAs stream contiguous slices of a large buffer into smem with
// cp.async.bulk through an mbarrier ring (lookahead = stages - 1).  Each stage is
// `pieces` copies that together cover `stage_bytes`; pieces come from `pieces`
// separate arrays (like the SoA decode cache) or from one contiguous region.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_probe tools/bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   smem_u32(b)), "r"(ph) : "memory");
}

// cache-like stage: 7 pieces (bits_in, bits_out, norm_in, norm_out, codes, zero, scale)
__constant__ int c_piece[7] = {4096, 1024, 256, 256, 4096, 1024, 1024};
__global__ void __launch_bounds__(128) k_cache(const uint8_t* buf, int tiles, int stages, int ntiles_cta,
                                               unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int stage_bytes = 11776;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * stage_bytes);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int s = i % stages;
    const int64_t t = (int64_t)blockIdx.x * ntiles_cta + i;   // global tile
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(stage_bytes)
                 : "memory");
    size_t base = 0;
    int off = 0;
    for (int p = 0; p < 7; ++p) {
      const uint8_t* src = buf + base + (size_t)t * c_piece[p];
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + s * stage_bytes + off)),
          "l"(src), "r"(c_piece[p]), "r"(smem_u32(&full[s]))
          : "memory");
      base += (size_t)tiles * c_piece[p];
      off += c_piece[p];
    }
  };
  if (tid == 0)
    for (int i = 0; i < stages - 1 && i < ntiles_cta; ++i) issue(i);
  unsigned long long acc = 0;
  for (int i = 0; i < ntiles_cta; ++i) {
    const int s = i % stages;
    mbar_wait(&full[s], (i / stages) & 1);
    acc += sm[s * stage_bytes + tid];
    __syncthreads();
    if (tid == 0 && i + stages - 1 < ntiles_cta) issue(i + stages - 1);
  }
  if (acc == 0xFFFFFFFFFFFFull) sink[0] = acc;
}

// same, but issued the way k_udecode does: each warp's lane 0 issues a share of the
// pieces after waiting on an "empty" mbarrier that all 4 warps arrive on
__global__ void __launch_bounds__(128) k_cache_mb(const uint8_t* buf, int tiles, int stages, int ntiles_cta,
                                                  unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int stage_bytes = 11776;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int lo[5] = {0, 1, 4, 5, 7};   // warp w issues pieces [lo[w], lo[w+1])
  auto issue = [&](int i) {
    const int s = i % stages;
    if (i >= stages) mbar_wait(&empty[s], ((i / stages) - 1) & 1);
    const int64_t t = (int64_t)blockIdx.x * ntiles_cta + i;
    if (warp == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(stage_bytes)
                   : "memory");
    size_t base = 0;
    int off = 0;
    for (int p = 0; p < 7; ++p) {
      if (p >= lo[warp] && p < lo[warp + 1]) {
        const uint8_t* src = buf + base + (size_t)t * c_piece[p];
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + s * stage_bytes + off)),
            "l"(src), "r"(c_piece[p]), "r"(smem_u32(&full[s]))
            : "memory");
      }
      base += (size_t)tiles * c_piece[p];
      off += c_piece[p];
    }
  };
  if (lane == 0)
    for (int i = 0; i < stages - 1 && i < ntiles_cta; ++i) issue(i);
  unsigned long long acc = 0;
  for (int i = 0; i < ntiles_cta; ++i) {
    const int s = i % stages;
    if (lane == 0 && i + stages - 1 < ntiles_cta) issue(i + stages - 1);
    mbar_wait(&full[s], (i / stages) & 1);
    acc += sm[s * stage_bytes + tid];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
  }
  if (acc == 0xFFFFFFFFFFFFull) sink[0] = acc;
}

__global__ void __launch_bounds__(128) k_stream(const uint8_t* buf, size_t slice, int stage_bytes, int stages,
                                                int pieces, int soa, size_t array_bytes, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * stage_bytes);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nt = (int)(slice / stage_bytes);
  const int piece = stage_bytes / pieces;
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(stage_bytes)
                 : "memory");
    for (int p = 0; p < pieces; ++p) {
      const uint8_t* src;
      if (soa) src = buf + (size_t)p * array_bytes + ((size_t)blockIdx.x * nt + i) * piece;
      else src = buf + (size_t)blockIdx.x * slice + (size_t)i * stage_bytes + p * piece;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + s * stage_bytes + p * piece)),
          "l"(src), "r"(piece), "r"(smem_u32(&full[s]))
          : "memory");
    }
  };
  if (tid == 0)
    for (int i = 0; i < stages - 1 && i < nt; ++i) issue(i);
  unsigned long long acc = 0;
  for (int i = 0; i < nt; ++i) {
    const int s = i % stages;
    mbar_wait(&full[s], (i / stages) & 1);
    acc += sm[s * stage_bytes + tid];
    __syncthreads();   // every thread done with stage (i-1) % stages before it is refilled
    if (tid == 0 && i + stages - 1 < nt) issue(i + stages - 1);
  }
  if (acc == 0xFFFFFFFFFFFFull) sink[0] = acc;
}

int main() {
  const size_t total = 1ull << 30;   // bytes streamed per launch (1 GiB)
  uint8_t* buf;
  cudaMalloc(&buf, total + (64 << 20));
  cudaMemset(buf, 1, total + (64 << 20));
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int ctas_per_sm, stage_bytes, stages, pieces, soa; };
  const Cfg cfgs[] = {
      {4, 12288, 3, 1, 0}, {4, 12288, 3, 6, 1}, {4, 12288, 3, 6, 0}, {4, 12288, 4, 1, 0}, {4, 12288, 5, 1, 0},
      {2, 24576, 3, 1, 0}, {2, 24576, 4, 1, 0}, {1, 49152, 4, 1, 0}, {8, 12288, 2, 1, 0}, {4, 24576, 2, 1, 0},
      {4, 6144, 6, 1, 0},  {4, 12288, 3, 12, 1}, {4, 12288, 4, 6, 1},
  };
  for (const Cfg& c : cfgs) {
    const int ctas = sms * c.ctas_per_sm;
    const size_t slice = (total / ctas) / c.stage_bytes * c.stage_bytes;
    const size_t smem = (size_t)c.stages * c.stage_bytes + 8 * c.stages + 1024;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const size_t array_bytes = (size_t)ctas * slice / c.pieces;
    for (int w = 0; w < 2; ++w)
      k_stream<<<ctas, 128, smem>>>(buf, slice, c.stage_bytes, c.stages, c.pieces, c.soa, array_bytes, sink);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r)
      k_stream<<<ctas, 128, smem>>>(buf, slice, c.stage_bytes, c.stages, c.pieces, c.soa, array_bytes, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = (double)ctas * slice * reps / (ms * 1e-3) / 1e9;
    printf("ctas/SM %d stage %6d B x %d stages, %2d pieces (%s): %7.0f GB/s  (%s)\n", c.ctas_per_sm, c.stage_bytes,
           c.stages, c.pieces, c.soa ? "separate arrays" : "contiguous", gbs, cudaGetErrorString(cudaGetLastError()));
  }
  // cache-like: 16384 tiles (C3), 592 CTAs, ~28 tiles each
  for (int mode = 0; mode < 2; ++mode)
  for (int stages : {3, 4}) {
    const int tiles = 16384 + 592;   // a little slack so every CTA gets ntiles_cta tiles
    const int ctas = sms * 4, ntiles_cta = 16384 / ctas + 1;
    const size_t smem = (size_t)stages * 11776 + 8 * stages + 1024;
    auto kern = mode ? k_cache_mb : k_cache;
    const size_t smem2 = smem + 8 * stages;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    for (int w = 0; w < 2; ++w) kern<<<ctas, 128, smem2>>>(buf, tiles, stages, ntiles_cta, sink);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) kern<<<ctas, 128, smem2>>>(buf, tiles, stages, ntiles_cta, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)ctas * ntiles_cta * 11776;
    printf("%s cache-like 7 arrays, %d stages, %d CTAs x %d tiles (%.0f MB): %.1f us/launch -> %7.0f GB/s\n", mode ? "[per-warp issue + empty mbarrier]" : "[thread 0 + syncthreads]", stages,
           ctas, ntiles_cta, bytes / 1e6, ms * 1e3 / reps, bytes * reps / (ms * 1e-3) / 1e9);
  }
  return 0;
}
