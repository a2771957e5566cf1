// Probe: tcgen05.mma kind::i8 with A (u8) in TMEM, B (s8) from SMEM, D s32 in TMEM.
//  D1 = A[128 x 64] . B1[16 x 64]^T, B1 K-major SWIZZLE_128B (2 MMAs of K = 32)
//  D2 = A[128 x 64] . B2[64 x 48],   B2 MN-major SWIZZLE_NONE (2 MMAs of K = 32)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tc_i8_probe tools/tc_i8_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__host__ __device__ constexpr uint32_t idesc_i8(int n, int b_mn_major) {
  // D s32 (2), A u8 (0), B s8 (1), A K-major, B major per arg, N >> 3, M = 128
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void __launch_bounds__(128, 1) k_probe(const uint8_t* A, const int8_t* B1, const int8_t* B2, int* D1, int* D2) {
  __shared__ __align__(1024) uint8_t sb1[2048];      // 16 rows x 128 B, SW128
  __shared__ __align__(1024) uint8_t sb2[3 * 1024];  // [3 chunks][64 k][16 B]
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  const int t = threadIdx.x, warp = t >> 5;
  // B1: element (n, k) -> atom n/8, row n%8, chunk k/16 swizzled with row
  for (int i = t; i < 16 * 64; i += 128) {
    const int n = i / 64, k = i % 64;
    const int off = (n / 8) * 1024 + (n % 8) * 128 + (((k / 16) ^ (n % 8)) * 16) + (k % 16);
    sb1[off] = (uint8_t)B1[n * 64 + k];
  }
  // B2: element (k, n) -> chunk n/16, row k, byte n%16
  for (int i = t; i < 64 * 48; i += 128) {
    const int k = i / 48, n = i % 48;
    sb2[(n / 16) * 1024 + k * 16 + (n % 16)] = (uint8_t)B2[k * 48 + n];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tptr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tptr;
  // A row t -> TMEM lane t, columns 0..15 (4 K bytes per column, little endian)
  uint32_t r[16];
  for (int c = 0; c < 16; ++c) r[c] = *reinterpret_cast<const uint32_t*>(A + t * 64 + 4 * c);
  tmem_st16(tbase + ((uint32_t)(warp * 32) << 16), r);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    for (int ks = 0; ks < 2; ++ks) {
      mma_i8_ts(tbase + 64, tbase + 8 * ks, desc_sw128(smem_u32(sb1) + 32 * ks), idesc_i8(16, 0), ks);
      mma_i8_ts(tbase + 80, tbase + 8 * ks, desc_none(smem_u32(sb2) + ks * 32 * 16, 128, 1024), idesc_i8(48, 1), ks);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t d[16];
  tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + 64, d);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) D1[t * 16 + i] = (int)d[i];
  for (int part = 0; part < 3; ++part) {
    tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + 80 + 16 * part, d);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) D2[t * 48 + 16 * part + i] = (int)d[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

int main() {
  const int M = 128, K = 64;
  uint8_t* hA = (uint8_t*)malloc(M * K);
  int8_t* hB1 = (int8_t*)malloc(16 * K);
  int8_t* hB2 = (int8_t*)malloc(K * 48);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = rand() & 0xFF;
  for (int i = 0; i < 16 * K; ++i) hB1[i] = (int8_t)(rand() & 0xFF);
  for (int i = 0; i < K * 48; ++i) hB2[i] = (int8_t)(rand() & 0xFF);
  uint8_t* dA; int8_t *dB1, *dB2; int *dD1, *dD2;
  cudaMalloc(&dA, M * K); cudaMalloc(&dB1, 16 * K); cudaMalloc(&dB2, K * 48);
  cudaMalloc(&dD1, M * 16 * 4); cudaMalloc(&dD2, M * 48 * 4);
  cudaMemcpy(dA, hA, M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB1, hB1, 16 * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB2, hB2, K * 48, cudaMemcpyHostToDevice);
  k_probe<<<1, 128>>>(dA, dB1, dB2, dD1, dD2);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  int* D1 = (int*)malloc(M * 16 * 4); int* D2 = (int*)malloc(M * 48 * 4);
  cudaMemcpy(D1, dD1, M * 16 * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(D2, dD2, M * 48 * 4, cudaMemcpyDeviceToHost);
  int bad1 = 0, bad2 = 0;
  for (int m = 0; m < M; ++m) {
    for (int n = 0; n < 16; ++n) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)hA[m * K + k] * hB1[n * K + k];
      if (s != D1[m * 16 + n]) { if (bad1 < 4) printf("D1[%d][%d] %d != %ld\n", m, n, D1[m * 16 + n], s); ++bad1; }
    }
    for (int n = 0; n < 48; ++n) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)hA[m * K + k] * hB2[k * 48 + n];
      if (s != D2[m * 48 + n]) { if (bad2 < 4) printf("D2[%d][%d] %d != %ld\n", m, n, D2[m * 48 + n], s); ++bad2; }
    }
  }
  printf("D1 (K-major SW128 B, N=16) mismatches: %d / %d\n", bad1, M * 16);
  printf("D2 (MN-major INTERLEAVE B, N=48) mismatches: %d / %d\n", bad2, M * 48);
  return 0;
}
