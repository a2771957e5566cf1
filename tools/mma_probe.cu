// Probe: (1) mma.sync m16n8k32 s8 x u8 fragment layout, (2) m16n8k16 f16
// with fp16-subnormal A operands, (3) legacy IMMA / HMMA issue throughput on
// sm_100a.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__device__ __forceinline__ void imma(int* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void hmma(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// A: 16x32 int8 row-major, B: 32x8 u8 (B[k][n]), D: 16x8 int32
__global__ void k_imma_layout(const int8_t* A, const uint8_t* B, int* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  uint32_t a[4], b[2];
  auto packA = [&](int row, int k0) {
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= (uint32_t)(uint8_t)A[row * 32 + k0 + i] << (8 * i);
    return r;
  };
  auto packB = [&](int k0, int col) {
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= (uint32_t)B[(k0 + i) * 8 + col] << (8 * i);
    return r;
  };
  a[0] = packA(g, 4 * t);
  a[1] = packA(g + 8, 4 * t);
  a[2] = packA(g, 16 + 4 * t);
  a[3] = packA(g + 8, 16 + 4 * t);
  b[0] = packB(4 * t, g);
  b[1] = packB(16 + 4 * t, g);
  int d[4] = {0, 0, 0, 0};
  imma(d, a, b);
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2];
  D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

// A: 16x16 f16 row-major (bits), B: 16x8 f16 (B[k][n]), D 16x8 f32
__global__ void k_hmma_layout(const uint16_t* A, const uint16_t* B, float* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  uint32_t a[4], b[2];
  auto pk = [](uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); };
  a[0] = pk(A[g * 16 + 2 * t], A[g * 16 + 2 * t + 1]);
  a[1] = pk(A[(g + 8) * 16 + 2 * t], A[(g + 8) * 16 + 2 * t + 1]);
  a[2] = pk(A[g * 16 + 2 * t + 8], A[g * 16 + 2 * t + 9]);
  a[3] = pk(A[(g + 8) * 16 + 2 * t + 8], A[(g + 8) * 16 + 2 * t + 9]);
  b[0] = pk(B[(2 * t) * 8 + g], B[(2 * t + 1) * 8 + g]);
  b[1] = pk(B[(2 * t + 8) * 8 + g], B[(2 * t + 9) * 8 + g]);
  float d[4] = {0, 0, 0, 0};
  hmma(d, a, b);
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2];
  D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

template <bool INT>
__global__ void k_mma_tput(int iters, float* sink) {
  uint32_t a[4] = {threadIdx.x, 3u, 5u, 7u}, b[2] = {11u, 13u};
  if (INT) {
    int d0[4] = {0}, d1[4] = {0}, d2[4] = {0}, d3[4] = {0};
    for (int i = 0; i < iters; ++i) {
      imma(d0, a, b); imma(d1, a, b); imma(d2, a, b); imma(d3, a, b);
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = (float)(d0[0] + d1[1] + d2[2] + d3[3]);
  } else {
    float d0[4] = {0}, d1[4] = {0}, d2[4] = {0}, d3[4] = {0};
    for (int i = 0; i < iters; ++i) {
      hmma(d0, a, b); hmma(d1, a, b); hmma(d2, a, b); hmma(d3, a, b);
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = d0[0] + d1[1] + d2[2] + d3[3];
  }
}

static float h2f(uint16_t h) {
  __half x;
  memcpy(&x, &h, 2);
  return __half2float(x);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, clock %d kHz\n", sms, clk);
  // (1) IMMA layout
  int8_t hA[16 * 32];
  uint8_t hB[32 * 8];
  srand(1);
  for (int i = 0; i < 16 * 32; ++i) hA[i] = (int8_t)(rand() % 256 - 128);
  for (int i = 0; i < 32 * 8; ++i) hB[i] = (uint8_t)(rand() % 256);
  int8_t* dA; uint8_t* dB; int* dD;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, 16 * 8 * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  k_imma_layout<<<1, 32>>>(dA, dB, dD);
  int hD[128];
  cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 8; ++c) {
      int s = 0;
      for (int k = 0; k < 32; ++k) s += (int)hA[r * 32 + k] * (int)hB[k * 8 + c];
      bad += s != hD[r * 8 + c];
    }
  printf("IMMA s8.u8 m16n8k32 layout: %s (%d mismatches)\n", bad ? "MISMATCH" : "ok", bad);

  // (2) HMMA with subnormal A = c * 4^j * 2^-24 and normal B
  uint16_t hA2[256], hB2[128];
  for (int i = 0; i < 256; ++i) {
    int c = rand() % 4, j = rand() % 5;
    hA2[i] = (uint16_t)(c << (2 * j));          // subnormal bit pattern
  }
  for (int i = 0; i < 128; ++i) {
    __half x = __float2half((float)(rand() % 2000) / 997.0f);
    memcpy(&hB2[i], &x, 2);
  }
  uint16_t *dA2, *dB2; float* dD2;
  cudaMalloc(&dA2, 512); cudaMalloc(&dB2, 256); cudaMalloc(&dD2, 512);
  cudaMemcpy(dA2, hA2, 512, cudaMemcpyHostToDevice);
  cudaMemcpy(dB2, hB2, 256, cudaMemcpyHostToDevice);
  k_hmma_layout<<<1, 32>>>(dA2, dB2, dD2);
  float hD2[128];
  cudaMemcpy(hD2, dD2, 512, cudaMemcpyDeviceToHost);
  double maxrel = 0;
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int k = 0; k < 16; ++k) s += (double)h2f(hA2[r * 16 + k]) * (double)h2f(hB2[k * 8 + c]);
      double e = fabs(s - hD2[r * 8 + c]) / (fabs(s) + 1e-30);
      if (s != 0 && e > maxrel) maxrel = e;
      if (s == 0 && hD2[r * 8 + c] != 0) maxrel = 1;
    }
  printf("HMMA f16 subnormal-A max rel err %.3e (%s)\n", maxrel, maxrel < 1e-6 ? "ok" : "FLUSHED/BAD");
  // (2b) subnormal A x subnormal B (P' lo parts are often fp16 subnormals)
  for (int i = 0; i < 128; ++i) hB2[i] = (uint16_t)(1 + rand() % 1000);   // subnormal B
  cudaMemcpy(dB2, hB2, 256, cudaMemcpyHostToDevice);
  k_hmma_layout<<<1, 32>>>(dA2, dB2, dD2);
  cudaMemcpy(hD2, dD2, 512, cudaMemcpyDeviceToHost);
  maxrel = 0;
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int k = 0; k < 16; ++k) s += (double)h2f(hA2[r * 16 + k]) * (double)h2f(hB2[k * 8 + c]);
      double e = fabs(s - hD2[r * 8 + c]) / (fabs(s) + 1e-300);
      if (s != 0 && e > maxrel) maxrel = e;
      if (s == 0 && hD2[r * 8 + c] != 0) maxrel = 1;
    }
  printf("HMMA f16 subnormal-A x subnormal-B max rel err %.3e (%s) sample ref %.3e got %.3e\n", maxrel,
         maxrel < 1e-6 ? "ok" : "FLUSHED/BAD", 0.0, hD2[0]);
  // (2c) mixed-magnitude accumulation: normal B (~1) and tiny B (~1e-7 normal) in the same dot
  for (int i = 0; i < 128; ++i) {
    __half x = __float2half((i % 2) ? 1.0f : 3e-5f);
    memcpy(&hB2[i], &x, 2);
  }
  cudaMemcpy(dB2, hB2, 256, cudaMemcpyHostToDevice);
  k_hmma_layout<<<1, 32>>>(dA2, dB2, dD2);
  cudaMemcpy(hD2, dD2, 512, cudaMemcpyDeviceToHost);
  maxrel = 0;
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int k = 0; k < 16; ++k) s += (double)h2f(hA2[r * 16 + k]) * (double)h2f(hB2[k * 8 + c]);
      double e = fabs(s - hD2[r * 8 + c]) / (fabs(s) + 1e-300);
      if (s != 0 && e > maxrel) maxrel = e;
    }
  printf("HMMA mixed-magnitude B max rel err %.3e\n", maxrel);

  // (3) throughput
  float* sink;
  cudaMalloc(&sink, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 2; ++it) {
    for (int warps = 4; warps <= 16; warps *= 2) {
      const int iters = 4096, blocks = sms * 2;
      k_mma_tput<true><<<blocks, warps * 32>>>(iters, sink);
      cudaEventRecord(e0);
      k_mma_tput<true><<<blocks, warps * 32>>>(iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double n = (double)blocks * warps * iters * 4;
      printf("IMMA m16n8k32: warps/CTA %2d: %.3f ms, %.1f TOPS, %.2f mma/clk/SM (at %d MHz)\n", warps, ms,
             n * 16 * 8 * 32 * 2 / ms / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
      k_mma_tput<false><<<blocks, warps * 32>>>(iters, sink);
      cudaEventRecord(e0);
      k_mma_tput<false><<<blocks, warps * 32>>>(iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("HMMA m16n8k16: warps/CTA %2d: %.3f ms, %.1f TFLOPS, %.2f mma/clk/SM\n", warps, ms,
             n * 16 * 8 * 16 * 2 / ms / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3));
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
