// HMMA m16n8k16 (f16 x f16 -> f32) accumulation precision with realistic PV
// operands: B = P' split hi/lo (log-uniform P'), A = 2-bit codes encoded either
// as fp16 subnormals c*4^e*2^-24 or as normals (c + 8) or c * 2^-10.
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__device__ __forceinline__ void hmma(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// T trials of one 16x8x16 MMA each
__global__ void k(const uint16_t* A, const uint16_t* B, float* D, int chain) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, tr = blockIdx.x;
  const uint16_t* a_ = A + tr * 256;
  const uint16_t* b_ = B + tr * 128;
  auto pk = [](uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); };
  uint32_t a[4], b[2];
  a[0] = pk(a_[g * 16 + 2 * t], a_[g * 16 + 2 * t + 1]);
  a[1] = pk(a_[(g + 8) * 16 + 2 * t], a_[(g + 8) * 16 + 2 * t + 1]);
  a[2] = pk(a_[g * 16 + 2 * t + 8], a_[g * 16 + 2 * t + 9]);
  a[3] = pk(a_[(g + 8) * 16 + 2 * t + 8], a_[(g + 8) * 16 + 2 * t + 9]);
  b[0] = pk(b_[(2 * t) * 8 + g], b_[(2 * t + 1) * 8 + g]);
  b[1] = pk(b_[(2 * t + 8) * 8 + g], b_[(2 * t + 9) * 8 + g]);
  float d[4] = {0, 0, 0, 0};
  for (int i = 0; i < chain; ++i) hmma(d, a, b);
  float* o = D + tr * 128;
  o[g * 8 + 2 * t] = d[0];
  o[g * 8 + 2 * t + 1] = d[1];
  o[(g + 8) * 8 + 2 * t] = d[2];
  o[(g + 8) * 8 + 2 * t + 1] = d[3];
}

static uint16_t f2h(float x) { __half h = __float2half_rn(x); uint16_t u; memcpy(&u, &h, 2); return u; }
static double h2d(uint16_t u) { __half h; memcpy(&h, &u, 2); return (double)__half2float(h); }

int main() {
  const int T = 2048;
  uint16_t* hA = (uint16_t*)malloc(T * 256 * 2);
  uint16_t* hB = (uint16_t*)malloc(T * 128 * 2);
  float* hD = (float*)malloc(T * 128 * 4);
  uint16_t *dA, *dB; float* dD;
  cudaMalloc(&dA, T * 256 * 2); cudaMalloc(&dB, T * 128 * 2); cudaMalloc(&dD, T * 128 * 4);
  srand(7);
  const char* enc[3] = {"subnormal c*4^e*2^-24", "normal c*2^-10 (+0 for c=0)", "normal 8+c"};
  const char* bmode[3] = {"B=P' hi only, logU[1e-6,3]", "B=P' hi only, U[0.5,1]", "B=P' hi, logU[1e-3,3]"};
  for (int bm = 0; bm < 3; ++bm)
    for (int e = 0; e < 3; ++e)
      for (int chain = 1; chain <= 2; chain *= 2) {
        for (int tr = 0; tr < T; ++tr) {
          for (int i = 0; i < 256; ++i) {
            int c = rand() % 4, row = i / 16, ex = row % 5;
            uint16_t v;
            if (e == 0) v = (uint16_t)(c << (2 * ex));
            else if (e == 1) v = f2h((float)c * ldexpf(1.f, -10));
            else v = f2h(8.f + c);
            hA[tr * 256 + i] = v;
          }
          for (int i = 0; i < 128; ++i) {
            double u = (double)rand() / RAND_MAX;
            double P = bm == 0 ? exp(log(1e-6) + u * (log(3.0) - log(1e-6)))
                     : bm == 1 ? 0.5 + 0.5 * u : exp(log(1e-3) + u * (log(3.0) - log(1e-3)));
            hB[tr * 128 + i] = f2h((float)P);
          }
        }
        cudaMemcpy(dA, hA, T * 256 * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, T * 128 * 2, cudaMemcpyHostToDevice);
        k<<<T, 32>>>(dA, dB, dD, chain);
        cudaMemcpy(hD, dD, T * 128 * 4, cudaMemcpyDeviceToHost);
        double maxrel = 0, sumrel = 0, bias = 0;
        int cnt = 0;
        for (int tr = 0; tr < T; ++tr)
          for (int r = 0; r < 16; ++r)
            for (int c = 0; c < 8; ++c) {
              double s = 0;
              for (int kk = 0; kk < 16; ++kk) s += h2d(hA[tr * 256 + r * 16 + kk]) * h2d(hB[tr * 128 + kk * 8 + c]);
              s *= chain;
              if (s == 0) continue;
              double rel = (hD[tr * 128 + r * 8 + c] - s) / fabs(s);
              maxrel = fmax(maxrel, fabs(rel));
              sumrel += fabs(rel);
              bias += rel;
              ++cnt;
            }
        printf("%-28s A=%-28s chain=%d: max rel %.2e mean |rel| %.2e mean signed %.2e\n", bmode[bm], enc[e], chain,
               maxrel, sumrel / cnt, bias / cnt);
      }
  return 0;
}
