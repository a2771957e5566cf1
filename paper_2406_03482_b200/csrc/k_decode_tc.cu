// Tensor-core fused QJL decode (K2 score estimator + K3 online softmax . V) for
// P2 value caches on sm_100a.
//
//  * Data movement: one producer warp streams each 128-token tile of the packed
//    cache (sign bits, fp16 norms, 2-bit codes, fp16 zero/scale) HBM -> smem with
//    cp.async.bulk (TMA bulk copies) into a kStages mbarrier ring; consumer warps
//    never issue global loads on the hot path.
//  * Scores (estimator.py:149-170 identity 2*sum_set(Sq) - sum(Sq)): the query
//    sketch of every query head is quantized to a 32-bit fixed-point integer and
//    split into four int8 digits; rows of an m16n8k32 IMMA A operand are
//    (digit, query) pairs, so one IMMA computes 4 digits x 4 query heads x 8
//    tokens x 32 sign bits with exact int32 accumulation.  The B operand is the
//    packed sign word itself, masked in place: `w & (0x01010101 << 2q)` turns 4
//    sign bits into 4 u8 lanes of value 2^(2q)*bit -- 2 LOP3 per 8 bits, no
//    unpacking; the 2^s weights are folded into the digits.
//  * PV: out[q][d] = sum_t P'[t][q] c[t][d] + sum_t p[t][q] zero[t][g], with
//    P' = p * scale split hi/lo in fp16 (22-bit P'), codes entering an m16n8k16
//    HMMA as EXACT fp16 subnormals c * 4^e * 2^-24 produced by a single LOP3 on
//    a PRMT of two tokens' code words (P2 layout puts lane-row g's 16 dims in
//    code word g), rescaled by 2^24/4^e per output row at the end.
//  * Online softmax in the log2 domain per query head; one partial (m, l, acc)
//    per (CTA, unit segment); CTAs own equal contiguous ranges of the flattened
//    (unit, tile) space (stream-K) so every SM gets the same number of tiles.
#include "common.cuh"
#include "kernels.h"

namespace qjl {
namespace tc {

constexpr int kNW = 4;             // consumer warps
constexpr int kTile = 32 * kNW;    // tokens per pipeline stage
constexpr int kStages = 4;
constexpr int kThreads = 32 * (kNW + 1);
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct Params {
  qjl_key_cache_t kc;
  qjl_value_cache_t vc;
  int64_t n;
  int G;
  int units;
  int tpu;               // tiles per unit
  int64_t total_tiles;
  int ctas;
  int max_seg;           // partial slots per unit
  const uint4* afrag;    // [units][KC][32 lanes] (4 x u32 A regs)
  const float4* qconst;  // [units][4 queries] {k_in, b_in, k_out, b_out}
  float* part;           // [units][max_seg][G][2 + 128]
};

__host__ __device__ __forceinline__ int64_t tile_begin(int c, int64_t T, int C) {
  return (int64_t)c * T / C;
}
__host__ __device__ __forceinline__ int cta_of_tile(int64_t t, int64_t T, int C) {
  return (int)(((t + 1) * (int64_t)C + T - 1) / T) - 1;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void imma(int* d, const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void hmma(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Code slot p (0..7 within each 16-bit half of x) -> fp16 NORMAL 1 + c*4^s/1024,
// s = 3 + (p & 1): the half-word is first shifted so slot p lands on mantissa
// slot s (one SHF per m-tile: slots {0,1} << 6, {2,3} << 2, {4,5} >> 2,
// {6,7} >> 6; bits spilling across the half boundary are masked off), then one
// LOP3 masks the code and ORs in the exponent of 1.0.  Normal operands keep the
// HMMA fp32 sum accurate to ~1e-7; fp16 subnormal operands measured ~2e-4
// (tools/hmma_precision.cu).  The offset sum_t P' is removed with the exact
// FFMA accumulator Y = sum_t p * scale (offset/step ratio <= 16).
template <int PAIR>   // PAIR = p >> 1 = m-tile & 3
__device__ __forceinline__ uint32_t code_shift(uint32_t x) {
  if constexpr (PAIR == 0) return x << 6;
  else if constexpr (PAIR == 1) return x << 2;
  else if constexpr (PAIR == 2) return x >> 2;
  else return x >> 6;
}
template <int S>      // S = 3 or 4
__device__ __forceinline__ uint32_t code_h2(uint32_t xs) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(xs), "r"(0x00030003u << (2 * S)), "r"(0x3C003C00u));
  return r;   // (xs & mask) | one
}

// --------------------------------------------------------------- smem layout
template <int KCI, int KCO>
struct Layout {
  static constexpr int kBitsIn = kTile * KCI * 4;
  static constexpr int kBitsOut = kTile * KCO * 4;
  static constexpr int kNorm = kTile * 2;
  static constexpr int kCodes = kTile * 32;
  static constexpr int kConst = kTile * 8;
  static constexpr int oBitsIn = 0;
  static constexpr int oBitsOut = oBitsIn + kBitsIn;
  static constexpr int oNormIn = oBitsOut + kBitsOut;
  static constexpr int oNormOut = oNormIn + kNorm;
  static constexpr int oCodes = oNormOut + (KCO ? kNorm : 0);
  static constexpr int oZero = oCodes + kCodes;
  static constexpr int oScale = oZero + kConst;
  static constexpr int kStageBytes = oScale + kConst;
  static constexpr int oPbuf = kStages * kStageBytes;              // per warp 2 KB
  static constexpr int oRed = oPbuf + kNW * 2048;                  // flush scratch
  static constexpr int kRec = 2 + 4 + 128;                          // m, l, Z[4], acc[128]
  static constexpr int kRedBytes = kNW * 4 * kRec * 4;
  static constexpr int oBar = oRed + kRedBytes;
  static constexpr int kTotal = oBar + 2 * kStages * 8;
};

// ----------------------------------------------------------------- prep kernel
// Per unit: Sq = S_full . q (fp64), per-side sigma = max|Sq|/2^30, weighted
// integer sketch, 4 signed-byte digits laid out as IMMA A fragments.
template <typename TQ, typename TS, int KCI, int KCO>
__global__ void __launch_bounds__(256) k_prep(const TQ* __restrict__ q, int G, const TS* __restrict__ s_full,
                                              int64_t s_unit_stride, float inv_t, uint4* __restrict__ afrag,
                                              float4* __restrict__ qconst) {
  constexpr int MI = KCI * 32, MO = KCO * 32, MT = MI + MO, KC = KCI + KCO;
  constexpr int d = 128;
  __shared__ double qs[4][d];
  __shared__ double sq[4][MT];
  __shared__ int32_t si[4][MT];
  __shared__ double red[4][2][2];   // [q][side][max, sum]
  const int u = blockIdx.x;
  const TS* S = s_full + (int64_t)u * s_unit_stride;
  for (int i = threadIdx.x; i < 4 * d; i += blockDim.x) {
    const int g = i / d;
    qs[g][i % d] = g < G ? to_f64(q[((int64_t)u * G + g) * d + i % d]) : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < MT; r += blockDim.x) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    const TS* row = S + (int64_t)r * d;
    for (int c = 0; c < d; ++c) {
      const double s = to_f64(row[c]);
      a0 = fma(s, qs[0][c], a0);
      a1 = fma(s, qs[1][c], a1);
      a2 = fma(s, qs[2][c], a2);
      a3 = fma(s, qs[3][c], a3);
    }
    // the generic path rounds Sq to fp32 before use; keep the same values
    sq[0][r] = (double)(float)a0;
    sq[1][r] = (double)(float)a1;
    sq[2][r] = (double)(float)a2;
    sq[3][r] = (double)(float)a3;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int g = threadIdx.x >> 1, side = threadIdx.x & 1;
    const int lo = side ? MI : 0, hi = side ? MT : MI;
    double mx = 0.0;
    for (int j = lo; j < hi; ++j) mx = fmax(mx, fabs(sq[g][j]));
    red[g][side][0] = mx > 0.0 ? mx / 1073741824.0 : 1.0;   // sigma = max/2^30
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * MT; i += blockDim.x) {
    const int g = i / MT, j = i % MT;
    const int side = j >= MI;
    const double sigma = red[g][side][0];
    const int jl = side ? j - MI : j;
    const double x = rint(sq[g][j] / (sigma * (double)(1 << (jl & 7))));
    si[g][j] = (int32_t)x;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int g = threadIdx.x >> 1, side = threadIdx.x & 1;
    const int lo = side ? MI : 0, hi = side ? MT : MI;
    double s = 0.0;
    for (int j = lo; j < hi; ++j) s += (double)si[g][j] * (double)(1 << ((j - lo) & 7));
    red[g][side][1] = s * red[g][side][0];
  }
  __syncthreads();
  // A fragments: element (row, k) of chunk c lives in lane (row%8)*4 + (k%16)/4,
  // reg (row>=8) + 2*(k>=16), byte k%4; row = digit*4 + query; k <-> sign bit p.
  for (int i = threadIdx.x; i < KC * 32; i += blockDim.x) {
    const int c = i / 32, lane = i % 32;
    const int gl = lane >> 2, ql = lane & 3;
    uint32_t regs[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int row = gl + ((r & 1) ? 8 : 0);
        const int k = ((r & 2) ? 16 : 0) + 4 * ql + b;
        const int qd = row & 3, digit = row >> 2;
        const int kk = k & 15;
        const int p = 8 * (kk & 3) + 2 * (kk >> 2) + (k >= 16 ? 1 : 0);
        const int side = c >= KCI;
        const int j = (side ? MI + (c - KCI) * 32 : c * 32) + p;
        int32_t x = si[qd][j];
        int8_t dg = 0;
#pragma unroll
        for (int t = 0; t <= 3; ++t) {
          const int8_t lo8 = (int8_t)(x & 0xFF);
          if (t == digit) dg = lo8;
          x = (x - (int32_t)lo8) >> 8;
        }
        v |= (uint32_t)(uint8_t)dg << (8 * b);
      }
      regs[r] = v;
    }
    afrag[((int64_t)u * KC + c) * 32 + lane] = make_uint4(regs[0], regs[1], regs[2], regs[3]);
  }
  if (threadIdx.x < 4) {
    const int g = threadIdx.x;
    const float ci = MI ? kEstimatorScale / (float)MI * inv_t * kLog2e : 0.f;
    const float co = MO ? kEstimatorScale / (float)MO * inv_t * kLog2e : 0.f;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (g < G) {
      v.x = (float)(2.0 * red[g][0][0] * ci);
      v.y = (float)(red[g][0][1] * ci);
      if (KCO) {
        v.z = (float)(2.0 * red[g][1][0] * co);
        v.w = (float)(red[g][1][1] * co);
      }
    }
    qconst[(int64_t)u * 4 + g] = v;
  }
}

// ----------------------------------------------------------------- main kernel
template <int KCI, int KCO>
__global__ void __launch_bounds__(kThreads, (KCI + KCO > 12) ? 1 : 2) k_decode_tc(const Params P) {
  using L = Layout<KCI, KCO>;
  constexpr int KC = KCI + KCO;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = P.ctas;
  const int64_t T = P.total_tiles;
  const int64_t r0 = tile_begin(blockIdx.x, T, C), r1 = tile_begin(blockIdx.x + 1, T, C);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kNW) {
    // ============================ producer =============================
    if (lane == 0) {
      const auto& kc = P.kc;
      const auto& vc = P.vc;
      for (int64_t t = r0; t < r1; ++t) {
        const int it = (int)(t - r0);
        const int s = it % kStages;
        if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
        const int u = (int)(t / P.tpu);
        const int64_t tok = (t % P.tpu) * kTile;
        const int64_t row = (int64_t)u * kc.capacity + tok;     // capacity % 128 == 0
        uint8_t* st = sm + s * L::kStageBytes;
        mbar_expect_tx(&full[s], L::kStageBytes);
        bulk_g2s(st + L::oBitsIn, kc.bits_in + row * (KCI * 4), L::kBitsIn, &full[s]);
        if (KCO) {
          bulk_g2s(st + L::oBitsOut, kc.bits_out + row * (KCO * 4), L::kBitsOut, &full[s]);
          bulk_g2s(st + L::oNormOut, kc.norm_out + row, L::kNorm, &full[s]);
        }
        bulk_g2s(st + L::oNormIn, kc.norm_in + row, L::kNorm, &full[s]);
        const int64_t vrow = (int64_t)u * vc.capacity + tok;
        bulk_g2s(st + L::oCodes, (const uint8_t*)vc.codes + vrow * 32, L::kCodes, &full[s]);
        bulk_g2s(st + L::oZero, (const uint8_t*)vc.zero + vrow * 8, L::kConst, &full[s]);
        bulk_g2s(st + L::oScale, (const uint8_t*)vc.scale + vrow * 8, L::kConst, &full[s]);
      }
    }
    return;
  }

  // ============================== consumers ==============================
  const int g = lane >> 2, q = lane & 3;
  const bool upper = g >= 4;          // lanes 16..31: digits 1/3, keep token 2q+1
  const int Q = g & 3;                // epilogue query of this lane
  const float wa = upper ? 256.f : 1.f, wb = upper ? 16777216.f : 65536.f;
  const uint32_t M0 = 0x01010101u << (2 * q), M1 = 0x02020202u << (2 * q);
  uint32_t* pbuf = reinterpret_cast<uint32_t*>(sm + L::oPbuf + warp * 2048);
  float* red = reinterpret_cast<float*>(sm + L::oRed);

  uint4 A[KC];
  float4 qc = make_float4(0.f, 0.f, 0.f, 0.f);
  float m_run = -INFINITY, l_run = 0.f;
  float Z[4] = {0.f, 0.f, 0.f, 0.f};   // sum_t p * zero_g   (lane's query Q)
  float Y[4] = {0.f, 0.f, 0.f, 0.f};   // sum_t p * scale_g  (HMMA offset removal)
  float acc[8][4];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
  int cur_u = -1;

  auto load_unit = [&](int u) {
#pragma unroll
    for (int c = 0; c < KC; ++c) A[c] = P.afrag[((int64_t)u * KC + c) * 32 + lane];
    qc = P.qconst[(int64_t)u * 4 + Q];
    m_run = -INFINITY;
    l_run = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) Z[i] = Y[i] = 0.f;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
  };

  auto flush = [&](int u) {
    // reduce l and Z over the 8 lanes sharing this lane's epilogue query
    constexpr int R = L::kRec;
    float l = l_run;
    float z[4] = {Z[0], Z[1], Z[2], Z[3]};
    float y[4] = {Y[0], Y[1], Y[2], Y[3]};
#pragma unroll
    for (int o = 1; o <= 16; o <<= 1) {
      if (o == 4 || o == 8) continue;
      l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        z[i] += __shfl_xor_sync(0xffffffffu, z[i], o);
        y[i] += __shfl_xor_sync(0xffffffffu, y[i], o);
      }
    }
    // Y of the accumulator query q (held by lane 4q, whose epilogue query is q)
    float yq[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) yq[i] = __shfl_sync(0xffffffffu, y[i], 4 * q);
    // per-warp record: [q][0]=m, [1]=l, [2..5]=Z, [6..133]=sum_t P' c
    float* rw = red + warp * 4 * R;
    if (q == 0 && !upper) {
      rw[Q * R + 0] = m_run;
      rw[Q * R + 1] = l;
#pragma unroll
      for (int i = 0; i < 4; ++i) rw[Q * R + 2 + i] = z[i];
    }
    // HMMA rows hold sum_t P' (1 + c 4^s / 1024), s = 3 (row g) or 4 (row g+8)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const float yg = yq[mt >> 1];
      rw[q * R + 6 + 16 * mt + g] = (acc[mt][0] + acc[mt][1] - yg) * 16.f;
      rw[q * R + 6 + 16 * mt + g + 8] = (acc[mt][2] + acc[mt][3] - yg) * 4.f;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kNW * 32) : "memory");
    const int tid = threadIdx.x;            // 0 .. kNW*32-1
    const int c0 = cta_of_tile((int64_t)u * P.tpu, T, C);
    const int slot = blockIdx.x - c0;
    for (int i = tid; i < P.G * 130; i += kNW * 32) {
      const int qq = i / 130, e = i % 130;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kNW; ++w) M = fmaxf(M, red[w * 4 * R + qq * R]);
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kNW; ++w) {
        const float* r = red + w * 4 * R + qq * R;
        const float f = (r[0] == -INFINITY) ? 0.f : ex2(r[0] - M);
        if (e == 1) v += f * r[1];
        else if (e >= 2) v += f * (r[6 + (e - 2)] + r[2 + ((e - 2) >> 5)]);
      }
      float* dst = P.part + (((int64_t)u * P.max_seg + slot) * P.G + qq) * 130;
      dst[e] = (e == 0) ? (M == -INFINITY ? -INFINITY : M * kLn2) : v;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kNW * 32) : "memory");
  };

  for (int64_t t = r0; t < r1; ++t) {
    const int it = (int)(t - r0);
    const int s = it % kStages;
    const int u = (int)(t / P.tpu);
    const int64_t tok0 = (t % P.tpu) * kTile + warp * 32;   // first token of this warp
    if (u != cur_u) {
      if (cur_u >= 0) flush(cur_u);
      load_unit(u);
      cur_u = u;
    }
    mbar_wait(&full[s], (it / kStages) & 1);
    const uint8_t* st = sm + s * L::kStageBytes;
    const uint32_t* bin = reinterpret_cast<const uint32_t*>(st + L::oBitsIn) + warp * 32 * KCI;
    const uint32_t* bout = reinterpret_cast<const uint32_t*>(st + L::oBitsOut) + warp * 32 * KCO;
    const __half* nin = reinterpret_cast<const __half*>(st + L::oNormIn) + warp * 32;
    const __half* nout = reinterpret_cast<const __half*>(st + L::oNormOut) + warp * 32;
    const uint32_t* codes = reinterpret_cast<const uint32_t*>(st + L::oCodes) + warp * 32 * 8;
    const uint2* zer = reinterpret_cast<const uint2*>(st + L::oZero) + warp * 32;
    const uint2* scl = reinterpret_cast<const uint2*>(st + L::oScale) + warp * 32;

    // -------------------- scores: 4 IMMA n-tiles of 8 tokens --------------------
    float lg[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int trow = 8 * j + g;                    // B column token of this lane
      uint32_t w_in[KCI], w_out[KCO > 0 ? KCO : 1];
#pragma unroll
      for (int c = 0; c < KCI; c += 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(bin + trow * KCI + c);
        w_in[c] = v.x; w_in[c + 1] = v.y; w_in[c + 2] = v.z; w_in[c + 3] = v.w;
      }
#pragma unroll
      for (int c = 0; c < KCO; c += 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(bout + trow * KCO + c);
        w_out[c] = v.x; w_out[c + 1] = v.y;
      }
      int di[4] = {0, 0, 0, 0}, dout[4] = {0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < KCI; ++c) imma(di, A[c], w_in[c] & M0, w_in[c] & M1);
#pragma unroll
      for (int c = 0; c < KCO; ++c) imma(dout, A[KCI + c], w_out[c] & M0, w_out[c] & M1);
      const float pi0 = (float)di[0] * wa + (float)di[2] * wb;   // token 2q
      const float pi1 = (float)di[1] * wa + (float)di[3] * wb;   // token 2q+1
      const float po0 = (float)dout[0] * wa + (float)dout[2] * wb;
      const float po1 = (float)dout[1] * wa + (float)dout[3] * wb;
      const float si = __shfl_xor_sync(0xffffffffu, upper ? pi0 : pi1, 16);
      const float so = __shfl_xor_sync(0xffffffffu, upper ? po0 : po1, 16);
      const float dot_in = (upper ? pi1 : pi0) + si;
      const float dot_out = (upper ? po1 : po0) + so;
      const int tk = 8 * j + 2 * q + (upper ? 1 : 0);
      const float nu_in = __half2float(nin[tk]);
      float l2 = nu_in * fmaf(qc.x, dot_in, -qc.y);
      if (KCO) l2 += __half2float(nout[tk]) * fmaf(qc.z, dot_out, -qc.w);
      lg[j] = (tok0 + tk < P.n) ? l2 : -INFINITY;
    }

    // -------------------- online softmax (log2 domain) --------------------
    float tmax = fmaxf(fmaxf(lg[0], lg[1]), fmaxf(lg[2], lg[3]));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
    const float m_new = fmaxf(m_run, tmax);
    const bool none = (m_new == -INFINITY);
    const float alpha = none ? 1.f : ex2(m_run - m_new);
    m_run = m_new;
    float p[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) p[j] = none ? 0.f : ex2(lg[j] - m_new);
    l_run = l_run * alpha + (p[0] + p[1]) + (p[2] + p[3]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      Z[i] *= alpha;
      Y[i] *= alpha;
    }
    const float a_acc = __shfl_sync(0xffffffffu, alpha, 4 * q);   // alpha of query q

    // -------------------- P' = p*scale (hi/lo fp16) -> per-warp B tiles ------
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int tk = 8 * j + 2 * q + (upper ? 1 : 0);
      const bool valid = tok0 + tk < P.n;
      const uint2 zr = zer[tk], sr = scl[tk];
      const float2 z01 = __half22float2(*reinterpret_cast<const __half2*>(&zr.x));
      const float2 z23 = __half22float2(*reinterpret_cast<const __half2*>(&zr.y));
      const float2 s01 = __half22float2(*reinterpret_cast<const __half2*>(&sr.x));
      const float2 s23 = __half22float2(*reinterpret_cast<const __half2*>(&sr.y));
      const float pj = p[j];
      const float zz[4] = {z01.x, z01.y, z23.x, z23.y};
      const float ss[4] = {s01.x, s01.y, s23.x, s23.y};
      float hi[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float Pp = valid ? pj * ss[i] : 0.f;
        Z[i] += valid ? pj * zz[i] : 0.f;
        Y[i] += Pp;
        const __half h = __float2half_rn(Pp);
        hi[i] = __half2float(h);
        lo[i] = Pp - hi[i];
      }
      const uint32_t h01 = pack_h2(hi[0], hi[1]), h23 = pack_h2(hi[2], hi[3]);
      const uint32_t l01 = pack_h2(lo[0], lo[1]), l23 = pack_h2(lo[2], lo[3]);
      // lower lanes keep hi of token 2q, upper lanes keep lo of token 2q+1
      const uint32_t snd0 = upper ? h01 : l01, snd1 = upper ? h23 : l23;
      const uint32_t rc0 = __shfl_xor_sync(0xffffffffu, snd0, 16);
      const uint32_t rc1 = __shfl_xor_sync(0xffffffffu, snd1, 16);
      uint4 wv;
      if (!upper) {   // hi column 2Q: {mine (token 2q), partner (token 2q+1)} per group
        wv.x = prmt(h01, rc0, 0x5410); wv.y = prmt(h01, rc0, 0x7632);
        wv.z = prmt(h23, rc1, 0x5410); wv.w = prmt(h23, rc1, 0x7632);
      } else {        // lo column 2Q+1: {partner (token 2q), mine (token 2q+1)}
        wv.x = prmt(rc0, l01, 0x5410); wv.y = prmt(rc0, l01, 0x7632);
        wv.z = prmt(rc1, l23, 0x5410); wv.w = prmt(rc1, l23, 0x7632);
      }
      const int ks = j >> 1, b = j & 1, gp = 2 * Q + (upper ? 1 : 0);
      *reinterpret_cast<uint4*>(pbuf + ((((ks * 8 + gp) * 4 + q) * 2 + b) * 4)) = wv;
    }
    __syncwarp();

    // -------------------- PV: 8 m-tiles x 2 k-steps of 16 tokens ---------------
    // Each tile's PV is accumulated by the tensor core from zero and folded into
    // the running fp32 accumulator with an IEEE FFMA that also applies the
    // online-softmax rescale.
    uint32_t xa[2], xb[2], ya[2], yb[2];
    uint32_t bg[4][2][2];   // [group][ks][b]
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int tb = 16 * ks + 2 * q;
      const uint32_t w0 = codes[(tb + 0) * 8 + g], w1 = codes[(tb + 1) * 8 + g];
      const uint32_t w8 = codes[(tb + 8) * 8 + g], w9 = codes[(tb + 9) * 8 + g];
      xa[ks] = prmt(w0, w1, 0x5410); xb[ks] = prmt(w0, w1, 0x7632);
      ya[ks] = prmt(w8, w9, 0x5410); yb[ks] = prmt(w8, w9, 0x7632);
      // per (ks, column g, quad q): 8 u32 laid out [b][grp]
      const uint4 B0 = *reinterpret_cast<const uint4*>(pbuf + ((ks * 8 + g) * 4 + q) * 8);
      const uint4 B1 = *reinterpret_cast<const uint4*>(pbuf + ((ks * 8 + g) * 4 + q) * 8 + 4);
      bg[0][ks][0] = B0.x; bg[1][ks][0] = B0.y; bg[2][ks][0] = B0.z; bg[3][ks][0] = B0.w;
      bg[0][ks][1] = B1.x; bg[1][ks][1] = B1.y; bg[2][ks][1] = B1.z; bg[3][ks][1] = B1.w;
    }
    // m-tile MT: rows g / g+8 use code slots 2*(MT&3) / +1 of half-word X (tokens
    // 2q, 2q+1) and Y (tokens 2q+8, 2q+9); one shift brings both to slots 3 / 4.
#define QJL_MT(MT, X, Y)                                                                         \
  {                                                                                              \
    float td[4] = {0.f, 0.f, 0.f, 0.f};                                                          \
    _Pragma("unroll") for (int ks = 0; ks < 2; ++ks) {                                           \
      const uint32_t xs = code_shift<(MT) & 3>(X[ks]), ys = code_shift<(MT) & 3>(Y[ks]);         \
      hmma(td, code_h2<3>(xs), code_h2<4>(xs), code_h2<3>(ys), code_h2<4>(ys),                   \
           bg[(MT) >> 1][ks][0], bg[(MT) >> 1][ks][1]);                                          \
    }                                                                                            \
    _Pragma("unroll") for (int i = 0; i < 4; ++i) acc[MT][i] = fmaf(acc[MT][i], a_acc, td[i]);  \
  }
    QJL_MT(0, xa, ya)
    QJL_MT(1, xa, ya)
    QJL_MT(2, xa, ya)
    QJL_MT(3, xa, ya)
    QJL_MT(4, xb, yb)
    QJL_MT(5, xb, yb)
    QJL_MT(6, xb, yb)
    QJL_MT(7, xb, yb)
#undef QJL_MT
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (cur_u >= 0) flush(cur_u);
}

// Merge per (unit, query): combine the unit's CTA-segment partials.
__global__ void k_merge_tc(const float* __restrict__ part, int max_seg, int G, int tpu, int64_t T, int C,
                           float* __restrict__ out, float* __restrict__ lse) {
  const int ug = blockIdx.x;
  const int u = ug / G, qq = ug % G;
  const int c0 = cta_of_tile((int64_t)u * tpu, T, C);
  const int c1 = cta_of_tile((int64_t)u * tpu + tpu - 1, T, C);
  const int ns = c1 - c0 + 1;
  float M = -INFINITY;
  for (int s = 0; s < ns; ++s) M = fmaxf(M, part[(((int64_t)u * max_seg + s) * G + qq) * 130]);
  float L = 0.f, a = 0.f;
  for (int s = 0; s < ns; ++s) {
    const float* W = part + (((int64_t)u * max_seg + s) * G + qq) * 130;
    if (W[0] == -INFINITY) continue;
    const float f = expf(W[0] - M);
    L += f * W[1];
    if (threadIdx.x < 128) a += f * W[2 + threadIdx.x];
  }
  if (threadIdx.x < 128) out[(int64_t)ug * 128 + threadIdx.x] = a / L;
  if (lse && threadIdx.x == 0) lse[ug] = M + logf(L);
}

struct Plan {
  int tpu, ctas, max_seg;
  int64_t T;
  size_t afrag_off, qconst_off, part_off, total;
};

template <int KCI, int KCO>
static int occupancy() {
  using L = Layout<KCI, KCO>;
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(k_decode_tc<KCI, KCO>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_decode_tc<KCI, KCO>, kThreads, L::kTotal);
    occ = o > 0 ? o : 1;
  }
  return occ;
}

static bool kc_dispatch(int kci, int kco, int* id) {
  const int pairs[][2] = {{8, 2}, {8, 4}, {8, 0}, {16, 2}, {16, 0}, {16, 4}};
  for (int i = 0; i < 6; ++i)
    if (pairs[i][0] == kci && pairs[i][1] == kco) { *id = i; return true; }
  return false;
}

static int occupancy_by_id(int id) {
  switch (id) {
    case 0: return occupancy<8, 2>();
    case 1: return occupancy<8, 4>();
    case 2: return occupancy<8, 0>();
    case 3: return occupancy<16, 2>();
    case 4: return occupancy<16, 0>();
    case 5: return occupancy<16, 4>();
  }
  return 1;
}

static Plan make_plan(const qjl_key_cache_t& kc, int64_t n, int G, int id) {
  Plan p;
  p.tpu = (int)((n + kTile - 1) / kTile);
  p.T = (int64_t)kc.units * p.tpu;
  const int64_t slots = (int64_t)device_sm_count() * occupancy_by_id(id);
  p.ctas = (int)(p.T < slots ? p.T : slots);
  int ms = 1;
  for (int u = 0; u < kc.units; ++u) {
    const int c0 = cta_of_tile((int64_t)u * p.tpu, p.T, p.ctas);
    const int c1 = cta_of_tile((int64_t)u * p.tpu + p.tpu - 1, p.T, p.ctas);
    ms = ms > c1 - c0 + 1 ? ms : c1 - c0 + 1;
  }
  p.max_seg = ms;
  const int KC = (kc.m_in + kc.m_out) / 32;
  p.afrag_off = 0;
  p.qconst_off = ((size_t)kc.units * KC * 32 * 16 + 255) / 256 * 256;
  p.part_off = p.qconst_off + ((size_t)kc.units * 4 * 16 + 255) / 256 * 256;
  p.total = p.part_off + (size_t)kc.units * p.max_seg * G * 130 * 4;
  return p;
}

}  // namespace tc

bool decode_tc_supported(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int G) {
  int id;
  return vc.layout == QJL_VLAYOUT_P2 && kc.d == 128 && G >= 1 && G <= 4 &&
         tc::kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id) && kc.capacity % tc::kTile == 0 &&
         vc.capacity % tc::kTile == 0 && getenv("QJL_FORCE_SIMT") == nullptr;
}

size_t decode_tc_workspace(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, int G) {
  int id;
  tc::kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id);
  (void)vc;
  return tc::make_plan(kc, n, G, id).total;
}

template <int KCI, int KCO>
static int launch_tc_impl(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n,
                          const void* q, int q_dtype, int G, const qjl_sketch_t& sk, float inv_t,
                          float* out, float* lse, void* ws, const tc::Plan& plan, cudaStream_t st) {
  using namespace tc;
  uint8_t* w = (uint8_t*)ws;
  uint4* afrag = (uint4*)(w + plan.afrag_off);
  float4* qconst = (float4*)(w + plan.qconst_off);
  float* part = (float*)(w + plan.part_off);
#define QJL_PREP(TQ, TS)                                                                         \
  k_prep<TQ, TS, KCI, KCO><<<kc.units, 256, 0, st>>>((const TQ*)q, G, (const TS*)sk.s_full,      \
                                                     sk.unit_stride, inv_t, afrag, qconst)
#define QJL_PREP_S(TQ)                                                   \
  switch (sk.dtype) {                                                    \
    case QJL_BF16: QJL_PREP(TQ, __nv_bfloat16); break;                   \
    case QJL_F16: QJL_PREP(TQ, __half); break;                           \
    case QJL_F32: QJL_PREP(TQ, float); break;                            \
    default: QJL_PREP(TQ, double); break;                                \
  }
  switch (q_dtype) {
    case QJL_BF16: QJL_PREP_S(__nv_bfloat16); break;
    case QJL_F16: QJL_PREP_S(__half); break;
    case QJL_F32: QJL_PREP_S(float); break;
    default: QJL_PREP_S(double); break;
  }
#undef QJL_PREP_S
#undef QJL_PREP
  QJL_LAUNCH_CHECK("decode_tc_prep");
  Params P;
  P.kc = kc;
  P.vc = vc;
  P.n = n;
  P.G = G;
  P.units = kc.units;
  P.tpu = plan.tpu;
  P.total_tiles = plan.T;
  P.ctas = plan.ctas;
  P.max_seg = plan.max_seg;
  P.afrag = afrag;
  P.qconst = qconst;
  P.part = part;
  occupancy<KCI, KCO>();
  timing_begin(st);
  k_decode_tc<KCI, KCO><<<plan.ctas, kThreads, Layout<KCI, KCO>::kTotal, st>>>(P);
  timing_end(st);
  QJL_LAUNCH_CHECK("decode_tc");
  k_merge_tc<<<kc.units * G, 128, 0, st>>>(part, plan.max_seg, G, plan.tpu, plan.T, plan.ctas, out, lse);
  QJL_LAUNCH_CHECK("decode_tc_merge");
  return QJL_OK;
}

int launch_decode_tc(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, const void* q,
                     int q_dtype, int G, const qjl_sketch_t& sk, float inv_t, float* out, float* lse,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
  int id;
  if (!tc::kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id)) return QJL_ERR_UNSUPPORTED;
  const tc::Plan plan = tc::make_plan(kc, n, G, id);
  if (ws_bytes < plan.total) {
    set_error("decode workspace needs %zu bytes", plan.total);
    return QJL_ERR_WORKSPACE;
  }
  switch (id) {
    case 0: return launch_tc_impl<8, 2>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, st);
    case 1: return launch_tc_impl<8, 4>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, st);
    case 2: return launch_tc_impl<8, 0>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, st);
    case 3: return launch_tc_impl<16, 2>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, st);
    case 4: return launch_tc_impl<16, 0>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, st);
    case 5: return launch_tc_impl<16, 4>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, st);
  }
  return QJL_ERR_UNSUPPORTED;
}

}  // namespace qjl
