// Tensor-core fused QJL decode (K2 score estimator + K3 online softmax . V) for
// P2 value caches on sm_100a -- v5.
//
// One decode step = 2 launches chained with programmatic dependent launch:
//   k_prep   one CTA per unit: Sq = S_full . q for the unit's G <= 4 query heads,
//            quantized to a 32-bit fixed-point integer and split into four int8
//            digits laid out as the score IMMA's B fragments; zeroes the unit's
//            merge counter.
//   k_decode stream-K over the flattened (unit, 128-token tile) space; each CTA
//            folds its segment of a unit into one partial, and the CTA that
//            finishes a unit last (atomic counter) merges the unit's partials and
//            writes out / lse -- no separate merge launch.
//
// Inside k_decode (4 warps, 32 tokens per warp per stage):
//  * Data movement: thread 0 streams every 128-token tile of the packed cache
//    (sign bits, fp16 norms, 2-bit codes, fp16 zero/scale) HBM -> smem with
//    cp.async.bulk into a kStages mbarrier ring, kLookahead tiles ahead.
//  * Scores (estimator.py:149-170, 2*sum_set(Sq) - sum(Sq)): m16n8k32 IMMA, A = the
//    packed sign word masked in place (`w & 0x01010101 << 2q`: four sign bits ->
//    four u8 lanes of value 2^(2q)*bit), B = the query-sketch digits; one IMMA =
//    16 tokens x 32 bits x 4 query heads x 2 digits, exact int32 accumulation.
//  * PV (attention.py:71 over kvcache.py:164-166 dequantization):
//      out[q][d] = sum_t p[t][q] zero[t][g(d)] + sum_t P'[t][q][g(d)] c[t][d],
//    P' = p * scale.  The code term is an m16n8k32 IMMA as well: A = one P2 code
//    word masked in place (`w & 3 << 2s` per byte: 4 tokens x 1 dim, value c*4^s,
//    the 4^s row weight is divided out at the end), B = P' in 24-bit fixed point
//    relative to the tile's bound ptop * max(scale), split into three balanced
//    int8 digits by one FFMA (float magic-number rounding) and PRMTs: lo/mid in
//    one n-tile, hi in a second.  Exact int32 accumulation per tile, FFMA2 into
//    the fp32 running sum.  (16-bit P' was measured at 2e-4 relative error on flat
//    softmaxes: tokens below 2^-16 of the tile bound round to zero.)
//  * Online softmax in the log2 domain per query head; running state is rescaled
//    only when some head's maximum moved (warp-uniform branch).
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace qjl {
namespace tc {

constexpr int kNW = 4;             // warps per CTA (all compute; thread 0 also issues copies)
constexpr int kTile = 32 * kNW;    // tokens per pipeline stage
#ifndef QJL_DEC_STAGES
#define QJL_DEC_STAGES 4
#endif
#ifndef QJL_DEC_LOOKAHEAD
#define QJL_DEC_LOOKAHEAD 2
#endif
constexpr int kStages = QJL_DEC_STAGES;
// tiles in flight ahead of the one being consumed; kStages - kLookahead - 1 tiles of
// slack let the issuing warp run ahead of the slowest warp without blocking
constexpr int kLookahead = QJL_DEC_LOOKAHEAD;
#ifndef QJL_DEC_MINB
#define QJL_DEC_MINB 3
#endif
constexpr int kThreads = 32 * kNW;
constexpr int kRec = 130;          // per (partial, query): m (log2 domain), l, out[128]
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kPMax = 8.0e6f;                  // P' fixed-point full scale (< 2^23 - 32896)
constexpr float kMagic = 8421504.f;              // 2^23 + 32896 (see the P' digits)

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
  const uint4* afrag;    // [units][KC][32 lanes] score B fragments (4 x u32)
  const float4* qconst;  // [units][4 queries] {k_in, b_in, k_out, b_out}
  float* part;           // [units][max_seg][G][kRec]
  int* counters;         // [units] finished segments (zeroed by k_prep)
  float* out;            // [units][G][128]
  float* lse;            // [units][G] or null
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
// D += A(u8) . B(s8), m16n8k32
__device__ __forceinline__ void imma_u8s8(int* d, const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}
// D = A(u8) . B(s8), m16n8k32, zero accumulator
__device__ __forceinline__ void imma_u8s8_z(int* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                            uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};\n"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0));
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
// packed fp32 FMA (sm_100 FFMA2): d = a * b + c elementwise
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rc, {%6, %7};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 h2f2(uint32_t h) {
  return __half22float2(*reinterpret_cast<const __half2*>(&h));
}
__device__ __forceinline__ uint32_t hmax2u(uint32_t a, uint32_t b) {
  __half2 r = __hmax2(*reinterpret_cast<const __half2*>(&a), *reinterpret_cast<const __half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
template <int K>
__device__ __forceinline__ uint32_t word_of(const uint4& v) {
  if constexpr (K == 0) return v.x;
  else if constexpr (K == 1) return v.y;
  else if constexpr (K == 2) return v.z;
  else return v.w;
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
  static constexpr int kBbufWarp = 1536;                          // P' B fragments: lo/mid 1 KB, hi 512 B
  static constexpr int oBbuf = kStages * kStageBytes;
  static constexpr int oBq = oBbuf + kNW * kBbufWarp;              // score B fragments [KC][32 lanes] x 16 B
  static constexpr int kBq = (KCI + KCO) * 32 * 16;
  static constexpr int oRed = oBbuf;                               // flush scratch aliases both
  static constexpr int kRedBytes = kNW * 4 * kRec * 4;
  static constexpr int kScratch = kRedBytes > kNW * kBbufWarp + kBq ? kRedBytes : kNW * kBbufWarp + kBq;
  static constexpr int oFlag = oBbuf + kScratch;
  static constexpr int oBar = oFlag + 16;
  static constexpr int kTotal = oBar + 2 * kStages * 8;
};

// ----------------------------------------------------------------- prep kernel
// One CTA per unit, one thread per sketch row: Sq = S_full . q (fp32 products of
// the 16-bit operands, exact; fp64 for wider sketches), per-side sigma =
// max|Sq| / 2^30, weighted integer sketch x_j = rint(Sq_j / (sigma * 2^(j mod 8))),
// 4 signed-byte digits laid out as the IMMA B operand: column n of n-tile nt =
// (query n/2, digit 2*nt + n%2).
template <typename A, typename T>
__device__ __forceinline__ A to_acc(T x) {
  if constexpr (std::is_same<A, float>::value) return to_f32(x);
  else return to_f64(x);
}

template <typename TQ, typename TS, int KCI, int KCO>
__global__ void __launch_bounds__(640) k_prep(const TQ* __restrict__ q, int G, const TS* __restrict__ s_full,
                                              int64_t s_unit_stride, float inv_t, uint4* __restrict__ bfrag,
                                              float4* __restrict__ qconst, int* __restrict__ counters) {
  constexpr int MI = KCI * 32, MO = KCO * 32, MT = MI + MO, KC = KCI + KCO;
  constexpr int d = 128;
  using acc_t = typename std::conditional<(sizeof(TS) <= 2), float, double>::type;
  __shared__ acc_t qs[4][d];
  __shared__ float sq[4][MT];
  __shared__ int32_t si[4][MT];
  __shared__ unsigned int mxbits[4][2];
  __shared__ double red[4][2][2];   // [q][side][sigma, sum]
  const int u = blockIdx.x;
  const TS* S = s_full + (int64_t)u * s_unit_stride;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int i = threadIdx.x; i < 4 * d; i += blockDim.x) {
    const int g = i / d;
    qs[g][i % d] = g < G ? to_acc<acc_t>(q[((int64_t)u * G + g) * d + i % d]) : (acc_t)0;
  }
  if (threadIdx.x < 8) mxbits[threadIdx.x >> 1][threadIdx.x & 1] = 0u;
  if (threadIdx.x == 0) counters[u] = 0;
  __syncthreads();
  {
    const int r = threadIdx.x;               // blockDim.x == MT
    const TS* row = S + (int64_t)r * d;
    constexpr int EPV = 16 / (int)sizeof(TS);
    acc_t a[4] = {0, 0, 0, 0};
#pragma unroll 4
    for (int e0 = 0; e0 < d; e0 += EPV) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(row + e0));
      const TS* sv = reinterpret_cast<const TS*>(&raw);
#pragma unroll
      for (int k = 0; k < EPV; ++k) {
        const acc_t s = to_acc<acc_t>(sv[k]);
#pragma unroll
        for (int g = 0; g < 4; ++g) a[g] = fma(s, qs[g][e0 + k], a[g]);
      }
    }
    float wm[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      sq[g][r] = (float)a[g];
      wm[g] = warp_max(fabsf((float)a[g]));   // rows of a warp are on one side (MI % 32 == 0)
    }
    if (lane == 0) {
      const int side = r >= MI;
#pragma unroll
      for (int g = 0; g < 4; ++g) atomicMax(&mxbits[g][side], __float_as_uint(wm[g]));
    }
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int g = threadIdx.x >> 1, side = threadIdx.x & 1;
    const double mx = (double)__uint_as_float(mxbits[g][side]);
    red[g][side][0] = mx > 0.0 ? mx / 1073741824.0 : 1.0;   // sigma = max/2^30
  }
  __syncthreads();
  // integer sketch; one warp per (query, side) segment, warp-reduced checksum
  for (int seg = wid; seg < 8; seg += nwarp) {
    const int g = seg >> 1, side = seg & 1;
    const int lo = side ? MI : 0, hi = side ? MT : MI;
    const double inv = 1.0 / red[g][side][0];
    long long acc = 0;
    for (int j = lo + lane; j < hi; j += 32) {
      const int sh = (j - lo) & 7;
      const int32_t x = (int32_t)rint((double)sq[g][j] * inv / (double)(1 << sh));
      si[g][j] = x;
      acc += (long long)x * (1ll << sh);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[g][side][1] = (double)acc * red[g][side][0];
  }
  __syncthreads();
  // B fragment of m16n8k32: element (k, n) lives in lane n*4 + (k%16)/4, reg
  // (k >= 16), byte k%4.  k <-> sign bit p of the chunk word: k = 4q + i holds
  // bit 8i + 2q, k = 16 + 4q + i holds bit 8i + 2q + 1 (the A side masks the
  // sign word with 0x01010101 << 2q / 0x02020202 << 2q).
  for (int i = threadIdx.x; i < KC * 32; i += blockDim.x) {
    const int c = i / 32, ln = i % 32;
    const int n = ln >> 2, ql = ln & 3;
    const int qd = n >> 1;
    uint32_t regs[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {          // r = nt*2 + reg
      const int nt = r >> 1, reg = r & 1;
      const int digit = 2 * nt + (n & 1);
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int p = 8 * b + 2 * ql + reg;
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
    bfrag[((int64_t)u * KC + c) * 32 + ln] = make_uint4(regs[0], regs[1], regs[2], regs[3]);
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
// Token order inside a warp's 32-token slice: score m-tile h covers tokens
// 16h..16h+15 (IMMA rows), so lane g (= lane >> 2) scores tokens g + 8i, i = 0..3,
// for query head q = lane & 3.  The PV IMMA takes k = 4j + i <-> token j + 8i, so
// the four P' digits a score lane produces for one query form exactly one B
// register (k-block j = g) -- only a 1 KB per-warp smem transpose to the B
// fragment lanes is needed, no shuffles.
template <int KCI, int KCO>
__global__ void __launch_bounds__(kThreads, (KCI + KCO > 12) ? 2 : QJL_DEC_MINB) k_decode_tc(const Params P) {
  using L = Layout<KCI, KCO>;
  constexpr int KC = KCI + KCO;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = P.ctas;
  const int64_t T = P.total_tiles;
  const int64_t r0 = tile_begin(blockIdx.x, T, C), r1 = tile_begin(blockIdx.x + 1, T, C);
  const int ntiles = (int)(r1 - r0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // (unit, tile-in-unit) of the first tile; advanced incrementally (no 64-bit div per tile)
  const int u_first = (int)(r0 / P.tpu);
  const int lt_first = (int)(r0 - (int64_t)u_first * P.tpu);
  int iss_u = u_first, iss_lt = lt_first, iss_i = 0;     // issuer cursor (thread 0 only)
  auto issue_next = [&]() {   // bulk-copy tile r0 + iss_i into stage iss_i % kStages
    const int i = iss_i;
    const int s = i % kStages;
    if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
    const int64_t tok = (int64_t)iss_lt * kTile;
    const int64_t row = (int64_t)iss_u * P.kc.capacity + tok;     // capacity % 128 == 0
    const int64_t vrow = (int64_t)iss_u * P.vc.capacity + tok;
    uint8_t* st = sm + s * L::kStageBytes;
    mbar_expect_tx(&full[s], L::kStageBytes);
    bulk_g2s(st + L::oBitsIn, P.kc.bits_in + row * (KCI * 4), L::kBitsIn, &full[s]);
    if (KCO) {
      bulk_g2s(st + L::oBitsOut, P.kc.bits_out + row * (KCO * 4), L::kBitsOut, &full[s]);
      bulk_g2s(st + L::oNormOut, P.kc.norm_out + row, L::kNorm, &full[s]);
    }
    bulk_g2s(st + L::oNormIn, P.kc.norm_in + row, L::kNorm, &full[s]);
    bulk_g2s(st + L::oCodes, (const uint8_t*)P.vc.codes + vrow * 32, L::kCodes, &full[s]);
    bulk_g2s(st + L::oZero, (const uint8_t*)P.vc.zero + vrow * 8, L::kConst, &full[s]);
    bulk_g2s(st + L::oScale, (const uint8_t*)P.vc.scale + vrow * 8, L::kConst, &full[s]);
    ++iss_i;
    if (++iss_lt == P.tpu) { iss_lt = 0; ++iss_u; }
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < kLookahead && i < ntiles; ++i) issue_next();

  const int g = lane >> 2, q = lane & 3;      // q = this lane's query head (scores)
  const uint32_t M0 = 0x01010101u << (2 * q), M1 = 0x02020202u << (2 * q);
  uint32_t* bbuf = reinterpret_cast<uint32_t*>(sm + L::oBbuf + warp * L::kBbufWarp);
  uint32_t* hbuf = bbuf + 256;
  float* red = reinterpret_cast<float*>(sm + L::oRed);
  // P' B-fragment transpose (16-byte chunks of bbuf, bank-conflict free both ways):
  // source lane (g, q) holds k-block j = g of columns n = 2q (lo digit) / 2q + 1 (hi);
  // it belongs to B-fragment lane (n, g & 3), register b = g >> 2.
  const int wlo = (2 * q + (g >> 2)) * 8 + (((g & 3) + 2 * q) & 7);
  const int whi = (2 * q + (g >> 2)) * 8 + ((4 + (g & 3) + 2 * q) & 7);
  const int rb0 = ((lane >> 3) * 2) * 8 + ((lane + 2 * (lane >> 3)) & 7);
  // hi digits: only the even columns n = 2q of the second n-tile are used; chunk of
  // (query qq, k-lane qp, register b) = (2b + (qp >> 1)) * 8 + ((2qq + qp) & 7)
  const int whh = (2 * (g >> 2) + ((g & 3) >> 1)) * 8 + ((2 * q + (g & 3)) & 7);
  const int rh0 = (((lane & 3) >> 1)) * 8 + ((2 * (lane >> 3) + (lane & 3)) & 7);
  const bool hcol = ((lane >> 2) & 1) == 0;
  // P2 code words of this lane: k-blocks q and 4 + q of fragment row g
  const int cw0 = g * 8 + (q ^ ((g & 1) << 2));
  const int cw1 = g * 8 + ((4 + q) ^ ((g & 1) << 2));

  const uint4* bqs = reinterpret_cast<const uint4*>(sm + L::oBq) + lane;   // [c][32 lanes]
  float4 qc = make_float4(0.f, 0.f, 0.f, 0.f);
  float m_run = -INFINITY, l_run = 0.f;
  float2 Z01 = make_float2(0.f, 0.f), Z23 = make_float2(0.f, 0.f);   // sum_t p * zero_g
  float2 acc[8];                              // [MT] rows g / g + 8 of the PV m-tile, query q

  auto load_unit = [&](int u) {
    // the unit's query-sketch digits (score IMMA B operand) -> smem; every warp is past
    // the previous unit (flush ends with a CTA barrier)
    for (int i = threadIdx.x; i < KC * 32; i += kThreads)
      reinterpret_cast<uint4*>(sm + L::oBq)[i] = P.afrag[(int64_t)u * KC * 32 + i];
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
    qc = P.qconst[(int64_t)u * 4 + q];
    m_run = -INFINITY;
    l_run = 0.f;
    Z01 = Z23 = make_float2(0.f, 0.f);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) acc[mt] = make_float2(0.f, 0.f);
  };

  auto flush = [&](int u) {
    // l and Z: reduce over the 8 lanes of query q (lanes q + 4g)
    float l = l_run;
    float z[4] = {Z01.x, Z01.y, Z23.x, Z23.y};
#pragma unroll
    for (int o = 4; o <= 16; o <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
      for (int i = 0; i < 4; ++i) z[i] += __shfl_xor_sync(0xffffffffu, z[i], o);
    }
    // the record scratch aliases the P' transpose buffers: every warp must be done
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
    float* rw = red + (warp * 4 + q) * kRec;
    if (g == 0) {
      rw[0] = m_run;
      rw[1] = l;
    }
    // PV row (MT, r) = dim 16 MT + g + 8 r carries weight 4^(2 (MT & 1) + r)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const float w0 = (mt & 1) ? (1.f / 16.f) : 1.f;
      rw[2 + 16 * mt + g] = fmaf(acc[mt].x, w0, z[mt >> 1]);
      rw[2 + 16 * mt + g + 8] = fmaf(acc[mt].y, w0 * 0.25f, z[mt >> 1]);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
    const int c0 = cta_of_tile((int64_t)u * P.tpu, T, C);
    const int c1 = cta_of_tile((int64_t)u * P.tpu + P.tpu - 1, T, C);
    const int ns = c1 - c0 + 1, slot = blockIdx.x - c0;
    float* mypart = P.part + ((int64_t)u * P.max_seg + slot) * P.G * kRec;
    for (int i = threadIdx.x; i < P.G * kRec; i += kThreads) {
      const int qq = i / kRec, e = i % kRec;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kNW; ++w) M = fmaxf(M, red[(w * 4 + qq) * kRec]);
      float v = M;
      if (e) {
        v = 0.f;
#pragma unroll
        for (int w = 0; w < kNW; ++w) {
          const float* r = red + (w * 4 + qq) * kRec;
          const float f = (r[0] == -INFINITY) ? 0.f : ex2(r[0] - M);
          v = fmaf(f, r[e], v);
        }
      }
      mypart[i] = v;
    }
    int* flag = reinterpret_cast<int*>(sm + L::oFlag);
    if (ns > 1) {
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
      if (threadIdx.x == 0) *flag = (atomicAdd(&P.counters[u], 1) == ns - 1);
      asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
      if (!*flag) return;
      __threadfence();
    } else {
      asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
    }
    // this CTA finished the unit last: merge its ns partials
    const float* up = P.part + (int64_t)u * P.max_seg * P.G * kRec;
    for (int i = threadIdx.x; i < P.G * 128; i += kThreads) {
      const int qq = i >> 7, dim = i & 127;
      float M = -INFINITY;
      for (int s = 0; s < ns; ++s) M = fmaxf(M, __ldcg(up + (s * P.G + qq) * kRec));
      float Ls = 0.f, a = 0.f;
      for (int s = 0; s < ns; ++s) {
        const float* W = up + (s * P.G + qq) * kRec;
        const float ms = __ldcg(W);
        if (ms == -INFINITY) continue;
        const float f = ex2(ms - M);
        Ls = fmaf(f, __ldcg(W + 1), Ls);
        a = fmaf(f, __ldcg(W + 2 + dim), a);
      }
      P.out[((int64_t)u * P.G + qq) * 128 + dim] = a / Ls;
      if (P.lse && dim == 0) P.lse[(int64_t)u * P.G + qq] = (M + __log2f(Ls)) * kLn2;
    }
  };

  // one 32-token warp slice; MASK: some tokens are >= n (tail tile of a unit)
  auto tile = [&](const uint8_t* st, const int64_t tok0, auto mask_tag) {
    constexpr bool MASK = decltype(mask_tag)::value;
    const uint32_t* bin = reinterpret_cast<const uint32_t*>(st + L::oBitsIn) + warp * 32 * KCI;
    const uint32_t* bout = reinterpret_cast<const uint32_t*>(st + L::oBitsOut) + warp * 32 * KCO;
    const __half* nin = reinterpret_cast<const __half*>(st + L::oNormIn) + warp * 32;
    const __half* nout = reinterpret_cast<const __half*>(st + L::oNormOut) + warp * 32;
    const uint4* codes = reinterpret_cast<const uint4*>(st + L::oCodes + warp * 1024);
    const uint2* zer = reinterpret_cast<const uint2*>(st + L::oZero) + warp * 32;
    const uint2* scl = reinterpret_cast<const uint2*>(st + L::oScale) + warp * 32;

    // -------- scores: 2 IMMA m-tiles of 16 tokens (rows g, g+8) x 2 n-tiles -------
    // D[token][2q + i] of n-tile nt = digit 2nt+i of query q: every lane ends up
    // with all four digits of its own query for tokens g + 8i -- no shuffles.
    float lg[4];                       // token g + 8i
    {
      // both m-tiles at once: four independent accumulator chains per n-tile pair
      int din[2][2][4] = {}, dout[2][2][4] = {};      // [m-tile h][n-tile][reg]
#pragma unroll
      for (int c = 0; c < KCI; c += 4) {
        uint4 v[4];                                   // tokens g + 8k
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<const uint4*>(bin + (g + 8 * k) * KCI + c);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint4 bq = bqs[(c + e) * 32];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t wa = e == 0 ? v[2 * h].x : e == 1 ? v[2 * h].y : e == 2 ? v[2 * h].z : v[2 * h].w;
            const uint32_t wb = e == 0 ? v[2 * h + 1].x : e == 1 ? v[2 * h + 1].y
                              : e == 2 ? v[2 * h + 1].z : v[2 * h + 1].w;
            const uint4 a = make_uint4(wa & M0, wb & M0, wa & M1, wb & M1);
            imma_u8s8(din[h][0], a, bq.x, bq.y);
            imma_u8s8(din[h][1], a, bq.z, bq.w);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < KCO; c += 2) {
        uint2 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<const uint2*>(bout + (g + 8 * k) * KCO + c);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint4 bq = bqs[(KCI + c + e) * 32];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t wa = e == 0 ? v[2 * h].x : v[2 * h].y;
            const uint32_t wb = e == 0 ? v[2 * h + 1].x : v[2 * h + 1].y;
            const uint4 a = make_uint4(wa & M0, wb & M0, wa & M1, wb & M1);
            imma_u8s8(dout[h][0], a, bq.x, bq.y);
            imma_u8s8(dout[h][1], a, bq.z, bq.w);
          }
        }
      }
      // D[token][2q + i] of n-tile nt = digit 2nt+i of query q: rows g (regs 0, 1) and
      // g + 8 (regs 2, 3) of m-tile h = tokens g + 16h and g + 16h + 8
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int tk = g + 16 * h + 8 * e;
          // |digit partial| <= 2^21, so d0 + 256 d1 and d2 + 256 d3 are exact in int32
          const float din_f = fmaf((float)(din[h][1][2 * e] + 256 * din[h][1][2 * e + 1]), 65536.f,
                                   (float)(din[h][0][2 * e] + 256 * din[h][0][2 * e + 1]));
          float l2 = __half2float(nin[tk]) * fmaf(qc.x, din_f, -qc.y);
          if (KCO) {
            const float dout_f = fmaf((float)(dout[h][1][2 * e] + 256 * dout[h][1][2 * e + 1]), 65536.f,
                                      (float)(dout[h][0][2 * e] + 256 * dout[h][0][2 * e + 1]));
            l2 = fmaf(__half2float(nout[tk]), fmaf(qc.z, dout_f, -qc.w), l2);
          }
          lg[2 * h + e] = (!MASK || tok0 + tk < P.n) ? l2 : -INFINITY;
        }
      }
    }

    // -------------------- online softmax (log2 domain, query q) --------------------
    float tmax = fmaxf(fmaxf(lg[0], lg[1]), fmaxf(lg[2], lg[3]));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
    const float m_new = fmaxf(m_run, tmax);
    // nothing valid yet in this unit (every query head sees the same valid tokens,
    // so this is warp-uniform)
    if (MASK && m_new == -INFINITY) return;
    const float alpha = ex2(m_run - m_new);
    m_run = m_new;
    float p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = ex2(lg[i] - m_new);
    const float ptop = ex2(tmax - m_new);     // largest p of the tile for this query

    // value constants of this lane's tokens g + 8i (fp16 x 4 groups)
    uint2 zr[4], sr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      zr[i] = zer[g + 8 * i];
      sr[i] = scl[g + 8 * i];
      if (MASK && tok0 + g + 8 * i >= P.n) zr[i] = sr[i] = make_uint2(0u, 0u);  // rows past n
    }
    // tile bound of the value scales (query independent): fp16x2 max tree + 3 shuffles
    uint32_t hm = hmax2u(hmax2u(hmax2u(sr[0].x, sr[0].y), hmax2u(sr[1].x, sr[1].y)),
                         hmax2u(hmax2u(sr[2].x, sr[2].y), hmax2u(sr[3].x, sr[3].y)));
    hm = hmax2u(hm, __shfl_xor_sync(0xffffffffu, hm, 4));
    hm = hmax2u(hm, __shfl_xor_sync(0xffffffffu, hm, 8));
    hm = hmax2u(hm, __shfl_xor_sync(0xffffffffu, hm, 16));
    const float2 hmf = h2f2(hm);
    const float bound = ptop * fmaxf(hmf.x, hmf.y);      // >= every P' of query q in the tile
    const float K = bound > 0.f ? __fdividef(kPMax, bound) : 0.f;
    const float invK = bound * (1.f / kPMax);

    // rescale the running state only when some head's maximum moved
    if (__any_sync(0xffffffffu, alpha != 1.f)) {
      const float2 a2 = make_float2(alpha, alpha), z2 = make_float2(0.f, 0.f);
      l_run *= alpha;
      Z01 = fma2(Z01, a2, z2);
      Z23 = fma2(Z23, a2, z2);
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) acc[mt] = fma2(acc[mt], a2, z2);
    }
    l_run += (p[0] + p[1]) + (p[2] + p[3]);

    // -------- P' = p * scale in 24-bit fixed point -> three int8 digits per token --------
    // fma(p K, scale, 2^23 + 32896) leaves u = v + 32896 (v = rint(P' K) in [0, 8e6]) in
    // the 23 mantissa bits: v = 65536 hi + 256 mid + lo with balanced lo, mid in
    // [-128, 127]; byte 0 ^ 0x80 = lo, byte 1 ^ 0x80 = mid, byte 2 = hi.
    uint32_t wlo4[4], wmid4[4], whi4[4];
    {
      uint32_t wv[4][4];                  // [token i][group]
      const float2 mg = make_float2(kMagic, kMagic);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float pk = p[i] * K;
        const float2 pk2 = make_float2(pk, pk), pp = make_float2(p[i], p[i]);
        const float2 s01 = h2f2(sr[i].x), s23 = h2f2(sr[i].y);
        const float2 z01 = h2f2(zr[i].x), z23 = h2f2(zr[i].y);
        const float2 w01 = fma2(pk2, s01, mg), w23 = fma2(pk2, s23, mg);
        wv[i][0] = __float_as_uint(w01.x);
        wv[i][1] = __float_as_uint(w01.y);
        wv[i][2] = __float_as_uint(w23.x);
        wv[i][3] = __float_as_uint(w23.y);
        Z01 = fma2(pp, z01, Z01);
        Z23 = fma2(pp, z23, Z23);
      }
#pragma unroll
      for (int G = 0; G < 4; ++G) {
        const uint32_t p01 = prmt(wv[0][G], wv[1][G], 0x5140);
        const uint32_t p23 = prmt(wv[2][G], wv[3][G], 0x5140);
        const uint32_t h01 = prmt(wv[0][G], wv[1][G], 0x0062);
        const uint32_t h23 = prmt(wv[2][G], wv[3][G], 0x0062);
        wlo4[G] = prmt(p01, p23, 0x5410) ^ 0x80808080u;
        wmid4[G] = prmt(p01, p23, 0x7632) ^ 0x80808080u;
        whi4[G] = prmt(h01, h23, 0x5410);
      }
    }
    reinterpret_cast<uint4*>(bbuf)[wlo] = make_uint4(wlo4[0], wlo4[1], wlo4[2], wlo4[3]);
    reinterpret_cast<uint4*>(bbuf)[whi] = make_uint4(wmid4[0], wmid4[1], wmid4[2], wmid4[3]);
    reinterpret_cast<uint4*>(hbuf)[whh] = make_uint4(whi4[0], whi4[1], whi4[2], whi4[3]);
    __syncwarp();
    const uint4 B0 = reinterpret_cast<const uint4*>(bbuf)[rb0];       // k 4q' .. : groups 0..3
    const uint4 B1 = reinterpret_cast<const uint4*>(bbuf)[rb0 + 8];   // k 16 + 4q' ..
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
    const uint4 H0 = hcol ? reinterpret_cast<const uint4*>(hbuf)[rh0] : z4;
    const uint4 H1 = hcol ? reinterpret_cast<const uint4*>(hbuf)[rh0 + 16] : z4;
    const uint4 W0 = codes[cw0], W1 = codes[cw1];

    // -------------------- PV: 8 m-tiles (16 dims) x K = 32 tokens ---------------
    const float2 ik = make_float2(invK, invK), k65536 = make_float2(65536.f, 65536.f);
#define QJL_PV(MT)                                                                            \
    {                                                                                         \
      constexpr uint32_t mk0 = 0x03030303u << (4 * ((MT) & 1));                               \
      constexpr uint32_t mk1 = mk0 << 2;                                                      \
      const uint32_t x0 = word_of<((MT) >> 1)>(W0), x1 = word_of<((MT) >> 1)>(W1);                \
      int dd[4], dh[4];                                                                       \
      imma_u8s8_z(dd, x0 & mk0, x0 & mk1, x1 & mk0, x1 & mk1, word_of<((MT) >> 1)>(B0),        \
                  word_of<((MT) >> 1)>(B1));                                                  \
      imma_u8s8_z(dh, x0 & mk0, x0 & mk1, x1 & mk0, x1 & mk1, word_of<((MT) >> 1)>(H0),        \
                  word_of<((MT) >> 1)>(H1));                                                  \
      const float2 v = fma2(make_float2((float)dh[0], (float)dh[2]), k65536,                  \
                            make_float2((float)(dd[0] + 256 * dd[1]), (float)(dd[2] + 256 * dd[3]))); \
      acc[MT] = fma2(v, ik, acc[MT]);                                                         \
    }
    QJL_PV(0)
    QJL_PV(1)
    QJL_PV(2)
    QJL_PV(3)
    QJL_PV(4)
    QJL_PV(5)
    QJL_PV(6)
    QJL_PV(7)
#undef QJL_PV
    __syncwarp();
  };

  // everything above only touched the cache stream; the query sketch digits come from
  // k_prep, launched just before us with programmatic dependent launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int cur_u = -1;
  int u = u_first, lt = lt_first;
  for (int it = 0; it < ntiles; ++it) {
    const int s = it % kStages;
    if (u != cur_u) {
      if (cur_u >= 0) flush(cur_u);
      load_unit(u);
      cur_u = u;
    }
    if (threadIdx.x == 0 && it + kLookahead < ntiles) issue_next();
    const int64_t tok0 = (int64_t)lt * kTile + warp * 32;   // first token of this warp
    mbar_wait(&full[s], (it / kStages) & 1);
    const uint8_t* st = sm + s * L::kStageBytes;
    if (tok0 + 32 <= P.n) tile(st, tok0, std::false_type{});
    else tile(st, tok0, std::true_type{});
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++lt == P.tpu) { lt = 0; ++u; }
  }
  if (cur_u >= 0) flush(cur_u);
}

struct Plan {
  int tpu, ctas, max_seg;
  int64_t T;
  size_t afrag_off, qconst_off, part_off, cnt_off, total;
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

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

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
  p.qconst_off = align256((size_t)kc.units * KC * 32 * 16);
  p.part_off = p.qconst_off + align256((size_t)kc.units * 4 * 16);
  p.cnt_off = p.part_off + align256((size_t)kc.units * p.max_seg * G * kRec * 4);
  p.total = p.cnt_off + align256((size_t)kc.units * 4);
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
  int* counters = (int*)(w + plan.cnt_off);
  constexpr int MT = (KCI + KCO) * 32;
#define QJL_PREP(TQ, TS)                                                                         \
  k_prep<TQ, TS, KCI, KCO><<<kc.units, MT, 0, st>>>((const TQ*)q, G, (const TS*)sk.s_full,       \
                                                    sk.unit_stride, inv_t, afrag, qconst, counters)
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
  P.counters = counters;
  P.out = out;
  P.lse = lse;
  occupancy<KCI, KCO>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Layout<KCI, KCO>::kTotal;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = timing_enabled() ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  timing_begin(st);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_decode_tc<KCI, KCO>, P);
  timing_end(st);
  if (e != cudaSuccess) return cuda_status(e, "decode_tc");
  QJL_LAUNCH_CHECK("decode_tc");
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
