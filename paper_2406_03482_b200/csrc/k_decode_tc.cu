// Tensor-core fused QJL decode (K2 score estimator + K3 online softmax . V) for
// P2 value caches on sm_100a.
//
//  * Data movement: thread 0 streams each 128-token tile of the packed cache
//    (sign bits, fp16 norms, 2-bit codes, fp16 zero/scale) HBM -> smem with
//    cp.async.bulk (TMA bulk copies) into a kStages mbarrier ring, kLookahead
//    tiles ahead; the 4 warps never issue global loads on the hot path.
//  * Scores (estimator.py:149-170 identity 2*sum_set(Sq) - sum(Sq)): the query
//    sketch of every query head is quantized to a 32-bit fixed-point integer and
//    split into four int8 digits -- the B operand of an m16n8k32 IMMA whose
//    columns are (query, digit) pairs -- so one IMMA computes 16 tokens x 4 query
//    heads x 2 digits x 32 sign bits with exact int32 accumulation.  The A operand
//    is the packed sign word itself, masked in place: `w & (0x01010101 << 2q)`
//    turns 4 sign bits into 4 u8 lanes of value 2^(2q)*bit (2 LOP3 per 8 bits, no
//    unpacking); the 2^s weights are folded into the digits.
//  * PV: out[q][d] = sum_t P'[t][q] c[t][d] + sum_t p[t][q] zero[t][g], with
//    P' = p * scale split hi/lo in fp16 (22-bit P') as the B operand of an
//    m16n8k16 HMMA whose A operand is the 2-bit code turned into the NORMAL fp16
//    1 + c 4^s/1024 by one SHF + one LOP3 (P2 layout puts lane-row g's 16 dims in
//    code word g); the offset sum_t P' is removed with an exact FFMA accumulator.
//  * Online softmax in the log2 domain per query head; one partial (m, l, acc)
//    per (CTA, unit segment); CTAs own equal contiguous ranges of the flattened
//    (unit, tile) space (stream-K) so every SM gets the same number of tiles.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace qjl {
namespace tc {

constexpr int kNW = 4;             // warps per CTA (all compute; warp 0 lane 0 issues copies)
constexpr int kTile = 32 * kNW;    // tokens per pipeline stage
constexpr int kStages = 5;
constexpr int kLookahead = 3;      // tiles in flight ahead of the one being consumed
constexpr int kThreads = 32 * kNW;
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
// A = masked sign words (u8 lanes 2^s * bit), B = query-sketch digits (s8)
__device__ __forceinline__ void imma_u8s8(int* d, const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
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
  static constexpr int oRed = oPbuf;                               // flush scratch aliases P'
  static constexpr int kRec = 2 + 4 + 128;                          // m, l, Z[4], acc[128]
  static constexpr int kRedBytes = kNW * 4 * kRec * 4;
  static constexpr int kScratch = kRedBytes > kNW * 2048 ? kRedBytes : kNW * 2048;
  static constexpr int oBar = oPbuf + kScratch;
  static constexpr int kTotal = oBar + 2 * kStages * 8;
};

// ----------------------------------------------------------------- prep kernel
// Per unit: Sq = S_full . q (fp64, rounded to fp32 like the generic path),
// per-side sigma = max|Sq| / 2^30, weighted integer sketch
// x_j = rint(Sq_j / (sigma * 2^(j mod 8))), 4 signed-byte digits laid out as the
// IMMA B operand: column n of n-tile nt = (query n/2, digit 2*nt + n%2).
template <typename TQ, typename TS, int KCI, int KCO>
__global__ void __launch_bounds__(512) k_prep(const TQ* __restrict__ q, int G, const TS* __restrict__ s_full,
                                              int64_t s_unit_stride, float inv_t, uint4* __restrict__ bfrag,
                                              float4* __restrict__ qconst) {
  constexpr int MI = KCI * 32, MO = KCO * 32, MT = MI + MO, KC = KCI + KCO;
  constexpr int d = 128;
  // 16-bit sketch operands: products are exact in fp32; wider operands accumulate in fp64
  using acc_t = typename std::conditional<(sizeof(TS) <= 2), float, double>::type;
  __shared__ acc_t qs[4][d];
  __shared__ float sq[4][MT];
  __shared__ int32_t si[4][MT];
  __shared__ unsigned int mxbits[4][2];
  __shared__ double red[4][2][2];   // [q][side][sigma, sum]
  const int u = blockIdx.x;
  const TS* S = s_full + (int64_t)u * s_unit_stride;
  // let the decode kernel launch now (programmatic dependent launch): its prologue and
  // first bulk copies overlap this kernel; it waits (griddepcontrol.wait) before reading
  // anything written here
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int i = threadIdx.x; i < 4 * d; i += blockDim.x) {
    const int g = i / d;
    qs[g][i % d] = g < G ? (acc_t)to_f64(q[((int64_t)u * G + g) * d + i % d]) : (acc_t)0;
  }
  if (threadIdx.x < 8) {
    mxbits[threadIdx.x >> 1][threadIdx.x & 1] = 0u;
  }
  __syncthreads();
  // one warp per sketch row (coalesced 256-byte row reads), lane l owns columns
  // 4l..4l+3 of every query head; shuffle-reduce the four partial dots
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  acc_t qreg[4][4];
#pragma unroll
  for (int g = 0; g < 4; ++g)
#pragma unroll
    for (int e = 0; e < 4; ++e) qreg[g][e] = qs[g][4 * lane + e];
  float wmax[4][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
  for (int r = wid; r < MT; r += nwarp) {
    const TS* row = S + (int64_t)r * d + 4 * lane;
    acc_t a[4] = {0, 0, 0, 0};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const acc_t sv = (acc_t)to_f64(row[e]);
#pragma unroll
      for (int g = 0; g < 4; ++g) a[g] = fma(sv, qreg[g][e], a[g]);
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a[g] += __shfl_xor_sync(0xffffffffu, a[g], o);
    }
    const int side = r >= MI;
    if (lane < 4) sq[lane][r] = (float)a[lane];
#pragma unroll
    for (int g = 0; g < 4; ++g) wmax[g][side] = fmaxf(wmax[g][side], fabsf((float)a[g]));
  }
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) atomicMax(&mxbits[g][sd], __float_as_uint(wmax[g][sd]));
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
    const int c = i / 32, lane = i % 32;
    const int n = lane >> 2, ql = lane & 3;
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
    bfrag[((int64_t)u * KC + c) * 32 + lane] = make_uint4(regs[0], regs[1], regs[2], regs[3]);
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
// 4 warps per CTA, each owning 32 tokens of every 128-token stage; thread 0 also
// issues the bulk copies kLookahead tiles ahead (no dedicated producer warp, so
// three CTAs -- 12 warps -- fit per SM).
//
// Token order inside a warp's 32-token tile: score m-tile h covers tokens 16h..16h+15
// with IMMA rows g / g+8 = tokens 16h+g / 16h+g+8, and the PV k-step h uses the
// permuted k order k = 2j + e  <->  token 16h + j + 8e, so the fp16 pair (k, k+1)
// of a B fragment is exactly the token pair a score lane owns (no exchange).
template <int KCI, int KCO>
__global__ void __launch_bounds__(kThreads, (KCI + KCO > 12) ? 2 : 3) k_decode_tc(const Params P) {
  using L = Layout<KCI, KCO>;
  constexpr int KC = KCI + KCO;
  constexpr int R = L::kRec;
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

  const int g = lane >> 2, q = lane & 3;      // q = this lane's query head
  const uint32_t M0 = 0x01010101u << (2 * q), M1 = 0x02020202u << (2 * q);
  uint32_t* pbuf = reinterpret_cast<uint32_t*>(sm + L::oPbuf + warp * 2048);
  float* red = reinterpret_cast<float*>(sm + L::oRed);

  uint4 Bq[KC];                               // query-sketch digits (IMMA B operand)
  float4 qc = make_float4(0.f, 0.f, 0.f, 0.f);
  float m_run = -INFINITY, l_run = 0.f;
  float Z[4] = {0.f, 0.f, 0.f, 0.f};          // sum_t p * zero_g   (query q)
  float Y[4] = {0.f, 0.f, 0.f, 0.f};          // sum_t p * scale_g  (HMMA offset removal)
  float acc[8][4];                            // PV: rows = dims, cols (2q, 2q+1) = query q hi/lo
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;

  auto load_unit = [&](int u) {
#pragma unroll
    for (int c = 0; c < KC; ++c) Bq[c] = P.afrag[((int64_t)u * KC + c) * 32 + lane];
    qc = P.qconst[(int64_t)u * 4 + q];
    m_run = -INFINITY;
    l_run = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) Z[i] = Y[i] = 0.f;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
  };

  auto flush = [&](int u) {
    // the P' buffers are reused as scratch: every warp must be done with its tile
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
    // l, Z, Y: reduce over the 8 lanes of query q (lanes q + 4g)
    float l = l_run;
    float z[4] = {Z[0], Z[1], Z[2], Z[3]};
    float y[4] = {Y[0], Y[1], Y[2], Y[3]};
#pragma unroll
    for (int o = 4; o <= 16; o <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        z[i] += __shfl_xor_sync(0xffffffffu, z[i], o);
        y[i] += __shfl_xor_sync(0xffffffffu, y[i], o);
      }
    }
    float* rw = red + warp * 4 * R;
    if (g == 0) {
      rw[q * R + 0] = m_run;
      rw[q * R + 1] = l;
#pragma unroll
      for (int i = 0; i < 4; ++i) rw[q * R + 2 + i] = z[i];
    }
    // HMMA rows hold sum_t P' (1 + c 4^s / 1024), s = 3 (row g) or 4 (row g+8)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const float yg = y[mt >> 1];
      rw[q * R + 6 + 16 * mt + g] = (acc[mt][0] + acc[mt][1] - yg) * 16.f;
      rw[q * R + 6 + 16 * mt + g + 8] = (acc[mt][2] + acc[mt][3] - yg) * 4.f;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
    const int c0 = cta_of_tile((int64_t)u * P.tpu, T, C);
    const int slot = blockIdx.x - c0;
    for (int i = threadIdx.x; i < P.G * 130; i += kThreads) {
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
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
  };

  // one 32-token warp tile; MASK: some tokens are >= n (tail tile of a unit)
  auto tile = [&](const uint8_t* st, const int64_t tok0, auto mask_tag) {
    constexpr bool MASK = decltype(mask_tag)::value;
    const uint32_t* bin = reinterpret_cast<const uint32_t*>(st + L::oBitsIn) + warp * 32 * KCI;
    const uint32_t* bout = reinterpret_cast<const uint32_t*>(st + L::oBitsOut) + warp * 32 * KCO;
    const __half* nin = reinterpret_cast<const __half*>(st + L::oNormIn) + warp * 32;
    const __half* nout = reinterpret_cast<const __half*>(st + L::oNormOut) + warp * 32;
    const uint32_t* codes = reinterpret_cast<const uint32_t*>(st + L::oCodes) + warp * 32 * 8;
    const uint2* zer = reinterpret_cast<const uint2*>(st + L::oZero) + warp * 32;
    const uint2* scl = reinterpret_cast<const uint2*>(st + L::oScale) + warp * 32;

    // -------- scores: 2 IMMA m-tiles of 16 tokens (rows g, g+8) x 2 n-tiles -------
    // D[token][2q + i] of n-tile nt = digit 2nt+i of query q: every lane ends up
    // with all four digits of its own query for tokens g and g+8 -- no shuffles.
    float lg[4];                       // token 16h + g + 8e  ->  lg[2h + e]
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ta = 16 * h + g, tb = ta + 8;
      int din[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
      int dout[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
      for (int c = 0; c < KCI; c += 4) {
        const uint4 va = *reinterpret_cast<const uint4*>(bin + ta * KCI + c);
        const uint4 vb = *reinterpret_cast<const uint4*>(bin + tb * KCI + c);
        const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint4 a = make_uint4(wa[e] & M0, wb[e] & M0, wa[e] & M1, wb[e] & M1);
          imma_u8s8(din[0], a, Bq[c + e].x, Bq[c + e].y);
          imma_u8s8(din[1], a, Bq[c + e].z, Bq[c + e].w);
        }
      }
#pragma unroll
      for (int c = 0; c < KCO; c += 2) {
        const uint2 va = *reinterpret_cast<const uint2*>(bout + ta * KCO + c);
        const uint2 vb = *reinterpret_cast<const uint2*>(bout + tb * KCO + c);
        const uint32_t wa[2] = {va.x, va.y}, wb[2] = {vb.x, vb.y};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint4 a = make_uint4(wa[e] & M0, wb[e] & M0, wa[e] & M1, wb[e] & M1);
          imma_u8s8(dout[0], a, Bq[KCI + c + e].x, Bq[KCI + c + e].y);
          imma_u8s8(dout[1], a, Bq[KCI + c + e].z, Bq[KCI + c + e].w);
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {      // e = 0: token ta (c0, c1); e = 1: token tb (c2, c3)
        const int tk = e ? tb : ta;
        // |digit partial| <= 2^21, so d0 + 256 d1 and d2 + 256 d3 are exact in int32
        const float din_f = fmaf((float)(din[1][2 * e] + 256 * din[1][2 * e + 1]), 65536.f,
                                 (float)(din[0][2 * e] + 256 * din[0][2 * e + 1]));
        float l2 = __half2float(nin[tk]) * fmaf(qc.x, din_f, -qc.y);
        if (KCO) {
          const float dout_f = fmaf((float)(dout[1][2 * e] + 256 * dout[1][2 * e + 1]), 65536.f,
                                    (float)(dout[0][2 * e] + 256 * dout[0][2 * e + 1]));
          l2 = fmaf(__half2float(nout[tk]), fmaf(qc.z, dout_f, -qc.w), l2);
        }
        lg[2 * h + e] = (!MASK || tok0 + tk < P.n) ? l2 : -INFINITY;
      }
    }

    // -------------------- online softmax (log2 domain, query q) --------------------
    float tmax = fmaxf(fmaxf(lg[0], lg[1]), fmaxf(lg[2], lg[3]));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
    const float m_new = fmaxf(m_run, tmax);
    const bool none = MASK && (m_new == -INFINITY);
    const float alpha = none ? 1.f : ex2(m_run - m_new);
    m_run = m_new;
    float p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = none ? 0.f : ex2(lg[i] - m_new);
    l_run = fmaf(l_run, alpha, (p[0] + p[1]) + (p[2] + p[3]));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      Z[i] *= alpha;
      Y[i] *= alpha;
    }

    // -------- P' = p * scale_g, split hi/lo fp16, written as HMMA B fragments --------
    // B layout per warp: [k-step h][column 2q + lo][quad q'][b][group] half2 over the
    // k pair (2q' + 8b, +1) = tokens (16h + q' + 4b, +8): this lane's own pair
    // (tokens 16h + g, 16h + g + 8) is q' = g & 3, b = g >> 2.
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float hv[2][4], lv[2][4];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tk = 16 * h + g + 8 * e;
        const float pj = p[2 * h + e];
        uint2 zr = zer[tk], sr = scl[tk];
        if (MASK && tok0 + tk >= P.n) zr = sr = make_uint2(0u, 0u);   // garbage rows past n
        const float2 z01 = __half22float2(*reinterpret_cast<const __half2*>(&zr.x));
        const float2 z23 = __half22float2(*reinterpret_cast<const __half2*>(&zr.y));
        const float2 s01 = __half22float2(*reinterpret_cast<const __half2*>(&sr.x));
        const float2 s23 = __half22float2(*reinterpret_cast<const __half2*>(&sr.y));
        const float zz[4] = {z01.x, z01.y, z23.x, z23.y};
        const float ss[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float Pp = pj * ss[i];
          Z[i] = fmaf(pj, zz[i], Z[i]);
          Y[i] += Pp;
          hv[e][i] = __uint_as_float(__float_as_uint(Pp) & 0xFFFFE000u);   // 11 significant bits
          lv[e][i] = Pp - hv[e][i];
        }
      }
      uint32_t* dst = pbuf + (((h * 8 + 2 * q) * 4 + (g & 3)) * 2 + (g >> 2)) * 4;
      *reinterpret_cast<uint4*>(dst) = make_uint4(pack_h2(hv[0][0], hv[1][0]), pack_h2(hv[0][1], hv[1][1]),
                                                  pack_h2(hv[0][2], hv[1][2]), pack_h2(hv[0][3], hv[1][3]));
      *reinterpret_cast<uint4*>(dst + 32) = make_uint4(pack_h2(lv[0][0], lv[1][0]), pack_h2(lv[0][1], lv[1][1]),
                                                       pack_h2(lv[0][2], lv[1][2]), pack_h2(lv[0][3], lv[1][3]));
    }
    __syncwarp();

    // -------------------- PV: 8 m-tiles x 2 k-steps of 16 tokens ---------------
    // a0/a1: k pair (2q, 2q+1) = tokens (16h + q, 16h + q + 8); a2/a3: (16h + q + 4, + 12)
    uint32_t xa[2], xb[2], ya[2], yb[2];
    uint32_t bg[4][2][2];   // [group][ks][b]
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int tb = 16 * ks + q;
      const uint32_t w0 = codes[(tb + 0) * 8 + g], w1 = codes[(tb + 8) * 8 + g];
      const uint32_t w4 = codes[(tb + 4) * 8 + g], w5 = codes[(tb + 12) * 8 + g];
      xa[ks] = prmt(w0, w1, 0x5410); xb[ks] = prmt(w0, w1, 0x7632);
      ya[ks] = prmt(w4, w5, 0x5410); yb[ks] = prmt(w4, w5, 0x7632);
      const uint4 B0 = *reinterpret_cast<const uint4*>(pbuf + ((ks * 8 + g) * 4 + q) * 8);
      const uint4 B1 = *reinterpret_cast<const uint4*>(pbuf + ((ks * 8 + g) * 4 + q) * 8 + 4);
      bg[0][ks][0] = B0.x; bg[1][ks][0] = B0.y; bg[2][ks][0] = B0.z; bg[3][ks][0] = B0.w;
      bg[0][ks][1] = B1.x; bg[1][ks][1] = B1.y; bg[2][ks][1] = B1.z; bg[3][ks][1] = B1.w;
    }
    // m-tile MT: rows g / g+8 use code slots 2*(MT&3) / +1 of half-words X and Y;
    // one shift brings both to mantissa slots 3 / 4.
    // The tile's product is formed from zero and folded into the running sum with an
    // IEEE FFMA that also applies the online-softmax rescale (alpha is lane-local:
    // the accumulator columns of this lane belong to query q).  Accumulating straight
    // into the running sum drifts: the tensor core's fp32 adder truncates small
    // addends against a large accumulator (1.8e-4 at 32k tokens, growing with n).
#define QJL_MT(MT, X, Yw)                                                                        \
  {                                                                                              \
    float td[4] = {0.f, 0.f, 0.f, 0.f};                                                          \
    _Pragma("unroll") for (int ks = 0; ks < 2; ++ks) {                                           \
      const uint32_t xs = code_shift<(MT) & 3>(X[ks]), ys = code_shift<(MT) & 3>(Yw[ks]);        \
      hmma(td, code_h2<3>(xs), code_h2<4>(xs), code_h2<3>(ys), code_h2<4>(ys),                   \
           bg[(MT) >> 1][ks][0], bg[(MT) >> 1][ks][1]);                                          \
    }                                                                                            \
    _Pragma("unroll") for (int i = 0; i < 4; ++i) acc[MT][i] = fmaf(acc[MT][i], alpha, td[i]);  \
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
  };

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // merge kernel may launch
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


// Merge per (unit, query): combine the unit's CTA-segment partials.
__global__ void k_merge_tc(const float* __restrict__ part, int max_seg, int G, int tpu, int64_t T, int C,
                           float* __restrict__ out, float* __restrict__ lse) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: partials of the decode grid
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
  k_prep<TQ, TS, KCI, KCO><<<kc.units, 512, 0, st>>>((const TQ*)q, G, (const TS*)sk.s_full,      \
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
  cudaLaunchConfig_t mcfg = {};
  mcfg.gridDim = dim3(kc.units * G);
  mcfg.blockDim = dim3(128);
  mcfg.stream = st;
  mcfg.attrs = attr;
  mcfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&mcfg, k_merge_tc, (const float*)part, plan.max_seg, G, plan.tpu, plan.T, plan.ctas,
                         out, lse);
  if (e != cudaSuccess) return cuda_status(e, "decode_tc_merge");
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
