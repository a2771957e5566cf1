// tcgen05 (5th-gen tensor core) fused QJL decode -- K2 score estimator + K3 online
// softmax . V -- for P2T value caches on sm_100a.
//
// One decode step = 2 launches chained with programmatic dependent launch:
//   k_uprep   one CTA per unit: Sq = S_full . q for the unit's G <= 4 query heads,
//             quantized to a 32-bit fixed-point integer, split into four int8 digits and
//             written as the score MMA's B operand (K-major, SWIZZLE_128B image);
//             zeroes the unit's merge counter.
//   k_udecode stream-K over the flattened (unit, 128-token tile) space, 4 warps per CTA,
//             4 CTAs per SM (128 TMEM columns each).  The CTA that finishes a unit last
//             (atomic counter) merges the unit's partials.
//
// Per 128-token tile (all 128 threads; thread t owns token t for scoring and dim t for
// the value aggregation):
//  1. thread = token: the packed sign words (estimator.py:110-124 layout) are expanded in
//     place into the u8 A operand of the score MMA -- `w & 0x01010101 << s` puts sign bits
//     8i + s of word w into four byte lanes of value 2^s * bit -- and stored to TMEM
//     (tcgen05.st); the 2^s weights are folded into the B digits.
//  2. one thread issues tcgen05.mma kind::i8 (A from TMEM, B = query-sketch digits from
//     smem), M = 128 tokens, N = 16 (4 heads x 4 digits) per side: exact int32
//     2 * sum_set(Sq) (estimator.py:149-170) for every token and head.
//  3. thread = token: tcgen05.ld of its 32 accumulators -> logits of the 4 heads
//     (kvcache.py:311-329), CTA tile maximum (redux.sync + smem), online softmax in the
//     log2 domain (kvcache.py:38-44 / attention.py:56-71).
//  4. thread = token: P' = p * scale of its 4 heads x 4 value groups in 24-bit fixed
//     point relative to the tile bound, split into three int8 digits by one FFMA (float
//     magic-number rounding) + PRMTs -> the PV MMA's B operand (MN-major smem, one 16-byte
//     store per digit); zero-point term sum p * zero on the CUDA cores.
//     thread = dim: its P2T code words masked in place (`w & 3 << 2(d % 4)`: 4 tokens of
//     one dim, value c * 4^(d % 4)) -> A operand of the PV MMA in TMEM.
//  5. one thread issues tcgen05.mma kind::i8: D[dim][(digit, group, head)] over the 128
//     tokens (N = 48).
//  6. thread = dim: tcgen05.ld of its group's 12 accumulators -> fp32 running output.
#include <cstdio>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace qjl {
namespace ud {

#ifndef QJL_UD_ABLATE
#define QJL_UD_ABLATE 0     // perf experiments only: 1 no score MMA, 2 no PV MMA, 4 no sign expansion, 8 no P'/codes
#endif
#ifndef QJL_UD_SPLIT
#define QJL_UD_SPLIT 0      // 1: split-phase mbarriers between the warps, 0: CTA barriers
#endif
constexpr int kThreads = 128;      // 4 warps; thread t: token t (scores) and dim t (PV)
constexpr int kTile = 128;         // tokens per tile
#ifndef QJL_UD_STAGES
#define QJL_UD_STAGES 3
#endif
#ifndef QJL_UD_LA
#define QJL_UD_LA 2
#endif
constexpr int kStages = QJL_UD_STAGES;
constexpr int kLookahead = QJL_UD_LA;
constexpr int kRec = 130;          // per (partial, query): m (log2 domain), l, out[128]
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kPMax = 8.0e6f;                  // P' fixed-point full scale (< 2^23 - 32896)
constexpr float kMagic = 8421504.f;              // 2^23 + 32896

// Decode-step append: the new token of every unit, quantized inside the
// query-sketch kernel (which streams S_full anyway) and written at row `row` before the
// decode kernel -- PDL-ordered after it -- reads rows [0, row + 1).
struct Append {
  const void* k;               // [units][128] in the query dtype; nullptr: no append
  const void* v;               // [units][128]
  qjl_key_cache_t kc;
  qjl_value_cache_t vc;
  const int32_t* channels;     // [units][h]
  int h;
  int64_t row;
};

struct Params {
  qjl_key_cache_t kc;
  qjl_value_cache_t vc;
  int64_t n;
  int G;
  int units;
  int tpu;               // tiles per unit
  int64_t total_tiles;
  int ctas;
  int max_seg;
  int grouped;           // 1: every unit owns a group of CTAs that stride over its tiles
  const uint8_t* bsc;    // [units][NH][2048] score B operand images (SW128, K-major)
  const float4* qconst;  // [units][4 queries] {k_in, b_in, k_out, b_out}
  float* part;           // [units][max_seg][G][kRec]
  int* counters;         // [units]
  float* out;            // [units][G][128]
  float* lse;            // [units][G] or null
};

#ifndef QJL_UD_TRACE
#define QJL_UD_TRACE 0      // diagnostics only: per-CTA %globaltimer stamps (tools/trace_decode.py)
#endif
#if QJL_UD_TRACE
__device__ unsigned long long g_ud_trace[2048][4];   // [cta] {after wait, loop done, end, smid}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

__host__ __device__ __forceinline__ int64_t tile_begin(int c, int64_t T, int C) { return (int64_t)c * T / C; }
__host__ __device__ __forceinline__ int cta_of_tile(int64_t t, int64_t T, int C) {
  return (int)(((t + 1) * (int64_t)C + T - 1) / T) - 1;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the same on precomputed 32-bit shared-window addresses (no generic->shared conversion
// in the main loop)
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
#ifndef QJL_UD_EVICT_FIRST
#define QJL_UD_EVICT_FIRST 1   // the streamed cache tiles are read once per step: evict them first
#endif
// same, with an L2 cache-policy hint (the cache stream must not evict the small per-step
// data -- sketches, B images, partials -- that the prep and the merge re-read)
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bar_sync1() { asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}
// same, with a compile-time accumulate flag (no predicate computation per MMA)
template <int ACC>
__device__ __forceinline__ void tc_mma_i8c(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "n"(ACC));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(pred));
  return pred != 0;
}
// instruction descriptor: D s32, A u8 (K-major, from TMEM), B s8, M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int n, int b_mn_major) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
// K-major SWIZZLE_128B descriptor (rows of 128 B, 8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// SWIZZLE_NONE descriptor (MN-major: LBO = K-block stride, SBO = 16-byte MN-chunk stride)
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float warp_max_f32(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rc, {%6, %7};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 h2f2(uint32_t h) { return __half22float2(*reinterpret_cast<const __half2*>(&h)); }
__device__ __forceinline__ uint32_t hmax2u(uint32_t a, uint32_t b) {
  __half2 r = __hmax2(*reinterpret_cast<const __half2*>(&a), *reinterpret_cast<const __half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

// --------------------------------------------------------------- smem layout
template <int KCI, int KCO>
struct Layout {
  static constexpr int KC = KCI + KCO;
  static constexpr int NHI = KCI / 4, NHO = (KCO + 3) / 4, NH = NHI + NHO;   // 128-byte K halves of B
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
  static constexpr int oBsc = 0;                        // 1024-aligned
  static constexpr int oBpv = oBsc + NH * 2048;         // [4 heads][128 tokens][16 B] (MN-major chunks)
  static constexpr int oRed = oBsc;                     // flush scratch aliases Bsc/Bpv
  static constexpr int oStage = oBpv + 4 * 2048;
  static constexpr int oMax = oStage + kStages * kStageBytes;   // [4 warps][8] tile maxima
  static constexpr int oQc = oMax + 4 * 8 * 4;                  // [4 queries] float4 estimator constants
  static constexpr int oBar = oQc + 4 * 16;
  static constexpr int kBars = 2 * kStages + 6;
  static constexpr int oTmem = oBar + kBars * 8;
  static constexpr int oFlag = oTmem + 4;
  static constexpr int kTotal = oFlag + 12 + 1024;      // + alignment slack
  // TMEM columns: A_sc [0, 8 KC); after the score MMA: A_pv [0, 32), D_pv [32, 96);
  // D_sc (in: 16, out: 16) after both
  static constexpr int cDsc = (8 * KC > 96) ? 8 * KC : 96;
  static constexpr int kCols = cDsc + (KCO ? 32 : 16);
  static constexpr int kAlloc = kCols <= 128 ? 128 : 256;
};

// ----------------------------------------------------------------- prep kernel
template <typename A, typename T>
__device__ __forceinline__ A to_acc(T x) {
  if constexpr (std::is_same<A, float>::value) return to_f32(x);
  else return to_f64(x);
}

// One CTA per unit, one thread per sketch row: Sq = S_full . q (fp32 products of the
// 16-bit operands, exact; fp64 for wider sketches), per-side sigma = max|Sq| / 2^30,
// weighted integer sketch x_j = rint(Sq_j / (sigma * 2^(j mod 8))), four signed-byte
// digits.  B image: row n = 4 q + digit, K byte k of a side <-> chunk c = k / 32 and,
// within it, (s, i) = ((k % 32) / 4, k % 4) <-> sign bit j = 32 c + 8 i + s (the A side
// masks word c with 0x01010101 << s).
#ifndef QJL_PREP_ABLATE
#define QJL_PREP_ABLATE 0   // perf experiment only: 1 skip the S.q loop, 2 skip the B image build
#endif
template <typename TQ, typename TS, int KCI, int KCO, bool APPEND>
__global__ void __launch_bounds__(640) k_uprep(const TQ* __restrict__ q, int G, const TS* __restrict__ s_full,
                                               int64_t s_unit_stride, float inv_t, uint8_t* __restrict__ bsc,
                                               float4* __restrict__ qconst, int* __restrict__ counters,
                                               const Append A) {
  using L = Layout<KCI, KCO>;
  constexpr int MI = KCI * 32, MO = KCO * 32, MT = MI + MO;
  constexpr int d = 128;
  using acc_t = typename std::conditional<(sizeof(TS) <= 2), float, double>::type;
  constexpr bool F32 = std::is_same<acc_t, float>::value;
  __shared__ acc_t qs[F32 ? 1 : 4][d];                // fp64 path: [head][dim]
  __shared__ float4 qs4[F32 ? d : 1];                 // fp32 path: the 4 heads of a dim
  __shared__ float sq[4][MT];
  __shared__ __align__(16) uint8_t img[L::NH * 2048]; // the score B image, built in place
  __shared__ unsigned int mxbits[4][2];
  __shared__ double red[4][2][2];   // [q][side][sigma, sum]
  const int u = blockIdx.x;
  const TS* S = s_full + (int64_t)u * s_unit_stride;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  // 16-bit sketches: the thread's whole S row (256 B) is requested before anything else,
  // so one memory round trip covers it
  uint4 srow[F32 ? 16 : 1];
  if constexpr (F32) {
    const uint4* rp = reinterpret_cast<const uint4*>(S + (int64_t)threadIdx.x * d);
#pragma unroll
    for (int i = 0; i < 16; ++i) srow[i] = (QJL_PREP_ABLATE & 1) ? make_uint4(0, 0, 0, 0) : __ldg(rp + i);
  }
  if constexpr (F32) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      float v[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) v[g] = g < G ? to_f32(q[((int64_t)u * G + g) * d + i]) : 0.f;
      qs4[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
  } else {
    for (int i = threadIdx.x; i < 4 * d; i += blockDim.x) {
      const int g = i / d;
      qs[g][i % d] = g < G ? to_acc<acc_t>(q[((int64_t)u * G + g) * d + i % d]) : (acc_t)0;
    }
  }
  for (int i = threadIdx.x; i < L::NH * 128; i += blockDim.x) reinterpret_cast<uint4*>(img)[i] = make_uint4(0, 0, 0, 0);
  // decode-step append (APPEND): the new key / value of this unit
  __shared__ double kd[APPEND ? d : 1], vd[APPEND ? d : 1];
  __shared__ unsigned char outl_ch[APPEND ? d : 1];
  __shared__ uint32_t aw[APPEND ? MT / 32 : 1];   // sign words of the new key
  __shared__ double an[4][2];                 // [warp][inlier, outlier] sums of squares
  if (APPEND) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      kd[i] = to_f64(reinterpret_cast<const TQ*>(A.k)[(int64_t)u * d + i]);
      vd[i] = to_f64(reinterpret_cast<const TQ*>(A.v)[(int64_t)u * d + i]);
      outl_ch[i] = 0;
    }
  }
  // ---- decode-step append (APPEND), done before the dependent decode may launch: the
  // new row is written and fenced here, so the decode's first copies (issued before its
  // grid-dependency wait) already see it.  Row n is padding for the previous step's
  // decode (masked), so writing it while that decode drains is harmless.  Arithmetic:
  // K1's fp64 path and the value quantizer's (kvcache.py:293-306, :140-161).
  double vzero = 0.0, vscale = 0.0;
  uint32_t vbyte = 0;                         // this lane's P2T byte (dims 4a..4a+3)
  if constexpr (APPEND) {
    __syncthreads();                          // kd / vd / outl_ch
    if (threadIdx.x < A.h) outl_ch[A.channels[(int64_t)u * A.h + threadIdx.x]] = 1;
    {
      // S_r . k_new: exact products of the 16-bit operands, fp64 sum; bit = (p >= 0):
      // -0.0 -> 1, NaN -> 0 (estimator.py:119-121)
      const int r = threadIdx.x;
      double pr = 0.0;
      if constexpr (F32) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const TS* sv = reinterpret_cast<const TS*>(&srow[i]);
#pragma unroll
          for (int k = 0; k < 8; ++k) pr = fma((double)to_f32(sv[k]), kd[8 * i + k], pr);
        }
      } else {
        const TS* row = S + (int64_t)r * d;
        for (int e = 0; e < d; ++e) pr = fma(to_f64(row[e]), kd[e], pr);
      }
      const uint32_t bw = __ballot_sync(0xffffffffu, pr >= 0.0);
      if (lane == 0) aw[wid] = bw;
    }
    __syncthreads();                          // outl_ch, aw
    if (wid < 4) {
      // norms of the inlier / outlier parts (fp64, one fp16 rounding each), and the
      // value group wid = dims 32 wid .. 32 wid + 31
      const int dim = threadIdx.x;
      const double x2 = kd[dim] * kd[dim];
      const double sin = warp_sum_f64(outl_ch[dim] ? 0.0 : x2);
      const double sout = warp_sum_f64(outl_ch[dim] ? x2 : 0.0);
      if (lane == 0) {
        an[wid][0] = sin;
        an[wid][1] = sout;
      }
      const double x = vd[dim];
      double mn = x, mx = x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      const int levels = (1 << A.vc.bits) - 1;
      const double spread = mx - mn;
      vzero = mn;
      vscale = spread == 0.0 ? 0.0 : spread / (double)levels;
      int code = 0;
      if (spread != 0.0) code = (int)fmin(fmax(rint((x - mn) / vscale), 0.0), (double)levels);
      uint32_t b = (uint32_t)code << (2 * (lane & 3));
      b |= __shfl_xor_sync(0xffffffffu, b, 1);
      b |= __shfl_xor_sync(0xffffffffu, b, 2);
      vbyte = b;
    }
    __syncthreads();                          // an
    const int64_t crow = (int64_t)u * A.kc.capacity + A.row;
    if (threadIdx.x < MT / 32) {
      const int w = threadIdx.x;
      if (w < MI / 32) reinterpret_cast<uint32_t*>(A.kc.bits_in + crow * (MI / 8))[w] = aw[w];
      else reinterpret_cast<uint32_t*>(A.kc.bits_out + crow * (MO / 8))[w - MI / 32] = aw[w];
    }
    if (threadIdx.x == 0) {
      const double sin = (an[0][0] + an[1][0]) + (an[2][0] + an[3][0]);
      const double sout = (an[0][1] + an[1][1]) + (an[2][1] + an[3][1]);
      A.kc.norm_in[crow] = f16_canon(f64_to_f16_bits(sqrt(sin)));
      if (MO) A.kc.norm_out[crow] = f16_canon(f64_to_f16_bits(sqrt(sout)));
    }
    if (wid < 4) {
      const int64_t vrow = (int64_t)u * A.vc.capacity + A.row;
      if ((lane & 3) == 0) {
        int64_t byte;
        int sh;
        p2t_pos(vrow, threadIdx.x, &byte, &sh);
        reinterpret_cast<uint8_t*>(A.vc.codes)[byte] = (uint8_t)vbyte;
      }
      if (lane == 0) {
        reinterpret_cast<uint16_t*>(A.vc.zero)[vrow * 4 + wid] = f64_to_f16_bits(vzero);
        reinterpret_cast<uint16_t*>(A.vc.scale)[vrow * 4 + wid] = f64_to_f16_bits(vscale);
      }
    }
    __threadfence();
  }
  if (threadIdx.x < 8) mxbits[threadIdx.x >> 1][threadIdx.x & 1] = 0u;
  // let the decode kernel launch now: its prologue and first bulk copies overlap us
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __syncthreads();
  {
    const int r = threadIdx.x;               // blockDim.x == MT
    const TS* row = S + (int64_t)r * d;
    constexpr int EPV = 16 / (int)sizeof(TS);
    acc_t a[4] = {0, 0, 0, 0};
    float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);   // fp32 path, FFMA2 pairs
#pragma unroll
    for (int e0 = 0; e0 < d; e0 += EPV) {
      if (QJL_PREP_ABLATE & 1) break;
      const uint4 raw = F32 ? srow[(e0 / EPV) & (F32 ? 15 : 0)] : __ldg(reinterpret_cast<const uint4*>(row + e0));
      const TS* sv = reinterpret_cast<const TS*>(&raw);
#pragma unroll
      for (int k = 0; k < EPV; ++k) {
        const acc_t s = to_acc<acc_t>(sv[k]);
        if constexpr (F32) {                   // same per-head fma.rn chain, two heads per FFMA2
          const float4 qv = qs4[e0 + k];
          const float2 s2 = make_float2(s, s);
          a01 = fma2(s2, make_float2(qv.x, qv.y), a01);
          a23 = fma2(s2, make_float2(qv.z, qv.w), a23);
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g) a[g] = fma(s, qs[g][e0 + k], a[g]);
        }
      }
    }
    if constexpr (F32) {
      a[0] = a01.x; a[1] = a01.y; a[2] = a23.x; a[3] = a23.y;
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
  for (int seg = wid; seg < 8; seg += nwarp) {
    const int g = seg >> 1, side = seg & 1;
    const int lo = side ? MI : 0, hi = side ? MT : MI;
    const double inv = 1.0 / red[g][side][0];
    long long acc = 0;
    for (int j = lo + lane; j < hi; j += 32) {
      const int sh = (j - lo) & 7;
      int32_t x = (int32_t)rint((double)sq[g][j] * inv / (double)(1 << sh));
      acc += (long long)x * (1ll << sh);
      // four balanced int8 digits of x -> B image rows n = 4 g + t at K byte
      // k = 32 c + 4 s + i of the side (sign bit jj = 32 c + 8 i + s), SWIZZLE_128B
      const int jj = j - lo;
      const int kside = 32 * (jj >> 5) + 4 * (jj & 7) + ((jj >> 3) & 3);
      const int h = (side ? L::NHI : 0) + (kside >> 7), kk = kside & 127;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int8_t lo8 = (int8_t)(x & 0xFF);
        x = (x - (int32_t)lo8) >> 8;
        const int n = 4 * g + t;
        img[h * 2048 + (n >> 3) * 1024 + (n & 7) * 128 + ((((kk >> 4) ^ (n & 7)) << 4) | (kk & 15))] = (uint8_t)lo8;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[g][side][1] = (double)acc * red[g][side][0];
  }
  __syncthreads();
  // Everything above overlaps the previous decode's tail (this grid is launched with
  // programmatic dependent launch); the workspace writes below must wait for it.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) counters[u] = 0;
  // the B image (built in shared memory above) -> workspace, 16-byte stores
  {
    uint4* out = reinterpret_cast<uint4*>(bsc + (size_t)u * L::NH * 2048);
    for (int i = threadIdx.x; i < ((QJL_PREP_ABLATE & 2) ? 0 : L::NH * 128); i += blockDim.x)
      out[i] = reinterpret_cast<const uint4*>(img)[i];
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
// NQ: query heads the epilogue processes (1, 2 or 4 >= G): MHA (G = 1) skips the work of
// three padding heads
template <int KCI, int KCO, int NQ>
__global__ void __launch_bounds__(kThreads, (KCI + KCO > 12) ? 2 : 4) k_udecode(const Params P) {
  using L = Layout<KCI, KCO>;
  constexpr int KC = KCI + KCO;
  extern __shared__ uint8_t sm_raw[];
  // align to 1024 B (SWIZZLE_128B atoms) by pointer arithmetic on the shared array, so the
  // compiler keeps shared-window loads (LDS) instead of generic ones
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* empty = full + kStages;
  uint64_t* sc_bar = full + 2 * kStages;    // score MMA done (tcgen05.commit)
  uint64_t* pv_bar = sc_bar + 1;            // PV MMA done (tcgen05.commit)
  uint64_t* a_rdy = sc_bar + 2;             // 4 warps: score A operand in TMEM
  uint64_t* mx_rdy = sc_bar + 3;            // 4 warps: tile maxima in smem
  uint64_t* p_rdy = sc_bar + 4;             // 4 warps: PV operands (B smem, A TMEM) ready
  uint64_t* bsc_bar = sc_bar + 5;           // the unit's score B image landed (bulk copy)
  // 32-bit shared addresses of the barriers and stages, computed once
  const uint32_t s_sm = smem_u32(sm);
  const uint32_t a_full = s_sm + L::oBar, a_empty = a_full + 8 * kStages;
  const uint32_t a_sc = a_full + 16 * kStages, a_pv = a_sc + 8, a_ardy = a_sc + 16, a_mx = a_sc + 24,
                 a_p = a_sc + 32, a_bsc = a_sc + 40;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::oTmem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = P.ctas;
  const int64_t T = P.total_tiles;
  // Work split.  grouped: unit u owns CTAs [u C / U, (u + 1) C / U); CTA k of the group
  // takes tiles k, k + g, k + 2g, ... so a group streams each cache array nearly
  // contiguously at any moment (DRAM row locality).  Otherwise contiguous stream-K
  // ranges of the flattened (unit, tile) space.
  int u_first, lt_first, ntiles, lt_step;
  if (P.grouped) {
    u_first = cta_of_tile(blockIdx.x, C, P.units);
    const int g0 = (int)tile_begin(u_first, C, P.units), g1 = (int)tile_begin(u_first + 1, C, P.units);
    lt_first = blockIdx.x - g0;
    lt_step = g1 - g0;
    ntiles = lt_first < P.tpu ? (P.tpu - lt_first + lt_step - 1) / lt_step : 0;
  } else {
    const int64_t r0 = tile_begin(blockIdx.x, T, C), r1 = tile_begin(blockIdx.x + 1, T, C);
    ntiles = (int)(r1 - r0);
    u_first = (int)(r0 / P.tpu);
    lt_first = (int)(r0 - (int64_t)u_first * P.tpu);
    lt_step = 1;
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    mbar_init(sc_bar, 1);
    mbar_init(pv_bar, 1);
    mbar_init(a_rdy, 4);
    mbar_init(mx_rdy, 4);
    mbar_init(p_rdy, 4);
    mbar_init(bsc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(L::kAlloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint64_t dsc0 = desc_sw128(smem_u32(sm + L::oBsc));
  const uint64_t dpv0 = desc_none(smem_u32(sm + L::oBpv), 128, 2048);
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);   // this warp's TMEM lanes

  // Every warp's lane 0 issues a share of the tile's bulk copies (the issue sequence of
  // a single-thread cp.async.bulk is ~15 instructions; spreading them keeps the warps
  // balanced at the tile barriers).  Copies may complete before the expect_tx arrive;
  // the phase cannot complete until that arrive.
  int iss_u = u_first, iss_lt = lt_first, iss_i = 0, iss_s = 0;
  uint32_t iss_ph = 0;                      // parity of the empty barrier of stage iss_s
  // running cache rows of the next tile (advanced by adds, rebuilt at unit boundaries)
  int64_t iss_row = (int64_t)u_first * P.kc.capacity + (int64_t)lt_first * kTile;
  int64_t iss_vrow = (int64_t)u_first * P.vc.capacity + (int64_t)lt_first * kTile;
  const uint64_t pol = evict_first_policy();   // L2 policy of the cache stream (read once)
  auto issue_next = [&]() {
    const int s = iss_s;
    if (iss_i >= kStages) mbar_wait(a_empty + 8 * s, iss_ph);
    const int64_t row = iss_row, vrow = iss_vrow;
    const uint32_t st = s_sm + L::oStage + s * L::kStageBytes;
    const uint32_t fb = a_full + 8 * s;
    if (QJL_UD_ABLATE & 1024) {                    // memory test: bits_in + codes only (8 KB/tile)
      if (warp == 0) {
        mbar_expect_tx(fb, L::kBitsIn + L::kCodes);
        bulk_g2s(st + L::oBitsIn, P.kc.bits_in + row * (KCI * 4), L::kBitsIn, fb);
      } else if (warp == 1) {
        bulk_g2s(st + L::oCodes, (const uint8_t*)P.vc.codes + vrow * 32, L::kCodes, fb);
      }
    } else if (QJL_UD_ABLATE & 2048) {             // memory test: no norms (bits, codes, consts)
      if (warp == 0) {
        mbar_expect_tx(fb, L::kBitsIn + L::kCodes + L::kBitsOut + 2 * L::kConst);
        bulk_g2s(st + L::oBitsIn, P.kc.bits_in + row * (KCI * 4), L::kBitsIn, fb);
      } else if (warp == 1) {
        bulk_g2s(st + L::oCodes, (const uint8_t*)P.vc.codes + vrow * 32, L::kCodes, fb);
      } else if (warp == 2) {
        if (KCO) bulk_g2s(st + L::oBitsOut, P.kc.bits_out + row * (KCO * 4), L::kBitsOut, fb);
      } else {
        bulk_g2s(st + L::oZero, (const uint8_t*)P.vc.zero + vrow * 8, L::kConst, fb);
        bulk_g2s(st + L::oScale, (const uint8_t*)P.vc.scale + vrow * 8, L::kConst, fb);
      }
    } else if (QJL_UD_EVICT_FIRST) {
      if (warp == 0) {
        mbar_expect_tx(fb, L::kStageBytes);
        bulk_g2s_hint(st + L::oBitsIn, P.kc.bits_in + row * (KCI * 4), L::kBitsIn, fb, pol);
      } else if (warp == 1) {
        bulk_g2s_hint(st + L::oCodes, (const uint8_t*)P.vc.codes + vrow * 32, L::kCodes, fb, pol);
      } else if (warp == 2) {
        bulk_g2s_hint(st + L::oNormIn, P.kc.norm_in + row, L::kNorm, fb, pol);
        if (KCO) {
          bulk_g2s_hint(st + L::oBitsOut, P.kc.bits_out + row * (KCO * 4), L::kBitsOut, fb, pol);
          bulk_g2s_hint(st + L::oNormOut, P.kc.norm_out + row, L::kNorm, fb, pol);
        }
      } else {
        bulk_g2s_hint(st + L::oZero, (const uint8_t*)P.vc.zero + vrow * 8, L::kConst, fb, pol);
        bulk_g2s_hint(st + L::oScale, (const uint8_t*)P.vc.scale + vrow * 8, L::kConst, fb, pol);
      }
    } else if (warp == 0) {
      mbar_expect_tx(fb, L::kStageBytes);
      bulk_g2s(st + L::oBitsIn, P.kc.bits_in + row * (KCI * 4), L::kBitsIn, fb);
    } else if (warp == 1) {
      bulk_g2s(st + L::oCodes, (const uint8_t*)P.vc.codes + vrow * 32, L::kCodes, fb);
    } else if (warp == 2) {
      bulk_g2s(st + L::oNormIn, P.kc.norm_in + row, L::kNorm, fb);
      if (KCO) {
        bulk_g2s(st + L::oBitsOut, P.kc.bits_out + row * (KCO * 4), L::kBitsOut, fb);
        bulk_g2s(st + L::oNormOut, P.kc.norm_out + row, L::kNorm, fb);
      }
    } else {
      bulk_g2s(st + L::oZero, (const uint8_t*)P.vc.zero + vrow * 8, L::kConst, fb);
      bulk_g2s(st + L::oScale, (const uint8_t*)P.vc.scale + vrow * 8, L::kConst, fb);
    }

    ++iss_i;
    if (++iss_s == kStages) {
      iss_s = 0;
      if (iss_i > kStages) iss_ph ^= 1;     // stages are re-armed from the second round on
    }
    iss_lt += lt_step;
    iss_row += (int64_t)lt_step * kTile;
    iss_vrow += (int64_t)lt_step * kTile;
    if (iss_lt >= P.tpu) {
      iss_lt = 0;
      ++iss_u;
      iss_row = (int64_t)iss_u * P.kc.capacity;
      iss_vrow = (int64_t)iss_u * P.vc.capacity;
    }
  };

  // the first copies overlap the prep grid (PDL); a decode step that appends a token
  // launches this kernel without PDL, so the prep's cache writes are complete here
  if (lane == 0)
    for (int i = 0; i < kLookahead && i < ntiles; ++i) issue_next();

  // per-thread running state: token-side partials (l, Z) and dim-side output (acc)
  float m_run[4], l_part[4], acc[4];
  float2 Z[4][2];                      // [q][group pair]
  // per-query estimator constants live in shared memory (L::oQc), not in 16 registers
  const float4* qcs = reinterpret_cast<const float4*>(sm + L::oQc);
  const float wrow = (tid & 3) == 0 ? 1.f : (tid & 3) == 1 ? 0.25f : (tid & 3) == 2 ? 0.0625f : 0.015625f;
  uint32_t tphase = 0;                      // parity of the per-tile barriers

  uint32_t bsc_phase = 0, bsc_par = 0;      // bsc_phase: 0 = wait for the copy before the next MMA
  auto load_unit = [&](int u) {
    bsc_phase = 0;
    // the unit's estimator constants -> smem; the first reader is behind the tile's first
    // CTA barrier (and the previous unit's last reader is behind flush's barriers)
    if (tid < 4) reinterpret_cast<float4*>(sm + L::oQc)[tid] = P.qconst[(int64_t)u * 4 + tid];
    // the unit's score B image: one bulk copy; only the MMA issuer waits for it
    if (tid == 0) {
      mbar_expect_tx(a_bsc, L::NH * 2048);
      bulk_g2s(s_sm + L::oBsc, P.bsc + (size_t)u * L::NH * 2048, L::NH * 2048, a_bsc);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      m_run[q] = -INFINITY;
      l_part[q] = 0.f;
      acc[q] = 0.f;
      Z[q][0] = Z[q][1] = make_float2(0.f, 0.f);
    }
  };

  auto flush = [&](int u) {
    if (QJL_UD_ABLATE & 4096) return;
    // token-side partials -> warp sums -> smem (the Bsc/Bpv region is free now)
    float v[20];
#pragma unroll
    for (int i = 0; i < 20; ++i) v[i] = 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      v[q] = l_part[q];
      v[4 + 4 * q + 0] = Z[q][0].x;
      v[4 + 4 * q + 1] = Z[q][0].y;
      v[4 + 4 * q + 2] = Z[q][1].x;
      v[4 + 4 * q + 3] = Z[q][1].y;
    }
    // CTA sums of the 20 token-side values, transposed through smem: every thread stores
    // its values, then warp w reduces values w, w + 4, ... (4 tokens per lane, then one
    // warp sum) -- 5 shuffle chains per warp instead of 20
    static_assert(L::NH * 2048 + 4 * 2048 >= (20 * kThreads + 20) * 4, "flush scratch must fit in Bsc/Bpv");
    float* tr = reinterpret_cast<float*>(sm + L::oRed);            // [20][128]
    float* red = tr + 20 * kThreads;                               // [20] CTA sums
    bar_sync1();                        // everyone is done with Bsc/Bpv
#pragma unroll
    for (int i = 0; i < 20; ++i)
      if (i < NQ || (i >= 4 && (i - 4) / 4 < NQ)) tr[i * kThreads + tid] = v[i];
    bar_sync1();
#pragma unroll
    for (int i0 = 0; i0 < 20; i0 += 4) {
      const int i = i0 + warp;
      if (i < NQ || (i >= 4 && (i - 4) / 4 < NQ)) {
        const float* t = tr + i * kThreads + lane;
        const float x = warp_sum((t[0] + t[32]) + (t[64] + t[96]));
        if (lane == 0) red[i] = x;
      }
    }
    bar_sync1();
    int ns, slot;
    if (P.grouped) {
      const int g0 = (int)tile_begin(u, C, P.units), g1 = (int)tile_begin(u + 1, C, P.units);
      ns = min(g1 - g0, P.tpu);
      slot = blockIdx.x - g0;
    } else {
      const int c0 = cta_of_tile((int64_t)u * P.tpu, T, C);
      const int c1 = cta_of_tile((int64_t)u * P.tpu + P.tpu - 1, T, C);
      ns = c1 - c0 + 1;
      slot = blockIdx.x - c0;
    }
    float* mypart = P.part + ((int64_t)u * P.max_seg + slot) * P.G * kRec;
    const int grp = tid >> 5;           // value group of dim tid
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (q < P.G) {
        const float lq = red[q];
        const float zq = red[4 + 4 * q + grp];
        if (tid == 0) {
          mypart[q * kRec + 0] = m_run[q];
          mypart[q * kRec + 1] = lq;
        }
        mypart[q * kRec + 2 + tid] = acc[q] + zq;
      }
    }
    int* flag = reinterpret_cast<int*>(sm + L::oFlag);
    if (ns > 1) {
      // publish: the CTA's partial writes are ordered before the counter increment by
      // one cumulative fence after the barrier (not one fence per thread)
      bar_sync1();
      if (tid == 0) {
        __threadfence();
        *flag = (atomicAdd(&P.counters[u], 1) == ns - 1);
      }
      bar_sync1();
      if (!*flag) return;
      __threadfence();
    } else {
      bar_sync1();
    }
    // last CTA of the unit: merge the ns partials.  (1) warp q turns the segments' (m, l)
    // into normalized weights w_s = 2^(m_s - M) / L in smem; (2) every thread sums its
    // (q, dim) outputs over the segments with all loads of a chunk in flight.
    const float* up = P.part + (int64_t)u * P.max_seg * P.G * kRec;
    float* wgt = reinterpret_cast<float*>(sm + L::oRed);          // [ns][4] (Bsc/Bpv are free)
    if (warp < P.G) {
      const int qq = warp;
      float M = -INFINITY;
      for (int s0 = lane; s0 < ns; s0 += 32) M = fmaxf(M, __ldcg(up + (s0 * P.G + qq) * kRec));
      M = warp_max_f32(M);
      float Ls = 0.f;
      for (int s0 = lane; s0 < ns; s0 += 32) {
        const float* W = up + (s0 * P.G + qq) * kRec;
        const float mv = __ldcg(W);
        const float f = (mv == -INFINITY) ? 0.f : ex2(mv - M);
        wgt[s0 * 4 + qq] = f;
        Ls = fmaf(f, __ldcg(W + 1), Ls);
      }
      Ls = warp_sum(Ls);
      __syncwarp();
      const float invL = 1.f / Ls;
      for (int s0 = lane; s0 < ns; s0 += 32) wgt[s0 * 4 + qq] *= invL;
      if (P.lse && lane == 0) P.lse[(int64_t)u * P.G + qq] = (M + __log2f(Ls)) * kLn2;
    }
    bar_sync1();
    {
      const int dim = tid;                                         // 128 threads = 128 dims
      float o[4] = {0.f, 0.f, 0.f, 0.f};
      for (int s0 = 0; s0 < ns; s0 += 8) {
        float av[4][8];
#pragma unroll
        for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            av[qq][k] = (qq < P.G && s0 + k < ns) ? __ldcg(up + ((s0 + k) * P.G + qq) * kRec + 2 + dim) : 0.f;
#pragma unroll
        for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (s0 + k < ns) o[qq] = fmaf(wgt[(s0 + k) * 4 + qq], av[qq][k], o[qq]);
      }
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq)
        if (qq < P.G) P.out[((int64_t)u * P.G + qq) * 128 + dim] = o[qq];
    }
  };

  asm volatile("griddepcontrol.wait;" ::: "memory");   // Bsc / qconst come from k_uprep
#if QJL_UD_TRACE
  if (tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_ud_trace[blockIdx.x][0] = gtimer();
    g_ud_trace[blockIdx.x][3] = smid;
  }
#endif
  const int n32 = (int)P.n;                            // n <= capacity < 2^30 (supported())
  int cur_u = -1;
  int u = u_first, lt = lt_first;
  int s = 0;
  uint32_t full_phase = 0;
  for (int it = 0; it < ntiles; ++it) {
    if (u != cur_u) {
      if (cur_u >= 0) flush(cur_u);
      load_unit(u);
      cur_u = u;
    }
    if (lane == 0 && it + kLookahead < ntiles) issue_next();
    mbar_wait(a_full + 8 * s, full_phase);
    const uint8_t* st = sm + L::oStage + s * L::kStageBytes;
    if (QJL_UD_ABLATE & 512) {                       // memory pipeline only
      __syncwarp();
      if (lane == 0) mbar_arrive(a_empty + 8 * s);
      lt += lt_step;
      if (lt >= P.tpu) { lt = 0; ++u; }
      if (++s == kStages) { s = 0; full_phase ^= 1; }
      tphase ^= 1;
      continue;
    }
    auto body = [&](auto mask_tag) {
    constexpr bool MASK = decltype(mask_tag)::value;
    const bool valid = !MASK || lt * kTile + tid < n32;            // this thread's token is < n

    // ---------------- 1. score A operand: masked sign words -> TMEM ----------------
    {
      uint32_t wv[KC];
      const uint4* bi = reinterpret_cast<const uint4*>(st + L::oBitsIn + tid * KCI * 4);
#pragma unroll
      for (int c = 0; c < KCI / 4; ++c) {
        const uint4 x = bi[c];
        wv[4 * c] = x.x; wv[4 * c + 1] = x.y; wv[4 * c + 2] = x.z; wv[4 * c + 3] = x.w;
      }
      if (KCO) {
        const uint2* bo = reinterpret_cast<const uint2*>(st + L::oBitsOut + tid * KCO * 4);
#pragma unroll
        for (int c = 0; c < KCO / 2; ++c) {
          const uint2 x = bo[c];
          wv[KCI + 2 * c] = x.x; wv[KCI + 2 * c + 1] = x.y;
        }
      }
      if (!(QJL_UD_ABLATE & 4)) {
#pragma unroll
        for (int c = 0; c < KC; c += 2) {
          uint32_t r[16];
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int b = 0; b < 8; ++b) r[8 * e + b] = wv[c + e] & (0x01010101u << b);
          tmem_st16(tlane + 8 * c, r);
        }
      }
    }
    tmem_wait_st();
    tc_fence_before();
#if QJL_UD_SPLIT
    __syncwarp();
    if (lane == 0) mbar_arrive(a_ardy);
#else
    bar_sync1();
#endif
    if (warp == 0 && !(QJL_UD_ABLATE & 1)) {
      if (elect_one()) {
        if (QJL_UD_SPLIT) mbar_wait(a_ardy, tphase);
        if (bsc_phase == 0) {                      // first tile of a unit: B image landed?
          mbar_wait(a_bsc, bsc_par);
          bsc_par ^= 1;
          bsc_phase = 1;
        }
        tc_fence_after();
        constexpr uint32_t ID = idesc_i8(16, 0);
        // descriptor start-address field is in 16-byte units: K chunk c -> +2 per 32 B,
        // +128 per 2 KB half image
        tc_mma_i8c<0>(tbase + L::cDsc, tbase, dsc0, ID);
#pragma unroll
        for (int c = 1; c < KCI; ++c)
          tc_mma_i8c<1>(tbase + L::cDsc, tbase + 8 * c, dsc0 + (uint64_t)((c >> 2) * 128 + (c & 3) * 2), ID);
        if (KCO) {
          constexpr int h0 = L::NHI * 128;
          tc_mma_i8c<0>(tbase + L::cDsc + 16, tbase + 8 * KCI, dsc0 + (uint64_t)h0, ID);
#pragma unroll
          for (int c = 1; c < KCO; ++c)
            tc_mma_i8c<1>(tbase + L::cDsc + 16, tbase + 8 * (KCI + c),
                          dsc0 + (uint64_t)(h0 + (c >> 2) * 128 + (c & 3) * 2), ID);
        }
        tc_commit(a_sc);
      }
      __syncwarp();
    }

    // token-side inputs that do not depend on the MMA
    const float nin = __half2float(reinterpret_cast<const __half*>(st + L::oNormIn)[tid]);
    const float nout = KCO ? __half2float(reinterpret_cast<const __half*>(st + L::oNormOut)[tid]) : 0.f;
    uint2 zr = reinterpret_cast<const uint2*>(st + L::oZero)[tid];
    uint2 sr = reinterpret_cast<const uint2*>(st + L::oScale)[tid];
    if (!valid) zr = sr = make_uint2(0u, 0u);              // rows past n

    // ---------------- 3. logits, tile maxima ----------------
    if (!(QJL_UD_ABLATE & 1)) mbar_wait(a_sc, tphase);
    tc_fence_after();
    float lg[4] = {nin, nin + 1.f, nin + 2.f, nin + 3.f};
    if (!(QJL_UD_ABLATE & 16)) {
      uint32_t dr[32];
      if (NQ == 4) {
        tmem_ld16(tlane + L::cDsc, dr);
        if (KCO) tmem_ld16(tlane + L::cDsc + 16, dr + 16);
      } else if (NQ == 2) {
        tmem_ld8(tlane + L::cDsc, dr);
        if (KCO) tmem_ld8(tlane + L::cDsc + 16, dr + 16);
      } else {
        tmem_ld4(tlane + L::cDsc, dr);
        if (KCO) tmem_ld4(tlane + L::cDsc + 16, dr + 16);
      }
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int* di = reinterpret_cast<const int*>(dr + 4 * q);
        const float fi = fmaf((float)(di[2] + 256 * di[3]), 65536.f, (float)(di[0] + 256 * di[1]));
        const float4 qc = qcs[q];
        float l2 = nin * fmaf(qc.x, fi, -qc.y);
        if (KCO) {
          const int* dq = reinterpret_cast<const int*>(dr + 16 + 4 * q);
          const float fo = fmaf((float)(dq[2] + 256 * dq[3]), 65536.f, (float)(dq[0] + 256 * dq[1]));
          l2 = fmaf(nout, fmaf(qc.z, fo, -qc.w), l2);
        }
        lg[q] = valid ? l2 : -INFINITY;
      }
    }
    {
      float* mx = reinterpret_cast<float*>(sm + L::oMax);
      const uint32_t hm = hmax2u(sr.x, sr.y);
      const float2 hf = h2f2(hm);
      const float smax_w = warp_max_f32(fmaxf(hf.x, hf.y));
      float tm[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < NQ; ++q) tm[q] = warp_max_f32(lg[q]);
      if (lane == 0) {
        *reinterpret_cast<float4*>(mx + warp * 8) = make_float4(tm[0], tm[1], tm[2], tm[3]);
        mx[warp * 8 + 4] = smax_w;
        if (QJL_UD_SPLIT) mbar_arrive(a_mx);   // release: the maxima are visible
      }
    }
    // A_pv row of dim tid (the score MMA is done, its A columns are free): 32 columns of
    // 4 tokens, value c * 4^(tid % 4) -- independent of the softmax, so it overlaps the
    // wait for the other warps' maxima
    // (the code words are read from the stage only here, so they hold no registers
    // across the score epilogue; the stage is released right after)
    {
      const uint32_t mk = 0x03030303u << (2 * (tid & 3));
      const uint4* cs = reinterpret_cast<const uint4*>(st + L::oCodes + (tid >> 2) * 128);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t cw[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint4 x = cs[4 * h + k];
          cw[4 * k] = x.x & mk; cw[4 * k + 1] = x.y & mk; cw[4 * k + 2] = x.z & mk; cw[4 * k + 3] = x.w & mk;
        }
        if (!(QJL_UD_ABLATE & 8)) tmem_st16(tlane + 16 * h, cw);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(a_empty + 8 * s);            // stage fully read by this warp
#if QJL_UD_SPLIT
    mbar_wait(a_mx, tphase);
#else
    if (!(QJL_UD_ABLATE & 64)) bar_sync1();
#endif

    // ---------------- 4. softmax, P' digits (tokens), code operand (dims) ----------------
    float tmax[4], smax;
    {
      const float* mx = reinterpret_cast<const float*>(sm + L::oMax);
      float4 a = *reinterpret_cast<const float4*>(mx), b = *reinterpret_cast<const float4*>(mx + 8),
             c = *reinterpret_cast<const float4*>(mx + 16), e = *reinterpret_cast<const float4*>(mx + 24);
      tmax[0] = fmaxf(fmaxf(a.x, b.x), fmaxf(c.x, e.x));
      tmax[1] = fmaxf(fmaxf(a.y, b.y), fmaxf(c.y, e.y));
      tmax[2] = fmaxf(fmaxf(a.z, b.z), fmaxf(c.z, e.z));
      tmax[3] = fmaxf(fmaxf(a.w, b.w), fmaxf(c.w, e.w));
      smax = fmaxf(fmaxf(mx[4], mx[12]), fmaxf(mx[20], mx[28]));
    }
    // p = 2^(lg - m_new) = pt * et with pt = 2^(lg - tmax) <= 1 and the tile-uniform
    // et = 2^(tmax - m_new); P' K = pt * scale * kPMax / smax <= kPMax, and the PV sums
    // come back scaled by invK = et * smax / kPMax
    const float ksm = smax > 0.f ? kPMax * rcp_approx(smax) : 0.f;
    float alpha[4], p[4], pk[4], invK[4];
    bool moved = false;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float m_new = fmaxf(m_run[q], tmax[q]);          // finite: every tile has a valid token
      alpha[q] = ex2(m_run[q] - m_new);
      moved |= alpha[q] != 1.f;
      m_run[q] = m_new;
      const float et = ex2(tmax[q] - m_new);
      const float pt = ex2(lg[q] - tmax[q]);
      p[q] = pt * et;
      pk[q] = pt * ksm;
      invK[q] = et * smax * (1.f / kPMax);
    }
    if (moved) {                                          // CTA-uniform
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float2 a2 = make_float2(alpha[q], alpha[q]), z2 = make_float2(0.f, 0.f);
        l_part[q] *= alpha[q];
        acc[q] *= alpha[q];
        Z[q][0] = fma2(Z[q][0], a2, z2);
        Z[q][1] = fma2(Z[q][1], a2, z2);
      }
    }
    const float2 z01 = h2f2(zr.x), z23 = h2f2(zr.y);
    const float2 s01 = h2f2(sr.x), s23 = h2f2(sr.y);
    uint32_t wv[4][4];                                    // [head q][group]
    {
      const float2 mg = make_float2(kMagic, kMagic);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        l_part[q] += p[q];
        const float2 pp = make_float2(p[q], p[q]);
        Z[q][0] = fma2(pp, z01, Z[q][0]);
        Z[q][1] = fma2(pp, z23, Z[q][1]);
        const float2 pk2 = make_float2(pk[q], pk[q]);
        const float2 w01 = fma2(pk2, s01, mg), w23 = fma2(pk2, s23, mg);
        wv[q][0] = __float_as_uint(w01.x);
        wv[q][1] = __float_as_uint(w01.y);
        wv[q][2] = __float_as_uint(w23.x);
        wv[q][3] = __float_as_uint(w23.y);
      }
    }
    // B_pv row of this token: column n = 16 q + 4 G + digit, digit = lo, mid, hi, 0 of
    // v(q, G) = rint(P' K): fma leaves u = v + 32896 in the mantissa, so the word
    // (w ^ 0x8080) & 0xFFFFFF is {lo, mid, hi, 0} (balanced digits) -- one LOP3 per (q, G)
    {
      uint4* bpv = reinterpret_cast<uint4*>(sm + L::oBpv) + tid;
#pragma unroll
      for (int q = 0; q < NQ && !(QJL_UD_ABLATE & 8); ++q) {
        uint32_t o[4];
#pragma unroll
        for (int G = 0; G < 4; ++G) {
          asm("lop3.b32 %0, %1, 0x8080, 0xFFFFFF, 0x28;" : "=r"(o[G]) : "r"(wv[q][G]));   // (a ^ b) & c
        }
        bpv[128 * q] = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // B_pv -> tensor core
    tmem_wait_st();
    tc_fence_before();
#if QJL_UD_SPLIT
    __syncwarp();
    if (lane == 0) mbar_arrive(a_p);
#else
    bar_sync1();
#endif

    // ---------------- 5. PV MMA ----------------
    if (warp == 0 && !(QJL_UD_ABLATE & 2)) {
      if (elect_one()) {
        if (QJL_UD_SPLIT) mbar_wait(a_p, tphase);
        tc_fence_after();
        constexpr uint32_t ID = idesc_i8(16 * NQ, 1);           // N = (head, group, digit)
        tc_mma_i8c<0>(tbase + 32, tbase, dpv0, ID);
        tc_mma_i8c<1>(tbase + 32, tbase + 8, dpv0 + 32, ID);       // + 512 B per 32 tokens
        tc_mma_i8c<1>(tbase + 32, tbase + 16, dpv0 + 64, ID);
        tc_mma_i8c<1>(tbase + 32, tbase + 24, dpv0 + 96, ID);
        tc_commit(a_pv);
      }
      __syncwarp();
    }

    // ---------------- 6. accumulate (thread = dim) ----------------
    if (!(QJL_UD_ABLATE & 2)) mbar_wait(a_pv, tphase);
    tc_fence_after();
    if (!(QJL_UD_ABLATE & 2)) {
      const int G = warp;                                   // value group of dim tid
      uint32_t dd[4][4];                                    // [head q][lo, mid, hi, pad]
#pragma unroll
      for (int q = 0; q < NQ; ++q) tmem_ld4(tlane + 32 + 16 * q + 4 * G, dd[q]);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float f = fmaf((float)(int)dd[q][2], 65536.f, (float)((int)dd[q][0] + 256 * (int)dd[q][1]));
        acc[q] = fmaf(f, invK[q] * wrow, acc[q]);
      }
    }
    };
    if ((lt + 1) * kTile <= n32) body(std::false_type{});
    else body(std::true_type{});
    lt += lt_step;
    if (lt >= P.tpu) { lt = 0; ++u; }
    if (++s == kStages) { s = 0; full_phase ^= 1; }
    tphase ^= 1;
  }
  // all tiles consumed: the next step's query-sketch kernel may start its math now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#if QJL_UD_TRACE
  if (tid == 0) g_ud_trace[blockIdx.x][1] = gtimer();
#endif
  if (cur_u >= 0) flush(cur_u);
  tc_fence_before();
  __syncthreads();
#if QJL_UD_TRACE
  if (tid == 0) g_ud_trace[blockIdx.x][2] = gtimer();
#endif
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(L::kAlloc));
}

// ===================================================================================
// Warp-specialized variant (KC <= 12): 8 warps per CTA, 2 CTAs per SM, 256 TMEM columns.
//   warps 0-3 ("T", thread t = token t): score accumulators -> logits, CTA tile maxima,
//             online softmax, P' digits (B operand of the PV MMA), zero-point sums;
//   warps 4-7 ("D", thread t = token t for the sign expansion, dim t for the values):
//             score A operand (tile i+1), PV A operand (tile i+1), both MMA issues, the
//             PV accumulators -> fp32 running output, and the cache streaming.
// The score accumulators and the P' operand are double buffered, so the T warps work
// on tile i while the D warps expand tile i+1 and run tile i's PV MMA.  All hand-offs
// are mbarriers (tcgen05.commit for MMA completion); there is no CTA-wide barrier in the
// steady state.  TMEM: A_sc [0, 96), D_sc[2] [96, 160), A_pv [160, 192), D_pv [192, 256).
// ===================================================================================
namespace wsd {
constexpr int kThreads = 256;
constexpr int kStages = 4;
constexpr int kLookahead = 2;
constexpr int cDsc0 = 96, cApv = 160, cDpv = 192;
}  // namespace wsd

template <int KCI, int KCO>
struct WLayout {
  static constexpr int KC = KCI + KCO;
  static constexpr int NHI = KCI / 4, NHO = (KCO + 3) / 4, NH = NHI + NHO;
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
  static constexpr int oBsc = 0;                                   // 1024-aligned, <= 6 KB
  static constexpr int oBpv = 6144;                                // [2][4 heads][128 tokens][16 B]
  static constexpr int oRed = oBpv;                                // flush scratch aliases B_pv
  static constexpr int oStage = oBpv + 2 * 8192;
  static constexpr int oMax = oStage + wsd::kStages * kStageBytes;  // [2][4 T warps][8] f32
  static constexpr int oPar = oMax + 2 * 4 * 8 * 4;                // [2][alpha 4, invK 4] f32
  static constexpr int oBar = oPar + 2 * 8 * 4;
  // full[S], empty[S], sc_done[2], sc_free[2], p_rdy[2], pvd[2], bsc
  static constexpr int kBars = 2 * wsd::kStages + 9;
  static constexpr int oTmem = oBar + kBars * 8;
  static constexpr int oFlag = oTmem + 4;
  static constexpr int kTotal = oFlag + 12 + 1024;
};

template <int KCI, int KCO>
__global__ void __launch_bounds__(wsd::kThreads, 2) k_wdecode(const Params P) {
  using L = WLayout<KCI, KCO>;
  constexpr int KC = KCI + KCO;
  static_assert(8 * KC <= wsd::cDsc0, "score A operand must fit below the accumulators");
  constexpr int S = wsd::kStages, LA = wsd::kLookahead;
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* empty = full + S;
  uint64_t* sc_done = full + 2 * S;   // [2] tcgen05.commit of the score MMA of tile i (buffer i & 1)
  uint64_t* sc_free = sc_done + 2;    // [2] 4 T warps read D_sc[i & 1]
  uint64_t* p_rdy = sc_done + 4;      // [2] 4 T warps wrote B_pv[i & 1] and par[i & 1]
  uint64_t* pvd = sc_done + 6;        // [2] tcgen05.commit of the PV MMA of tile i
  uint64_t* bsc_bar = sc_done + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::oTmem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wq = warp & 3, t4 = tid & 127;     // TMEM lane quadrant; token / dim of this thread
  const bool is_t = warp < 4;
  const int C = P.ctas;

  // grouped schedule only (host guarantees ctas >= units): unit u, tiles k, k + g, ...
  const int u = cta_of_tile(blockIdx.x, C, P.units);
  const int g0 = (int)tile_begin(u, C, P.units), g1 = (int)tile_begin(u + 1, C, P.units);
  const int k0 = blockIdx.x - g0, gstep = g1 - g0;
  const int ntiles = k0 < P.tpu ? (P.tpu - k0 + gstep - 1) / gstep : 0;
  if (ntiles == 0) return;                     // no tiles, no partial (ns counts only busy CTAs)

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sc_done[b], 1);
      mbar_init(&sc_free[b], 4);
      mbar_init(&p_rdy[b], 4);
      mbar_init(&pvd[b], 1);
    }
    mbar_init(bsc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tlane = tbase + ((uint32_t)(wq * 32) << 16);
  const uint64_t dsc0 = desc_sw128(smem_u32(sm + L::oBsc));
  const uint64_t dpv0 = desc_none(smem_u32(sm + L::oBpv), 128, 2048);
  auto tile_tok = [&](int i) -> int64_t { return (int64_t)(k0 + i * gstep) * kTile; };
  auto stage = [&](int i) -> const uint8_t* { return sm + L::oStage + (i % S) * L::kStageBytes; };

  // D warps' lane 0 stream the cache: the four warps split the seven copies of a tile
  auto issue = [&](int i) {
    const int s = i % S;
    if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
    const int64_t row = (int64_t)u * P.kc.capacity + tile_tok(i);
    const int64_t vrow = (int64_t)u * P.vc.capacity + tile_tok(i);
    uint8_t* st = sm + L::oStage + s * L::kStageBytes;
    if (wq == 0) {
      mbar_expect_tx(&full[s], L::kStageBytes);
      bulk_g2s(st + L::oBitsIn, P.kc.bits_in + row * (KCI * 4), L::kBitsIn, &full[s]);
    } else if (wq == 1) {
      bulk_g2s(st + L::oCodes, (const uint8_t*)P.vc.codes + vrow * 32, L::kCodes, &full[s]);
    } else if (wq == 2) {
      bulk_g2s(st + L::oNormIn, P.kc.norm_in + row, L::kNorm, &full[s]);
      if (KCO) {
        bulk_g2s(st + L::oBitsOut, P.kc.bits_out + row * (KCO * 4), L::kBitsOut, &full[s]);
        bulk_g2s(st + L::oNormOut, P.kc.norm_out + row, L::kNorm, &full[s]);
      }
    } else {
      bulk_g2s(st + L::oZero, (const uint8_t*)P.vc.zero + vrow * 8, L::kConst, &full[s]);
      bulk_g2s(st + L::oScale, (const uint8_t*)P.vc.scale + vrow * 8, L::kConst, &full[s]);
    }
  };

#ifndef QJL_WS_TCODES
#define QJL_WS_TCODES 1     // 1: the T warps build the PV code operand (balances the groups)
#endif
  auto codes_op = [&](int i) {               // P2T code words of dim t4 -> PV A operand
    const uint8_t* st = stage(i);
    uint32_t cw[32];
    const uint4* cs = reinterpret_cast<const uint4*>(st + L::oCodes + (t4 >> 2) * 128);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint4 x = cs[k];
      cw[4 * k] = x.x; cw[4 * k + 1] = x.y; cw[4 * k + 2] = x.z; cw[4 * k + 3] = x.w;
    }
    const uint32_t mk = 0x03030303u << (2 * (t4 & 3));
#pragma unroll
    for (int k = 0; k < 32; ++k) cw[k] &= mk;
    tmem_st16(tlane + wsd::cApv, cw);
    tmem_st16(tlane + wsd::cApv + 16, cw + 16);
  };
  // token-side state (T) / dim-side state (D)
  float m_run[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  float l_part[4] = {0.f, 0.f, 0.f, 0.f}, acc[4] = {0.f, 0.f, 0.f, 0.f};
  float2 Z[4][2];
#pragma unroll
  for (int q = 0; q < 4; ++q) Z[q][0] = Z[q][1] = make_float2(0.f, 0.f);

  if (!is_t) {
    // ================================ D warps ===================================
    const float wrow = (t4 & 3) == 0 ? 1.f : (t4 & 3) == 1 ? 0.25f : (t4 & 3) == 2 ? 0.0625f : 0.015625f;
    auto bar_d = [&]() { asm volatile("bar.sync 3, 128;" ::: "memory"); };
    auto signs = [&](int i) {                  // sign words of token t4 -> score A operand
      const uint8_t* st = stage(i);
      uint32_t wv[KC];
      const uint4* bi = reinterpret_cast<const uint4*>(st + L::oBitsIn + t4 * KCI * 4);
#pragma unroll
      for (int c = 0; c < KCI / 4; ++c) {
        const uint4 x = bi[c];
        wv[4 * c] = x.x; wv[4 * c + 1] = x.y; wv[4 * c + 2] = x.z; wv[4 * c + 3] = x.w;
      }
      if (KCO) {
        const uint2* bo = reinterpret_cast<const uint2*>(st + L::oBitsOut + t4 * KCO * 4);
#pragma unroll
        for (int c = 0; c < KCO / 2; ++c) {
          const uint2 x = bo[c];
          wv[KCI + 2 * c] = x.x; wv[KCI + 2 * c + 1] = x.y;
        }
      }
#pragma unroll
      for (int c = 0; c < KC; c += 2) {
        uint32_t r[16];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int b = 0; b < 8; ++b) r[8 * e + b] = wv[c + e] & (0x01010101u << b);
        tmem_st16(tlane + 8 * c, r);
      }
    };
    auto codes = [&](int i) {                  // P2T code words of dim t4 -> PV A operand
      const uint8_t* st = stage(i);
      uint32_t cw[32];
      const uint4* cs = reinterpret_cast<const uint4*>(st + L::oCodes + (t4 >> 2) * 128);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint4 x = cs[k];
        cw[4 * k] = x.x; cw[4 * k + 1] = x.y; cw[4 * k + 2] = x.z; cw[4 * k + 3] = x.w;
      }
      const uint32_t mk = 0x03030303u << (2 * (t4 & 3));
#pragma unroll
      for (int k = 0; k < 32; ++k) cw[k] &= mk;
      tmem_st16(tlane + wsd::cApv, cw);
      tmem_st16(tlane + wsd::cApv + 16, cw + 16);
    };
    auto mma_sc = [&](int i) {                 // elected thread of warp 4
      if (i >= 2) mbar_wait(&sc_free[i & 1], ((i - 2) >> 1) & 1);
      tc_fence_after();
      constexpr uint32_t ID = idesc_i8(16, 0);
      const uint32_t dsc = tbase + wsd::cDsc0 + 32 * (i & 1);
      tc_mma_i8c<0>(dsc, tbase, dsc0, ID);
#pragma unroll
      for (int c = 1; c < KCI; ++c)
        tc_mma_i8c<1>(dsc, tbase + 8 * c, dsc0 + (uint64_t)((c >> 2) * 128 + (c & 3) * 2), ID);
      if (KCO) {
        constexpr int h0 = L::NHI * 128;
        tc_mma_i8c<0>(dsc + 16, tbase + 8 * KCI, dsc0 + (uint64_t)h0, ID);
#pragma unroll
        for (int c = 1; c < KCO; ++c)
          tc_mma_i8c<1>(dsc + 16, tbase + 8 * (KCI + c), dsc0 + (uint64_t)(h0 + (c >> 2) * 128 + (c & 3) * 2), ID);
      }
      tc_commit(&sc_done[i & 1]);
    };

    // Software pipeline (iteration it): PV MMA of tile it, sign expansion of tile it+2
    // while that MMA runs, tile it's PV accumulators, code operand of tile it+1, and the
    // score MMA of tile it+2 -- the T warps always have the next score tile ready.
    if (lane == 0)
      for (int i = 0; i < LA + 2 && i < ntiles; ++i) issue(i);
    asm volatile("griddepcontrol.wait;" ::: "memory");   // the B image comes from k_uprep
    if (tid == 128) {
      mbar_expect_tx(bsc_bar, L::NH * 2048);
      bulk_g2s(sm + L::oBsc, P.bsc + (size_t)u * L::NH * 2048, L::NH * 2048, bsc_bar);
    }
    // prologue: score MMAs of tiles 0 and 1, code operand of tile 0
    mbar_wait(&full[0], 0);
    signs(0);
    if (!QJL_WS_TCODES) codes(0);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[0]);
    tmem_wait_st();
    tc_fence_before();
    bar_d();
    if (warp == 4) {
      if (elect_one()) {
        mbar_wait(bsc_bar, 0);
        mma_sc(0);
      }
      __syncwarp();
    }
    if (ntiles > 1) {
      mbar_wait(&full[1], 0);
      mbar_wait(&sc_done[0], 0);               // A_sc free
      tc_fence_after();
      signs(1);
      tmem_wait_st();
      tc_fence_before();
      bar_d();
      if (warp == 4) {
        if (elect_one()) mma_sc(1);
        __syncwarp();
      }
    }
    for (int it = 0; it < ntiles; ++it) {
      if (lane == 0 && it + LA + 2 < ntiles) issue(it + LA + 2);
      // 1. PV MMA of tile it (A_pv(it) was written and fenced in the previous iteration)
      mbar_wait(&p_rdy[it & 1], (it >> 1) & 1);
      const float* par = reinterpret_cast<const float*>(sm + L::oPar) + 8 * (it & 1);
      const float4 al = *reinterpret_cast<const float4*>(par), ik = *reinterpret_cast<const float4*>(par + 4);
      bar_d();                                 // par read by every D thread before the MMA
      if (warp == 4) {
        if (elect_one()) {
          tc_fence_after();
          constexpr uint32_t ID = idesc_i8(64, 1);
          const uint64_t bd = dpv0 + (uint64_t)((it & 1) * 512);      // + 8 KB per buffer
          tc_mma_i8c<0>(tbase + wsd::cDpv, tbase + wsd::cApv, bd, ID);
          tc_mma_i8c<1>(tbase + wsd::cDpv, tbase + wsd::cApv + 8, bd + 32, ID);
          tc_mma_i8c<1>(tbase + wsd::cDpv, tbase + wsd::cApv + 16, bd + 64, ID);
          tc_mma_i8c<1>(tbase + wsd::cDpv, tbase + wsd::cApv + 24, bd + 96, ID);
          tc_commit(&pvd[it & 1]);
        }
        __syncwarp();
      }
      // 2. score operand of tile it+2 while the PV MMA runs
      const bool more2 = it + 2 < ntiles;
      if (more2) {
        mbar_wait(&full[(it + 2) % S], ((it + 2) / S) & 1);
        mbar_wait(&sc_done[(it + 1) & 1], ((it + 1) >> 1) & 1);   // MMA_sc(it+1) done with A_sc
        tc_fence_after();
        signs(it + 2);
      }
      // 3. tile it's PV accumulators
      mbar_wait(&pvd[it & 1], (it >> 1) & 1);
      tc_fence_after();
      {
        uint32_t dd[4][4];                     // [head q][lo, mid, hi, pad] of this dim's group
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_ld4(tlane + wsd::cDpv + 16 * q + 4 * wq, dd[q]);
        tmem_wait_ld();
        const float a4[4] = {al.x, al.y, al.z, al.w}, k4[4] = {ik.x, ik.y, ik.z, ik.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float f = fmaf((float)(int)dd[q][2], 65536.f, (float)((int)dd[q][0] + 256 * (int)dd[q][1]));
          acc[q] = fmaf(f, k4[q] * wrow, acc[q] * a4[q]);
        }
      }
      // 4. code operand of tile it+1 (A_pv free: MMA_pv(it) done)
      if (it + 1 < ntiles) {
        if (!QJL_WS_TCODES) codes(it + 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(it + 1) % S]);
      }
      tmem_wait_st();
      tc_fence_before();
      // 5. score MMA of tile it+2
      if (more2) {
        bar_d();
        if (warp == 4) {
          if (elect_one()) mma_sc(it + 2);
          __syncwarp();
        }
      }
    }
  } else {
    // ================================ T warps ===================================
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float4 qcr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) qcr[q] = P.qconst[(int64_t)u * 4 + q];
    for (int it = 0; it < ntiles; ++it) {
      const uint8_t* st = stage(it);
      mbar_wait(&full[it % S], (it / S) & 1);
      const bool valid = tile_tok(it) + t4 < P.n;
      const float nin = __half2float(reinterpret_cast<const __half*>(st + L::oNormIn)[t4]);
      const float nout = KCO ? __half2float(reinterpret_cast<const __half*>(st + L::oNormOut)[t4]) : 0.f;
      uint2 zr = reinterpret_cast<const uint2*>(st + L::oZero)[t4];
      uint2 sr = reinterpret_cast<const uint2*>(st + L::oScale)[t4];
      if (!valid) zr = sr = make_uint2(0u, 0u);
      if (!QJL_WS_TCODES) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[it % S]);
      }
      // logits from the score accumulators of buffer it & 1
      mbar_wait(&sc_done[it & 1], (it >> 1) & 1);
      tc_fence_after();
      float lg[4];
      {
        uint32_t dr[32];
        const uint32_t dsc = tlane + wsd::cDsc0 + 32 * (it & 1);
        tmem_ld16(dsc, dr);
        if (KCO) tmem_ld16(dsc + 16, dr + 16);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sc_free[it & 1]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int* di = reinterpret_cast<const int*>(dr + 4 * q);
          const float fi = fmaf((float)(di[2] + 256 * di[3]), 65536.f, (float)(di[0] + 256 * di[1]));
          float l2 = nin * fmaf(qcr[q].x, fi, -qcr[q].y);
          if (KCO) {
            const int* dq = reinterpret_cast<const int*>(dr + 16 + 4 * q);
            const float fo = fmaf((float)(dq[2] + 256 * dq[3]), 65536.f, (float)(dq[0] + 256 * dq[1]));
            l2 = fmaf(nout, fmaf(qcr[q].z, fo, -qcr[q].w), l2);
          }
          lg[q] = valid ? l2 : -INFINITY;
        }
      }
      // CTA tile maxima over the 4 T warps (named barrier 2)
      float tmax[4], smax;
      {
        float* mx = reinterpret_cast<float*>(sm + L::oMax) + (it & 1) * 32;
        const float2 hf = h2f2(hmax2u(sr.x, sr.y));
        const float smax_w = warp_max_f32(fmaxf(hf.x, hf.y));
        float tm[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) tm[q] = warp_max_f32(lg[q]);
        if (lane == 0) {
          *reinterpret_cast<float4*>(mx + wq * 8) = make_float4(tm[0], tm[1], tm[2], tm[3]);
          mx[wq * 8 + 4] = smax_w;
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
        const float4 a = *reinterpret_cast<const float4*>(mx), b = *reinterpret_cast<const float4*>(mx + 8),
                     c = *reinterpret_cast<const float4*>(mx + 16), e = *reinterpret_cast<const float4*>(mx + 24);
        tmax[0] = fmaxf(fmaxf(a.x, b.x), fmaxf(c.x, e.x));
        tmax[1] = fmaxf(fmaxf(a.y, b.y), fmaxf(c.y, e.y));
        tmax[2] = fmaxf(fmaxf(a.z, b.z), fmaxf(c.z, e.z));
        tmax[3] = fmaxf(fmaxf(a.w, b.w), fmaxf(c.w, e.w));
        smax = fmaxf(fmaxf(mx[4], mx[12]), fmaxf(mx[20], mx[28]));
      }
      float alpha[4], p[4], K[4], invK[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float m_new = fmaxf(m_run[q], tmax[q]);
        alpha[q] = ex2(m_run[q] - m_new);
        m_run[q] = m_new;
        p[q] = ex2(lg[q] - m_new);
        const float bound = ex2(tmax[q] - m_new) * smax;
        K[q] = bound > 0.f ? kPMax * rcp_approx(bound) : 0.f;
        invK[q] = bound * (1.f / kPMax);
        l_part[q] = fmaf(l_part[q], alpha[q], p[q]);
      }
      const float2 z01 = h2f2(zr.x), z23 = h2f2(zr.y);
      const float2 s01 = h2f2(sr.x), s23 = h2f2(sr.y);
      uint32_t wv[4][4];
      {
        const float2 mg = make_float2(kMagic, kMagic);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 a2 = make_float2(alpha[q], alpha[q]), pp = make_float2(p[q], p[q]);
          const float2 z2 = make_float2(0.f, 0.f);
          Z[q][0] = fma2(pp, z01, fma2(Z[q][0], a2, z2));
          Z[q][1] = fma2(pp, z23, fma2(Z[q][1], a2, z2));
          const float pk = p[q] * K[q];
          const float2 pk2 = make_float2(pk, pk);
          const float2 w01 = fma2(pk2, s01, mg), w23 = fma2(pk2, s23, mg);
          wv[q][0] = __float_as_uint(w01.x);
          wv[q][1] = __float_as_uint(w01.y);
          wv[q][2] = __float_as_uint(w23.x);
          wv[q][3] = __float_as_uint(w23.y);
        }
      }
      if (QJL_WS_TCODES) {
        if (it >= 1) mbar_wait(&pvd[(it - 1) & 1], ((it - 1) >> 1) & 1);   // A_pv, B_pv, par free
        tc_fence_after();
        codes_op(it);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[it % S]);   // stage it fully read by this warp
      } else if (it >= 2) {
        mbar_wait(&pvd[it & 1], ((it - 2) >> 1) & 1);   // B_pv / par buffer free
      }
      {
        uint4* bpv = reinterpret_cast<uint4*>(sm + L::oBpv + (it & 1) * 8192) + t4;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t o[4];
#pragma unroll
          for (int G = 0; G < 4; ++G)
            asm("lop3.b32 %0, %1, 0x8080, 0xFFFFFF, 0x28;" : "=r"(o[G]) : "r"(wv[q][G]));
          bpv[128 * q] = make_uint4(o[0], o[1], o[2], o[3]);
        }
        if (t4 == 0) {
          float* par = reinterpret_cast<float*>(sm + L::oPar) + 8 * (it & 1);
          *reinterpret_cast<float4*>(par) = make_float4(alpha[0], alpha[1], alpha[2], alpha[3]);
          *reinterpret_cast<float4*>(par + 4) = make_float4(invK[0], invK[1], invK[2], invK[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // B_pv -> tensor core
      if (QJL_WS_TCODES) {
        tmem_wait_st();
        tc_fence_before();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_rdy[it & 1]);
    }
  }

  // ================================ flush ====================================
  __syncthreads();                              // both groups done; B_pv region is free
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  float* red = reinterpret_cast<float*>(sm + L::oRed);   // [4 T warps][20] + m_run[4] at 80
  if (is_t) {
    float v[20];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[q] = l_part[q];
      v[4 + 4 * q + 0] = Z[q][0].x;
      v[4 + 4 * q + 1] = Z[q][0].y;
      v[4 + 4 * q + 2] = Z[q][1].x;
      v[4 + 4 * q + 3] = Z[q][1].y;
    }
#pragma unroll
    for (int i = 0; i < 20; ++i) v[i] = warp_sum(v[i]);
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < 20; ++i) red[wq * 20 + i] = v[i];
    if (tid == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[80 + q] = m_run[q];
  }
  __syncthreads();
  const int ns = min(gstep, P.tpu), slot = k0;
  float* mypart = P.part + ((int64_t)u * P.max_seg + slot) * P.G * kRec;
  if (!is_t) {                                  // dim t4 of every head
    const int grp = t4 >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q < P.G) {
        float lq = 0.f, zq = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          lq += red[w * 20 + q];
          zq += red[w * 20 + 4 + 4 * q + grp];
        }
        if (t4 == 0) {
          mypart[q * kRec + 0] = red[80 + q];
          mypart[q * kRec + 1] = lq;
        }
        mypart[q * kRec + 2 + t4] = acc[q] + zq;
      }
    }
  }
  int* flag = reinterpret_cast<int*>(sm + L::oFlag);
  bool merge = true;
  if (ns > 1) {
    __threadfence();
    __syncthreads();
    if (tid == 0) *flag = (atomicAdd(&P.counters[u], 1) == ns - 1);
    __syncthreads();
    merge = *flag != 0;
    if (merge) __threadfence();
  } else {
    __syncthreads();
  }
  if (merge) {
    const float* up = P.part + (int64_t)u * P.max_seg * P.G * kRec;
    for (int i = tid; i < P.G * 128; i += wsd::kThreads) {
      const int qq = i >> 7, dim = i & 127;
      float M = -INFINITY, Ls = 0.f, a = 0.f;
      for (int s0 = 0; s0 < ns; s0 += 16) {
        float mv[16], lv[16], av[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float* W = up + ((s0 + k) * P.G + qq) * kRec;
          const bool ok = s0 + k < ns;
          mv[k] = ok ? __ldcg(W) : -INFINITY;
          lv[k] = ok ? __ldcg(W + 1) : 0.f;
          av[k] = ok ? __ldcg(W + 2 + dim) : 0.f;
        }
        float Mc = M;
#pragma unroll
        for (int k = 0; k < 16; ++k) Mc = fmaxf(Mc, mv[k]);
        const float rs = (M == -INFINITY) ? 0.f : ex2(M - Mc);
        Ls *= rs;
        a *= rs;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float f = (mv[k] == -INFINITY) ? 0.f : ex2(mv[k] - Mc);
          Ls = fmaf(f, lv[k], Ls);
          a = fmaf(f, av[k], a);
        }
        M = Mc;
      }
      P.out[((int64_t)u * P.G + qq) * 128 + dim] = a / Ls;
      if (P.lse && dim == 0) P.lse[(int64_t)u * P.G + qq] = (M + __log2f(Ls)) * kLn2;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

struct Plan {
  int tpu, ctas, max_seg, grouped, ws;
  int64_t T;
  size_t bsc_off, qconst_off, part_off, cnt_off, total;
};

template <int KCI, int KCO, int NQ>
static int occupancy() {
  using L = Layout<KCI, KCO>;
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(k_udecode<KCI, KCO, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    cudaFuncSetAttribute(k_udecode<KCI, KCO, NQ>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int o = 0;
    // The runtime's occupancy calculator reports 1 CTA/SM for kernels that use tcgen05
    // (it cannot know the TMEM footprint), so resident CTAs are derived from the
    // register file, shared memory and the 512 TMEM columns directly.
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_udecode<KCI, KCO, NQ>);
    int dev = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
    const int by_regs = 65536 / (regs_warp * (kThreads / 32));
    const int by_smem = smem_sm / (L::kTotal + 1024);
    o = by_regs < by_smem ? by_regs : by_smem;
    const int tmem_cap = 512 / L::kAlloc;
    occ = o < 1 ? 1 : (o > tmem_cap ? tmem_cap : o);
    if (const char* e = getenv("QJL_UD_OCC")) {        // experiments: fewer CTAs per SM
      const int v = atoi(e);
      if (v >= 1 && v < occ) occ = v;
    }
    if (getenv("QJL_DEBUG"))
      fprintf(stderr, "k_udecode<%d,%d,%d>: %d CTAs/SM (regs %d -> %d, smem %d/%d -> %d, tmem cols %d)\n", KCI,
              KCO, NQ, occ, fa.numRegs, by_regs, L::kTotal, smem_sm, by_smem, L::kAlloc);
  }
  return occ;
}

template <int KCI, int KCO>
static int occupancy_ws() {
  using L = WLayout<KCI, KCO>;
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(k_wdecode<KCI, KCO>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    cudaFuncSetAttribute(k_wdecode<KCI, KCO>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_wdecode<KCI, KCO>);
    int dev = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
    const int by_regs = 65536 / (regs_warp * (wsd::kThreads / 32));
    const int by_smem = smem_sm / (L::kTotal + 1024);
    int o = by_regs < by_smem ? by_regs : by_smem;
    occ = o < 1 ? 1 : (o > 2 ? 2 : o);        // 256 TMEM columns per CTA
    if (getenv("QJL_DEBUG"))
      fprintf(stderr, "k_wdecode<%d,%d>: %d CTAs/SM (regs %d -> %d, smem %d/%d -> %d)\n", KCI, KCO, occ,
              fa.numRegs, by_regs, L::kTotal, smem_sm, by_smem);
  }
  return occ;
}

static bool kc_dispatch(int kci, int kco, int* id) {
  const int pairs[][2] = {{8, 2}, {8, 4}, {8, 0}, {16, 2}, {16, 0}, {16, 4}};
  for (int i = 0; i < 6; ++i)
    if (pairs[i][0] == kci && pairs[i][1] == kco) { *id = i; return true; }
  return false;
}
static int nq_of(int G) { return G <= 1 ? 1 : G <= 2 ? 2 : 4; }
template <int NQ>
static int occupancy_by_id_nq(int id) {
  switch (id) {
    case 0: return occupancy<8, 2, NQ>();
    case 1: return occupancy<8, 4, NQ>();
    case 2: return occupancy<8, 0, NQ>();
    case 3: return occupancy<16, 2, NQ>();
    case 4: return occupancy<16, 0, NQ>();
    case 5: return occupancy<16, 4, NQ>();
  }
  return 1;
}
static int occupancy_by_id(int id, int G) {
  const int nq = nq_of(G);
  return nq == 1 ? occupancy_by_id_nq<1>(id) : nq == 2 ? occupancy_by_id_nq<2>(id) : occupancy_by_id_nq<4>(id);
}
static int occupancy_ws_by_id(int id) {
  switch (id) {
    case 0: return occupancy_ws<8, 2>();
    case 1: return occupancy_ws<8, 4>();
    case 2: return occupancy_ws<8, 0>();
  }
  return 0;
}
static int nh_by_id(int id) {
  const int nh[] = {3, 3, 2, 5, 4, 5};
  return nh[id];
}
static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

static Plan make_plan(const qjl_key_cache_t& kc, int64_t n, int G, int id) {
  Plan p;
  p.tpu = (int)((n + kTile - 1) / kTile);
  p.T = (int64_t)kc.units * p.tpu;
  // warp-specialized kernel (opt-in, QJL_UD_WS=1: measured 91 us vs 85 us for the
  // 4-CTA kernel at C3) when the score operand fits (KC <= 12) and every unit gets its
  // own CTA group
  p.ws = 0;
  if (id <= 2 && getenv("QJL_UD_WS") != nullptr) {
    const int64_t wslots = (int64_t)device_sm_count() * occupancy_ws_by_id(id);
    const int wctas = (int)(p.T < wslots ? p.T : wslots);
    if (wctas >= kc.units) {
      p.ws = 1;
      p.ctas = wctas;
    }
  }
  if (!p.ws) {
    const int64_t slots = (int64_t)device_sm_count() * occupancy_by_id(id, G);
    p.ctas = (int)(p.T < slots ? p.T : slots);
  }
  // contiguous stream-K ranges by default (every CTA within one tile of the mean); the
  // grouped schedule (QJL_UD_GROUPED=1) has uneven group sizes when CTAs / units is not
  // an integer and measured 2 % (C3) to 13 % (C5) slower
  p.grouped = (p.ctas >= kc.units && getenv("QJL_UD_GROUPED") != nullptr) ? 1 : 0;
  int ms = 1;
  for (int u = 0; u < kc.units; ++u) {
    int ns;
    if (p.grouped) {
      const int g = (int)(tile_begin(u + 1, p.ctas, kc.units) - tile_begin(u, p.ctas, kc.units));
      ns = g < p.tpu ? g : p.tpu;
    } else {
      ns = cta_of_tile((int64_t)u * p.tpu + p.tpu - 1, p.T, p.ctas) - cta_of_tile((int64_t)u * p.tpu, p.T, p.ctas) + 1;
    }
    ms = ms > ns ? ms : ns;
  }
  p.max_seg = ms;
  p.bsc_off = 0;
  p.qconst_off = align256((size_t)kc.units * nh_by_id(id) * 2048);
  p.part_off = p.qconst_off + align256((size_t)kc.units * 4 * 16);
  p.cnt_off = p.part_off + align256((size_t)kc.units * p.max_seg * G * kRec * 4);
  p.total = p.cnt_off + align256((size_t)kc.units * 4);
  return p;
}

}  // namespace ud

bool decode_umma_supported(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int G) {
  int id;
  return vc.layout == QJL_VLAYOUT_P2T && kc.d == 128 && G >= 1 && G <= 4 &&
         ud::kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id) && kc.capacity % ud::kTile == 0 &&
         vc.capacity % ud::kTile == 0 && kc.capacity < (int64_t(1) << 30) &&   // 32-bit token indices
         getenv("QJL_FORCE_SIMT") == nullptr;
}

size_t decode_umma_workspace(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, int G) {
  int id;
  ud::kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id);
  (void)vc;
  return ud::make_plan(kc, n, G, id).total;
}

template <int KCI, int KCO>
static int launch_umma_impl(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, const void* q,
                            int q_dtype, int G, const qjl_sketch_t& sk, float inv_t, float* out, float* lse, void* ws,
                            const ud::Plan& plan, const ud::Append& app, cudaStream_t st) {
  using namespace ud;
  if (app.k != nullptr && plan.ws) {             // the opt-in WS kernel prefetches before the prep ends
    set_error("decode_step: the warp-specialized decode (QJL_UD_WS) does not take appends");
    return QJL_ERR_UNSUPPORTED;
  }
  uint8_t* w = (uint8_t*)ws;
  uint8_t* bsc = w + plan.bsc_off;
  float4* qconst = (float4*)(w + plan.qconst_off);
  float* part = (float*)(w + plan.part_off);
  int* counters = (int*)(w + plan.cnt_off);
  constexpr int MT = (KCI + KCO) * 32;
  cudaLaunchAttribute pattr[1];
  pattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pattr[0].val.programmaticStreamSerializationAllowed = timing_enabled() ? 0 : 1;
  cudaLaunchConfig_t pcfg = {};
  pcfg.gridDim = dim3(kc.units);
  pcfg.blockDim = dim3(MT);
  pcfg.stream = st;
  pcfg.attrs = pattr;
  pcfg.numAttrs = 1;
  cudaError_t pe = cudaErrorInvalidValue;
#define QJL_UPREP(TQ, TS)                                                                              \
  pe = app.k ? cudaLaunchKernelEx(&pcfg, k_uprep<TQ, TS, KCI, KCO, true>, (const TQ*)q, G,            \
                                  (const TS*)sk.s_full, sk.unit_stride, inv_t, bsc, qconst, counters, app) \
             : cudaLaunchKernelEx(&pcfg, k_uprep<TQ, TS, KCI, KCO, false>, (const TQ*)q, G,           \
                                  (const TS*)sk.s_full, sk.unit_stride, inv_t, bsc, qconst, counters, app)
#define QJL_UPREP_S(TQ)                                                  \
  switch (sk.dtype) {                                                    \
    case QJL_BF16: QJL_UPREP(TQ, __nv_bfloat16); break;                  \
    case QJL_F16: QJL_UPREP(TQ, __half); break;                          \
    case QJL_F32: QJL_UPREP(TQ, float); break;                           \
    default: QJL_UPREP(TQ, double); break;                               \
  }
  switch (q_dtype) {
    case QJL_BF16: QJL_UPREP_S(__nv_bfloat16); break;
    case QJL_F16: QJL_UPREP_S(__half); break;
    case QJL_F32: QJL_UPREP_S(float); break;
    default: QJL_UPREP_S(double); break;
  }
#undef QJL_UPREP_S
#undef QJL_UPREP
  if (pe != cudaSuccess) return cuda_status(pe, "decode_umma_prep");
  QJL_LAUNCH_CHECK("decode_umma_prep");
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
  P.grouped = plan.grouped;
  P.bsc = bsc;
  P.qconst = qconst;
  P.part = part;
  P.counters = counters;
  P.out = out;
  P.lse = lse;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.ctas);
  if constexpr (KCI + KCO <= 12) {
    if (plan.ws) {
      occupancy_ws<KCI, KCO>();
      cfg.blockDim = dim3(wsd::kThreads);
      cfg.dynamicSmemBytes = WLayout<KCI, KCO>::kTotal;
    }
  }
  if (!plan.ws) {                               // (smem attributes: occupancy<> in launch_u)
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Layout<KCI, KCO>::kTotal;
  }
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = timing_enabled() ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  timing_begin(st);
  cudaError_t e = cudaSuccess;
  auto launch_u = [&]() -> cudaError_t {
    switch (nq_of(G)) {
      case 1: occupancy<KCI, KCO, 1>(); return cudaLaunchKernelEx(&cfg, k_udecode<KCI, KCO, 1>, P);
      case 2: occupancy<KCI, KCO, 2>(); return cudaLaunchKernelEx(&cfg, k_udecode<KCI, KCO, 2>, P);
      default: occupancy<KCI, KCO, 4>(); return cudaLaunchKernelEx(&cfg, k_udecode<KCI, KCO, 4>, P);
    }
  };
  if constexpr (KCI + KCO <= 12) {
    if (plan.ws) e = cudaLaunchKernelEx(&cfg, k_wdecode<KCI, KCO>, P);
    else e = launch_u();
  } else {
    e = launch_u();
  }
  timing_end(st);
  if (e != cudaSuccess) return cuda_status(e, "decode_umma");
  QJL_LAUNCH_CHECK("decode_umma");
  return QJL_OK;
}

static int launch_umma_any(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, const void* q,
                           int q_dtype, int G, const qjl_sketch_t& sk, float inv_t, float* out, float* lse, void* ws,
                           size_t ws_bytes, const ud::Append& app, cudaStream_t st) {
  int id;
  if (!ud::kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id)) return QJL_ERR_UNSUPPORTED;
  const ud::Plan plan = ud::make_plan(kc, n, G, id);
  if (ws_bytes < plan.total) {
    set_error("decode workspace needs %zu bytes", plan.total);
    return QJL_ERR_WORKSPACE;
  }
  switch (id) {
    case 0: return launch_umma_impl<8, 2>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, app, st);
    case 1: return launch_umma_impl<8, 4>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, app, st);
    case 2: return launch_umma_impl<8, 0>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, app, st);
    case 3: return launch_umma_impl<16, 2>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, app, st);
    case 4: return launch_umma_impl<16, 0>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, app, st);
    case 5: return launch_umma_impl<16, 4>(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, plan, app, st);
  }
  return QJL_ERR_UNSUPPORTED;
}

int launch_decode_umma(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, const void* q,
                       int q_dtype, int G, const qjl_sketch_t& sk, float inv_t, float* out, float* lse, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  ud::Append none{};
  return launch_umma_any(kc, vc, n, q, q_dtype, G, sk, inv_t, out, lse, ws, ws_bytes, none, st);
}

int launch_decode_step_umma(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, const void* q,
                            int q_dtype, int G, const qjl_sketch_t& sk, const int32_t* channels, int h,
                            const void* k_new, const void* v_new, float inv_t, float* out, float* lse, void* ws,
                            size_t ws_bytes, cudaStream_t st) {
  ud::Append app{};
  app.k = k_new;
  app.v = v_new;
  app.kc = kc;
  app.vc = vc;
  app.channels = channels;
  app.h = h;
  app.row = n;                                   // the new token's row; decode over n + 1
  return launch_umma_any(kc, vc, n + 1, q, q_dtype, G, sk, inv_t, out, lse, ws, ws_bytes, app, st);
}

}  // namespace qjl

#if QJL_UD_TRACE
extern "C" __attribute__((visibility("default"))) int qjl_debug_ud_trace(void* host, int ctas) {
  return (int)cudaMemcpyFromSymbol(host, qjl::ud::g_ud_trace, sizeof(unsigned long long) * 4 * ctas);
}
#endif
