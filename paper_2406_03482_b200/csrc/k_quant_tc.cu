// K1 on the 5th-gen tensor cores: key quantization K . S_full^T for bf16/fp16 keys
// (estimator.py:110-124 batched; kvcache.py:293-306 split via the zero-padded
// per-unit S_full) on sm_100a.
//
//  * persistent CTAs (one per SM) own equal contiguous ranges of the flattened
//    (unit, 128-token tile) space; the unit's S_full [MT x 128] stays resident in
//    shared memory (SWIZZLE_128B, K-major) and is reloaded only when the range
//    crosses into the next unit;
//  * warp 0: TMA producer -- 3-D tensor maps over keys [units][n][128] (tail rows
//    past n are zero-filled by the TMA unit) and S_full [units][MT][128];
//  * warp 1: single-thread tcgen05.mma issuer, M = 128 tokens, N = MT split into
//    NC chunks of CH <= 256 columns, K = 128 (8 x K16), fp32 accumulators in two
//    ping-pong TMEM buffers; A (the key tile) is read from TMEM (QJL_K1_ATMEM), so the
//    tensor core streams only S_full from shared memory and a key stage is free as soon
//    as the norm warps have read it (measured 145 -> 144 us at C4: shared-memory
//    bandwidth was not the limit);
//  * warps 2, 3, 12, 13 (K-half 0) and 14-17 (K-half 1): ||k_in||, ||k_out|| from the
//    staged key tile, one token row per thread pair: exact fp32 products, fp32 sums
//    with an error bound that decides the fp16 rounding, double-float (TwoSum)
//    recompute when it does not -> the reference's float64 norm at half precision;
//    with QJL_K1_ATMEM they also store their row halves into the TMEM A buffer of the
//    tile (warp w owns TMEM lanes 32 (w % 4) .. + 31, so norm warp w takes those rows);
//  * warps 4-11: epilogue, one set of 4 warps per TMEM buffer -- tcgen05.ld
//    32x32b (one token per thread), exact sign
//    test `x >= 0` (set.ge: -0.0 -> 1, NaN -> 0), 32 bits per word, stored as
//    the LSB-first sign words of the cache rows.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

#ifndef QJL_K1_ABLATE
#define QJL_K1_ABLATE 0      // perf experiments only (tools/k1_ablate.sh builds variants)
#endif

namespace qjl {
namespace qtc {

constexpr int kM = 128;          // tokens per tile (UMMA M)
constexpr int kK = 128;          // head dim
constexpr int kThreads = 576;   // 18 warps: TMA, MMA, norms (2, 3, 12, 13 | 14-17), epilogue (4-11)
#ifndef QJL_K1_PF
#define QJL_K1_PF 3
#endif
constexpr int kPf = QJL_K1_PF;   // key tiles prefetched into L2 ahead of the TMA stream

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
#ifndef QJL_K1_SUSPEND_NS
#define QJL_K1_SUSPEND_NS 0   // try_wait suspend-time hint (ns); 0 = default polling (measured faster)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
#if QJL_K1_SUSPEND_NS
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity), "n"(QJL_K1_SUSPEND_NS) : "memory");
#else
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
#endif
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// same, compile-time accumulate flag
template <int ACC>
__device__ __forceinline__ void tc_mma_f16c(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "n"(ACC));
}
// D (TMEM, f32) += A (TMEM: lane = token row, column j = K elements 2j, 2j + 1) x B (smem)
__device__ __forceinline__ void tc_mma_f16_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// K-major, SWIZZLE_128B smem matrix descriptor (rows of 128 B, 8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);           // start address
  d |= (uint64_t)1 << 16;                           // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                 // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                           // version (sm100)
  d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
  return d;
}
// instruction descriptor: D f32, A/B f16 (0) or bf16 (1), both K-major, M = 128
__host__ __device__ constexpr uint32_t make_idesc(int ab_format, int n) {
  return (1u << 4) | ((uint32_t)ab_format << 7) | ((uint32_t)ab_format << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(kM >> 4) << 24);
}

// 32 fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// exact sign word: bit i = (x_i >= 0) (set.ge: all-ones / zero, -0.0 -> 1, NaN -> 0),
// merged with LOP3 in four independent chains so the 32-deep OR dependency does
// not serialize the epilogue
__device__ __forceinline__ uint32_t sign_word(const uint32_t* r) {
  uint32_t a[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    uint32_t m;
    asm("set.ge.u32.f32 %0, %1, 0f00000000;" : "=r"(m) : "f"(__uint_as_float(r[i])));
    a[i & 3] |= m & (1u << i);
  }
  return (a[0] | a[1]) | (a[2] | a[3]);
}
#ifndef QJL_K1_FASTSIGN
#define QJL_K1_FASTSIGN 1
#endif
// Same bits with ~1.5 instructions per bit: x + 0 (one FFMA2 per pair) turns -0.0 into
// +0.0, then a funnel shift per element collects the sign bits and one NOT flips them.
// A NaN projection has NaN in every column of its row (the NaN key element meets every
// sketch row, padding zeros included), so checking the first column of the word keeps
// the reference's NaN -> 0.
__device__ __forceinline__ uint32_t sign_word_fast(const uint32_t* r) {
  uint32_t acc = 0;
#pragma unroll
  for (int i = 30; i >= 0; i -= 2) {
    float y0, y1;
    asm("{\n.reg .b64 a, b, c, o;\nmov.b64 a, {%2, %3};\nmov.b64 b, {%4, %4};\nmov.b64 c, {%5, %5};\n"
        "fma.rn.f32x2 o, a, b, c;\nmov.b64 {%0, %1}, o;\n}"
        : "=f"(y0), "=f"(y1)
        : "f"(__uint_as_float(r[i])), "f"(__uint_as_float(r[i + 1])), "f"(1.0f), "f"(0.0f));
    acc = __funnelshift_l(__float_as_uint(y1), acc, 1);
    acc = __funnelshift_l(__float_as_uint(y0), acc, 1);
  }
  const float x0 = __uint_as_float(r[0]);
  return (x0 != x0) ? 0u : ~acc;
}
#ifndef QJL_K1_ZEROACC
#define QJL_K1_ZEROACC 1
#endif
// QJL_K1_ZEROACC: every MMA accumulates onto a TMEM buffer the epilogue re-zeroed after
// draining it, so an all-zero dot product comes out as (+0) + (-0...) = +0 and the sign
// test needs no x + 0 (the sum of nonzero products is unchanged by adding +0)
__device__ __forceinline__ void tmem_zero64(uint32_t taddr) {
  const uint32_t z = 0u;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tmem_zero32(uint32_t taddr) {
  const uint32_t z = 0u;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(z)
      : "memory");
}
// sign word without the -0.0 fix-up (valid when accumulators start from +0): bit i =
// !sign(x_i), NaN rows -> 0
__device__ __forceinline__ uint32_t sign_word_raw(const uint32_t* r) {
  uint32_t acc = 0;
#pragma unroll
  for (int i = 31; i >= 0; --i) acc = __funnelshift_l(r[i], acc, 1);
  const float x0 = __uint_as_float(r[0]);
  return (x0 != x0) ? 0u : ~acc;
}
// 64 fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
      "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

#ifndef QJL_K1_ATMEM
#define QJL_K1_ATMEM 1   // A operand (the key tile) in TMEM, written by the norm warps
#endif
constexpr bool kAT = QJL_K1_ATMEM != 0;
static_assert(!kAT || QJL_K1_ZEROACC, "the TMEM-A MMAs always accumulate onto re-zeroed buffers");

#ifndef QJL_K1_HALFDRAIN
#define QJL_K1_HALFDRAIN 0  // 1: both epilogue sets drain every chunk, half the words each (measured 2 % slower)
#endif
#ifndef QJL_K1_TRACE
#define QJL_K1_TRACE 0      // diagnostics: per-CTA cycle counters of the MMA issuer (tools/k1_trace.py)
#endif
#if QJL_K1_TRACE
__device__ unsigned long long g_k1_trace[1024][6];   // [cta] {at_full wait, t_empty wait, b_full wait, issue, total, tiles}
#endif

template <int MT, int NC, int STAGES>
struct QLayout {
  static constexpr int CH = MT / NC;                       // columns per N chunk
  // TMEM accumulator buffers: NBUF of BUFW columns, so the MMA can run NBUF - 1 chunks
  // ahead of the epilogue.  kAT: columns [384, 512) hold two 64-column A buffers (one
  // 128 x 128 key tile each), the accumulators share [0, 384).
  static constexpr int BUFW = kAT ? (CH + 31) / 32 * 32 : CH <= 64 ? 64 : CH <= 128 ? 128 : 256;
  static constexpr int NBUF = (kAT ? 384 : 512) / BUFW;
  static constexpr int cA = 384;
  static constexpr int kBHalf = MT * 128;                  // one K-half of S_full (bytes)
  static constexpr int kABytes = kM * kK * 2;              // one key tile (32 KB)
  static constexpr int oB = 0;                             // S_full: [2 halves][MT rows][128 B]
  static constexpr int oA = 2 * kBHalf;                    // key tiles: [STAGES][2 halves][128][128 B]
  static constexpr int oBar = oA + STAGES * kABytes;
  // barriers: a_full[S], a_empty[S], b_full, b_empty, t_full[NBUF], t_empty[NBUF],
  // at_full[2], at_empty[2] (A buffers in TMEM)
  static constexpr int kBars = 2 * STAGES + 2 + 2 * NBUF + 4;
  static_assert(NBUF >= 2, "two accumulator buffers at least");
  static constexpr int oTmemPtr = oBar + kBars * 8;
  static constexpr int oMask = oTmemPtr + 16;              // per-unit outlier channel list
  static constexpr int oPart = oMask + 64 * 4;              // [2][128] K-half-1 partial sums
  static constexpr int kTotal = oPart + 2 * 128 * 4 + 1024; // + alignment slack
};

struct QParams {
  qjl_key_cache_t kc;
  int64_t n;                 // keys per unit in this call
  int64_t row_offset;        // first cache row
  const int32_t* channels;   // [units][h]
  int h;
  int tpu;                   // tiles per unit
  int64_t T;                 // total tiles
  int s_per_unit;            // 1: S_full has one slice per unit; 0: shared by all units
  int ablate;                // perf experiments only: 1 no epilogue math, 2 no norm math, 4 no MMA
  const uint8_t* keys;       // key base (for L2 prefetch of upcoming tiles)
  int64_t key_unit_bytes;    // bytes between units
};

template <int MT, int NC, int STAGES, int ABF>
__global__ void __launch_bounds__(kThreads, 1) k_quant_tc(const __grid_constant__ CUtensorMap tm_keys,
                                                          const __grid_constant__ CUtensorMap tm_s, const QParams P) {
  using L = QLayout<MT, NC, STAGES>;
  constexpr int CH = L::CH;
  constexpr uint32_t IDESC = make_idesc(ABF, CH);
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* a_full = bars;
  uint64_t* a_empty = bars + STAGES;
  uint64_t* b_full = bars + 2 * STAGES;
  uint64_t* b_empty = b_full + 1;
  uint64_t* t_full = b_full + 2;
  uint64_t* t_empty = t_full + L::NBUF;
  uint64_t* at_full = t_empty + L::NBUF;   // kAT: key tile it is in TMEM A buffer it % 2
  uint64_t* at_empty = at_full + 2;        // kAT: the MMAs reading A buffer b are done
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(sm + L::oTmemPtr);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * P.T / C, r1 = (int64_t)(blockIdx.x + 1) * P.T / C;
  const int ntiles = (int)(r1 - r0);
  const int m_in = P.kc.m_in, m_out = P.kc.m_out;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], kAT ? 8 : 1 + 8);   // (MMA commit unless A is in TMEM) + 8 norm warps
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&at_full[b], 8);          // the 8 norm warps stored their K-half rows
      mbar_init(&at_empty[b], 1);         // MMA commit
    }
    mbar_init(b_full, 1);
    mbar_init(b_empty, 1);
    for (int b = 0; b < L::NBUF; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], QJL_K1_HALFDRAIN ? 8 : 4);   // the epilogue warps draining the buffer
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_keys) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_s) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_ptr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // launched with programmatic serialization: the setup above overlaps the previous
  // kernel's tail (in a prefill, the S_full build); every global read and write follows
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem = *tmem_ptr;
  if (QJL_K1_ZEROACC) {
    // the accumulator buffers start at +0 (each epilogue warp zeroes its lane quadrant of
    // its set's buffer; afterwards the epilogue re-zeroes every group it drains)
    if (warp >= 4 && warp < 12) {
      const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp - 4) >> 2) * L::BUFW;
      for (int c = 0; c < L::BUFW; c += 64) tmem_zero64(base + c);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  const int u_first = (int)(r0 / P.tpu);
  const int lt_first = (int)(r0 - (int64_t)u_first * P.tpu);

  if (warp == 0) {
    // ================================ TMA producer ================================
    if (lane == 0) {
      int u = u_first, lt = lt_first, cur_u = -1, b_uses = 0;
      for (int it = 0; it < ntiles; ++it) {
        if (u != cur_u) {
          if (b_uses > 0) mbar_wait(b_empty, (b_uses - 1) & 1);   // MMAs of the previous unit are done
          mbar_expect_tx(b_full, 2 * L::kBHalf);
          const int us = P.s_per_unit ? u : 0;
          for (int hf = 0; hf < 2; ++hf)
            for (int c = 0; c < NC; ++c)
              tma_load_3d(sm + L::oB + hf * L::kBHalf + c * CH * 128, &tm_s, b_full, hf * 64, c * CH, us);
          cur_u = u;
          ++b_uses;
        }
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&a_empty[s], ((it / STAGES) - 1) & 1);
        mbar_expect_tx(&a_full[s], L::kABytes);
        uint8_t* a = sm + L::oA + s * L::kABytes;
        tma_load_3d(a, &tm_keys, &a_full[s], 0, lt * kM, u);
        tma_load_3d(a + L::kABytes / 2, &tm_keys, &a_full[s], 64, lt * kM, u);
        {   // pull the key tile kPf tiles ahead into L2 so its TMA refill hits L2
          int pu = u, plt = lt + kPf;
          while (plt >= P.tpu) { plt -= P.tpu; ++pu; }
          if (it + kPf < ntiles) {
            const int64_t rows = (int64_t)(P.n - (int64_t)plt * kM) < kM ? (P.n - (int64_t)plt * kM) : kM;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.keys + pu * P.key_unit_bytes +
                                                                             (int64_t)plt * kM * kK * 2),
                         "r"((uint32_t)(rows * kK * 2)) : "memory");
          }
        }
        if (++lt == P.tpu) { lt = 0; ++u; }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ==================================
    if (lane == 0) {
      int u = u_first, lt = lt_first, cur_u = -1, b_uses = 0, chunk = 0;
#if QJL_K1_TRACE
      long long tw_a = 0, tw_t = 0, tw_b = 0, t_iss = 0;
      const long long t_start = clock64();
#define K1T(var, stmt) { const long long c0_ = clock64(); stmt; var += clock64() - c0_; }
#else
#define K1T(var, stmt) stmt;
#endif
      for (int it = 0; it < ntiles; ++it) {
        if (u != cur_u) {
          K1T(tw_b, mbar_wait(b_full, b_uses & 1))
          cur_u = u;
          ++b_uses;
        }
        const int s = it % STAGES;
        const int ab = it & 1;                   // kAT: A buffer of this tile
        if (kAT) { K1T(tw_a, mbar_wait(&at_full[ab], (it >> 1) & 1)) }
        else { K1T(tw_a, mbar_wait(&a_full[s], (it / STAGES) & 1)) }
        tc_fence_after();
        // descriptors built once; the start-address field (bits 0-13, 16-byte units) takes
        // the K / chunk offsets as plain adds (all shared addresses are < 256 KB)
        const uint64_t ad0 = sw128_desc(smem_u32(sm + L::oA + s * L::kABytes));
        const uint64_t bd0 = sw128_desc(smem_u32(sm + L::oB));
        const uint32_t ta = tmem + L::cA + ab * 64;
        const bool do_mma = !(P.ablate & 4);
#pragma unroll
        for (int c = 0; c < NC; ++c, ++chunk) {
          const int buf = chunk % L::NBUF;
          if (chunk >= L::NBUF) { K1T(tw_t, mbar_wait(&t_empty[buf], ((chunk / L::NBUF) - 1) & 1)) }
          tc_fence_after();
          const uint32_t d_tmem = tmem + buf * L::BUFW;
          if (do_mma) {
#pragma unroll
            for (int k = 0; k < kK / 16; ++k) {
              const int hf = k >> 2, kk = k & 3;   // K-half, 32-byte step inside the 128-byte row
              const uint64_t bd = bd0 + (uint64_t)((hf * L::kBHalf + c * CH * 128 + kk * 32) >> 4);
              if (kAT) {
                tc_mma_f16_ta(d_tmem, ta + 8 * k, bd, IDESC);   // K16 = 8 columns of packed pairs
              } else {
                const uint64_t ad = ad0 + (uint64_t)((hf * (L::kABytes / 2) + kk * 32) >> 4);
                if (k == 0 && !QJL_K1_ZEROACC) tc_mma_f16c<0>(d_tmem, ad, bd, IDESC);
                else tc_mma_f16c<1>(d_tmem, ad, bd, IDESC);
              }
            }
          }
          tc_commit(&t_full[buf]);
        }
        if (kAT) tc_commit(&at_empty[ab]);       // A buffer free for tile it + 2
        else tc_commit(&a_empty[s]);             // key tile consumed by the tensor core
        const bool last_of_unit = (lt + 1 == P.tpu) || (it + 1 == ntiles);
        if (last_of_unit) tc_commit(b_empty);    // S_full of this unit no longer read
        if (++lt == P.tpu) { lt = 0; ++u; }
      }
#if QJL_K1_TRACE
      const long long t_tot = clock64() - t_start;
      g_k1_trace[blockIdx.x][0] = tw_a;
      g_k1_trace[blockIdx.x][1] = tw_t;
      g_k1_trace[blockIdx.x][2] = tw_b;
      g_k1_trace[blockIdx.x][3] = t_tot - tw_a - tw_t - tw_b;
      g_k1_trace[blockIdx.x][4] = t_tot;
      g_k1_trace[blockIdx.x][5] = ntiles;
#endif
#undef K1T
    }
  } else if (warp >= 14) {
    // ===================== norms, K-half 1: partial sums of squares ================
    const int nw = kAT ? (warp & 3) : warp - 14;    // kAT: rows of this warp's TMEM lane quadrant
    const int row = nw * 32 + lane;
    float* part = reinterpret_cast<float*>(sm + L::oPart);
    for (int it = 0; it < ntiles; ++it) {
      const int s = it % STAGES;
      mbar_wait(&a_full[s], (it / STAGES) & 1);
      const uint8_t* rowp = sm + L::oA + s * L::kABytes + L::kABytes / 2 + row * 128;
      float2 acc2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};           // 8 chains of 8 exact squares
      uint32_t kw[kAT ? 32 : 1];
      if (kAT) {
        // this row's K-half 1 (64 elements = 32 packed columns) -> TMEM A buffer it % 2
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 v = *reinterpret_cast<const uint4*>(rowp + ((j ^ (row & 7)) << 4));
          kw[4 * j] = v.x; kw[4 * j + 1] = v.y; kw[4 * j + 2] = v.z; kw[4 * j + 3] = v.w;
        }
        if (it >= 2) mbar_wait(&at_empty[it & 1], ((it >> 1) - 1) & 1);
        tc_fence_after();
        tmem_st32(tmem + ((uint32_t)(nw * 32) << 16) + L::cA + (it & 1) * 64 + 32, kw);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&at_full[it & 1]);
      }
      if (!(P.ablate & 2)) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t w[4];
          if (kAT) {
            w[0] = kw[4 * j]; w[1] = kw[4 * j + 1]; w[2] = kw[4 * j + 2]; w[3] = kw[4 * j + 3];
          } else {
            const uint4 v = *reinterpret_cast<const uint4*>(rowp + ((j ^ (row & 7)) << 4));
            w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = ABF ? make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xFFFF0000u))
                                 : __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
            float2& c = acc2[e];
            asm("{\n.reg .b64 x, y;\nmov.b64 x, {%2, %3};\nmov.b64 y, {%0, %1};\n"
                "fma.rn.f32x2 y, x, x, y;\nmov.b64 {%0, %1}, y;\n}"
                : "+f"(c.x), "+f"(c.y)
                : "f"(f.x), "f"(f.y));
          }
        }
      }
      part[(it & 1) * 128 + row] =
          ((acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y)) + ((acc2[2].x + acc2[2].y) + (acc2[3].x + acc2[3].y));
      asm volatile("bar.sync %0, 64;" ::"r"(4 + nw) : "memory");   // hand the partial to the pair
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_empty[s]);
    }
  } else if (warp < 4 || warp >= 12) {
    // ============================ norms (fp64, exact products) =====================
    const int nw = kAT ? (warp & 3) : warp < 4 ? warp - 2 : warp - 10;  // norm warp 0..3 (kAT: TMEM quadrant)
    const int ntid = nw * 32 + lane;             // token row of the tile
    int* chan = reinterpret_cast<int*>(sm + L::oMask);
    int u = u_first, lt = lt_first, cur_u = -1;
    for (int it = 0; it < ntiles; ++it) {
      if (u != cur_u) {
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (ntid < P.h) chan[ntid] = P.channels[(int64_t)u * P.h + ntid];
        asm volatile("bar.sync 2, 128;" ::: "memory");
        cur_u = u;
      }
      const int s = it % STAGES;
      mbar_wait(&a_full[s], (it / STAGES) & 1);
      const uint8_t* a = sm + L::oA + s * L::kABytes;
      // One token row per thread.  x^2 is exact in fp32 (<= 11-bit significands).  Fast
      // path: fp32 sum of squares with FFMA2 (4 chains, relative error <= 2^-19), and the
      // outlier channels summed exactly in fp64.  When the fp16 rounding of the inlier
      // norm is not decided by that bound, the row is recomputed as an unevaluated
      // double-float (TwoSum), which matches an fp64 accumulation to ~1e-14 relative.
      const int row = ntid;
      const int64_t tok = (int64_t)lt * kM + row;
      auto elem_pair = [&](uint32_t w) -> float2 {
        if (ABF) return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
        return __half22float2(*reinterpret_cast<const __half2*>(&w));
      };
      float all32 = 0.f;
      uint32_t kw[kAT ? 32 : 1];
      if (kAT) {
        // this row's K-half 0 -> TMEM A buffer it % 2, columns 0..31 (the MMA waits for it)
        const uint8_t* rowp = a + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 v = *reinterpret_cast<const uint4*>(rowp + ((j ^ (row & 7)) << 4));
          kw[4 * j] = v.x; kw[4 * j + 1] = v.y; kw[4 * j + 2] = v.z; kw[4 * j + 3] = v.w;
        }
        if (it >= 2) mbar_wait(&at_empty[it & 1], ((it >> 1) - 1) & 1);
        tc_fence_after();
        tmem_st32(tmem + ((uint32_t)(nw * 32) << 16) + L::cA + (it & 1) * 64, kw);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&at_full[it & 1]);
      }
      if (!(P.ablate & 2)) {
        float2 acc2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};         // 8 chains of 8 exact squares
#pragma unroll
        for (int hf = 0; hf < 1; ++hf) {         // K-half 0 here, K-half 1 in the pair warp
          const uint8_t* rowp = a + hf * (L::kABytes / 2) + row * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j) {          // 16-byte chunk j (swizzled position j ^ row%8)
            uint32_t w[4];
            if (kAT) {
              w[0] = kw[4 * j]; w[1] = kw[4 * j + 1]; w[2] = kw[4 * j + 2]; w[3] = kw[4 * j + 3];
            } else {
              const uint4 v = *reinterpret_cast<const uint4*>(rowp + ((j ^ (row & 7)) << 4));
              w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = elem_pair(w[e]);
              float2& c = acc2[e];
              asm("{\n.reg .b64 x, y;\nmov.b64 x, {%2, %3};\nmov.b64 y, {%0, %1};\n"
                  "fma.rn.f32x2 y, x, x, y;\nmov.b64 {%0, %1}, y;\n}"
                  : "+f"(c.x), "+f"(c.y)
                  : "f"(f.x), "f"(f.y));
            }
          }
        }
        all32 = ((acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y)) +
                ((acc2[2].x + acc2[2].y) + (acc2[3].x + acc2[3].y));
      }
      asm volatile("bar.sync %0, 64;" ::"r"(4 + nw) : "memory");     // pair's K-half-1 partial
      all32 += reinterpret_cast<const float*>(sm + L::oPart)[(it & 1) * 128 + row];
      double outl = 0.0;
      for (int j = 0; j < P.h; ++j) {             // outlier channels: read them back
        const int c = chan[j];
        const int hf = c >> 6, cc = c & 63;
        const uint8_t* rowp = a + hf * (L::kABytes / 2) + row * 128;
        const uint16_t bits = *reinterpret_cast<const uint16_t*>(rowp + ((((cc >> 3) ^ (row & 7)) << 4) | ((cc & 7) << 1)));
        const float x = ABF ? __uint_as_float((uint32_t)bits << 16) : __half2float(__ushort_as_half(bits));
        outl += (double)(x * x);                  // <= 64 exact terms, tiny fp64 work
      }
      // fp16 rounding decided in fp32: the exact squared norm lies within e32 of in32.
      // all32 = p0 + p1, each half summed in 8 fp32 chains of 8 exact squares combined
      // pairwise: <= 7 + 3 roundings of 2^-24 * (half sum) per half (all terms >= 0), one
      // more for p0 + p1, and outl32 and the subtraction add 2^-24 * all each: <= 13 *
      // 2^-24 * all = 7.7e-7 * all.  sqrt.rn and the widening products add <= 2 ulp per
      // side.  When both ends round to the same fp16 that is the norm.
      const float outl32 = (float)outl;
      const float in32 = fmaxf(all32 - outl32, 0.f);
      const float e32 = all32 * 8.5e-7f;
      uint16_t nin16 = f32_to_f16_bits(sqrtf(fmaxf(in32 - e32, 0.f)) * (1.f - 2.4e-7f));
      const bool in_ok = nin16 == f32_to_f16_bits(sqrtf(in32 + e32) * (1.f + 2.4e-7f));
      const float so = sqrtf(outl32);             // outl is exact; outl32 within 2^-24
      uint16_t nout16 = f32_to_f16_bits(so * (1.f - 4e-7f));
      if (nout16 != f32_to_f16_bits(so * (1.f + 4e-7f))) nout16 = f64_to_f16_bits(sqrt(outl));
      // Undecided rows (rare): the warp recomputes each one cooperatively -- lane l squares
      // elements 4l .. 4l + 3 of the row exactly and the fp64 sum is reduced across lanes
      // (exact for these 16-bit-significand squares), so a single undecided token costs the
      // warp ~20 instructions instead of a divergent 128-element double-float pass.
      unsigned amb = __ballot_sync(0xffffffffu, !in_ok) & (P.ablate & 2 ? 0u : 0xffffffffu);
      while (amb) {
        const int src = __ffs(amb) - 1;
        amb &= amb - 1;
        const int r = nw * 32 + src;               // token row being recomputed
        const int hf = lane >> 4, ch = (lane >> 1) & 7;
        const uint2 v = *reinterpret_cast<const uint2*>(a + hf * (L::kABytes / 2) + r * 128 +
                                                        ((ch ^ (r & 7)) << 4) + (lane & 1) * 8);
        const float2 f0 = elem_pair(v.x), f1 = elem_pair(v.y);
        double t = ((double)(f0.x * f0.x) + (double)(f0.y * f0.y)) + ((double)(f1.x * f1.x) + (double)(f1.y * f1.y));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == src) {
          const double v = t - outl;                 // NaN keys keep a NaN norm (np.linalg.norm)
          nin16 = f64_to_f16_bits(sqrt(v < 0.0 ? 0.0 : v));
        }
      }
      if (tok < P.n) {
        const int64_t no = row_off(u, P.row_offset + tok, 2, P.kc.capacity, P.kc.tile_stride);
        *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(P.kc.norm_in) + no) = f16_canon(nin16);
        if (m_out > 0) *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(P.kc.norm_out) + no) = f16_canon(nout16);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_empty[s]);
      if (++lt == P.tpu) { lt = 0; ++u; }
    }
  } else {
    // =============================== epilogue ====================================
    const int ew = warp & 3;                     // TMEM lane quadrant: lanes 32*ew .. 32*ew + 31
    const int set = (warp - 4) >> 2;             // this warp set drains the chunks of parity `set`
    const int row = ew * 32 + lane;              // token row of the tile
    int u = u_first, lt = lt_first, chunk = 0;
    for (int it = 0; it < ntiles; ++it) {
      const int64_t tok = (int64_t)lt * kM + row;
      const bool valid = tok < P.n;
      uint8_t* const rin = P.kc.bits_in + row_off(u, P.row_offset + tok, m_in / 8, P.kc.capacity, P.kc.tile_stride);
      uint8_t* const rout =
          m_out ? P.kc.bits_out + row_off(u, P.row_offset + tok, m_out / 8, P.kc.capacity, P.kc.tile_stride) : nullptr;
      for (int c = 0; c < NC; ++c, ++chunk) {
        if (!QJL_K1_HALFDRAIN && (chunk & 1) != set) continue;   // (whole-chunk mode: sets alternate chunks)
        const int buf = chunk % L::NBUF;
        mbar_wait(&t_full[buf], (chunk / L::NBUF) & 1);
        tc_fence_after();
        // QJL_K1_HALFDRAIN: both sets drain every chunk, set 0 its first ceil(W/2) sign words,
        // set 1 the rest, so a buffer is free after half the serial TMEM loads
        constexpr int W = CH / 32;
        const int wb = QJL_K1_HALFDRAIN ? (set ? (W + 1) / 2 : 0) : 0;
        const int we = QJL_K1_HALFDRAIN ? (set ? W : (W + 1) / 2) : W;
        const uint32_t tq = tmem + ((uint32_t)(ew * 32) << 16) + buf * L::BUFW;
        int w = wb;
#pragma unroll 1
        for (; w + 2 <= (P.ablate & 1 ? wb : we); w += 2) {
          uint32_t r[64];
          tmem_ld64(tq + w * 32, r);
          if (QJL_K1_ZEROACC) tmem_zero64(tq + w * 32);
          const uint32_t w0 = QJL_K1_ZEROACC ? sign_word_raw(r) : QJL_K1_FASTSIGN ? sign_word_fast(r) : sign_word(r);
          const uint32_t w1 = QJL_K1_ZEROACC ? sign_word_raw(r + 32)
                                             : QJL_K1_FASTSIGN ? sign_word_fast(r + 32) : sign_word(r + 32);
          const int sr = c * CH + w * 32;        // first sketch row of the word pair
          if (valid) {
            uint32_t* d0 = sr < m_in ? reinterpret_cast<uint32_t*>(rin) + (sr >> 5)
                                     : reinterpret_cast<uint32_t*>(rout) + ((sr - m_in) >> 5);
            const int s1 = sr + 32;
            uint32_t* d1 = s1 < m_in ? reinterpret_cast<uint32_t*>(rin) + (s1 >> 5)
                                     : reinterpret_cast<uint32_t*>(rout) + ((s1 - m_in) >> 5);
            if (d1 == d0 + 1 && ((reinterpret_cast<uintptr_t>(d0) & 7) == 0)) {
              *reinterpret_cast<uint2*>(d0) = make_uint2(w0, w1);
            } else {
              *d0 = w0;
              *d1 = w1;
            }
          }
        }
        if (w < we && !(P.ablate & 1)) {         // a single trailing 32-column word
          uint32_t r[32];
          tmem_ld32(tq + w * 32, r);
          if (QJL_K1_ZEROACC) tmem_zero32(tq + w * 32);
          const uint32_t wd = QJL_K1_ZEROACC ? sign_word_raw(r) : QJL_K1_FASTSIGN ? sign_word_fast(r) : sign_word(r);
          const int sr = c * CH + w * 32;
          if (valid) {
            if (sr < m_in)
              reinterpret_cast<uint32_t*>(rin)[sr >> 5] = wd;
            else
              reinterpret_cast<uint32_t*>(rout)[(sr - m_in) >> 5] = wd;
          }
        }
        if (QJL_K1_ZEROACC) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");   // zeros landed
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[buf]);
      }
      if (++lt == P.tpu) { lt = 0; ++u; }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ----------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

static bool encode_3d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, uint64_t d0, uint64_t d1,
                      uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box1) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  const cuuint32_t box[3] = {64, box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MT, int NC, int STAGES, int ABF>
static int launch_impl(const void* keys, int64_t n, int64_t kus, const qjl_sketch_t& sk, const int32_t* ch, int h,
                       const qjl_key_cache_t& kc, int64_t row_offset, cudaStream_t st) {
  using L = QLayout<MT, NC, STAGES>;
  const CUtensorMapDataType dt = ABF ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tk, ts;
  const uint64_t s_units = sk.unit_stride ? (uint64_t)kc.units : 1;
  if (!encode_3d(&tk, keys, dt, kK, (uint64_t)n, (uint64_t)kc.units, kK * 2, (uint64_t)kus * 2, kM) ||
      !encode_3d(&ts, sk.s_full, dt, kK, MT, s_units, kK * 2,
                 (uint64_t)(sk.unit_stride ? sk.unit_stride : (int64_t)MT * kK) * 2, L::CH)) {
    set_error("cuTensorMapEncodeTiled failed");
    return QJL_ERR_CUDA;
  }
  QParams P;
  P.kc = kc;
  P.n = n;
  P.row_offset = row_offset;
  P.channels = ch;
  P.h = h;
  P.tpu = (int)((n + kM - 1) / kM);
  P.T = (int64_t)kc.units * P.tpu;
  P.s_per_unit = sk.unit_stride ? 1 : 0;
  P.keys = (const uint8_t*)keys;
  P.ablate = QJL_K1_ABLATE;
  P.key_unit_bytes = kus * 2;
  auto kern = k_quant_tc<MT, NC, STAGES, ABF>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
  const int ctas = (int)(P.T < device_sm_count() ? P.T : device_sm_count());
  // programmatic serialization: the kernel's setup (barriers, TMEM allocation, tensor-map
  // prefetch) overlaps the previous kernel; it waits for it before touching memory
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = L::kTotal;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  timing_begin(st);
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tk, ts, P);
  timing_end(st);
  if (e != cudaSuccess) return cuda_status(e, "quantize_keys_tc");
  QJL_LAUNCH_CHECK("quantize_keys_tc");
  return QJL_OK;
}

}  // namespace qtc

int launch_quantize_keys_tc(const void* keys, int dtype, int64_t n, int64_t kus, const qjl_sketch_t& sk,
                            const int32_t* ch, int h, const qjl_key_cache_t& kc, int64_t row_offset,
                            cudaStream_t st) {
  using namespace qtc;
  if (kc.d != kK || !(dtype == QJL_BF16 || dtype == QJL_F16) || sk.dtype != dtype) return QJL_ERR_UNSUPPORTED;
  if (h > 64 || kus % 8 != 0 || kus == 0) return QJL_ERR_UNSUPPORTED;   // kus == 0: shared keys (SIMT)
  if (((uintptr_t)keys & 15) || ((uintptr_t)sk.s_full & 15)) return QJL_ERR_UNSUPPORTED;
  const int MT = kc.m_in + kc.m_out;
  const int abf = dtype == QJL_BF16;
#ifndef QJL_K1_NC576
#define QJL_K1_NC576 3       // 192-column chunks (2 TMEM buffers); 96-column chunks measured 24% slower
#endif
#define QJL_QT(MTV, NCV, SV)                                                                             \
  if (MT == MTV)                                                                                         \
    return abf ? launch_impl<MTV, NCV, SV, 1>(keys, n, kus, sk, ch, h, kc, row_offset, st)          \
               : launch_impl<MTV, NCV, SV, 0>(keys, n, kus, sk, ch, h, kc, row_offset, st);
  QJL_QT(256, kAT ? 2 : 1, 3)   // m = 256, no outliers (config 1 shape)
  QJL_QT(320, 2, 3)   // m_in 256 + m_out 64 (configs 3/5)
  QJL_QT(384, 2, 3)   // m_in 256 + m_out 128 (config 2)
  QJL_QT(512, kAT ? 4 : 2, 2)   // m = 512, no outliers
  QJL_QT(576, QJL_K1_NC576, 2)   // m_in 512 + m_out 64 (config 4)
#undef QJL_QT
  return QJL_ERR_UNSUPPORTED;
}

}  // namespace qjl

#if QJL_K1_TRACE
extern "C" __attribute__((visibility("default"))) int qjl_debug_k1_trace(void* host, int ctas) {
  return (int)cudaMemcpyFromSymbol(host, qjl::qtc::g_k1_trace, sizeof(unsigned long long) * 6 * ctas);
}
#endif
