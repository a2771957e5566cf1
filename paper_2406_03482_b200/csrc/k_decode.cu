// tcgen05 (5th-gen tensor core) QJL decode on tile-major P2T caches (sm_100a):
// K2 score estimator + K3 online softmax . V, and the scores-only K2.
//
// Cache: one contiguous record per (unit, 128-token tile) -- sign bits, fp16 norms,
// 2-bit value codes, fp16 zero/scale (include/qjl_b200.h) -- so a tile arrives with ONE
// bulk copy.
//
// One decode step = 2 launches chained with programmatic dependent launch (PDL):
//   k_uprep   one CTA per unit: Sq = S_full . q for the unit's G <= 4 query heads,
//             quantized to a 32-bit fixed-point integer, split into four int8 digits and
//             written as the score MMA's B operand (K-major, SWIZZLE_128B image); with an
//             append (decode step) it also quantizes the new token into row n.
//   k_udecode contiguous stream-K ranges over the flattened (unit, tile) space, 4 warps
//             per CTA, up to 4 CTAs per SM (128 TMEM columns each).  The CTA that
//             finishes a unit last (atomic counter) merges the unit's partials.
//
// Per 128-token tile (thread t owns token t for scoring and dim t for the values):
//  1. token: the packed sign words (estimator.py:110-124 layout) are expanded in place
//     into the u8 A operand of the score MMA -- `w & 0x01010101 << s` puts sign bits
//     8i + s of word w into four byte lanes of value 2^s * bit -- and stored to TMEM;
//     the 2^s weights are folded into the B digits.  [CTA barrier 1]
//  2. one thread: tcgen05.mma kind::i8 (A TMEM, B smem), M = 128 tokens, N = 16
//     (4 heads x 4 digits) per side: exact int32 2 * sum_set(Sq) (estimator.py:149-170).
//  3. token: logits of the heads (kvcache.py:311-329), warp maxima (redux.sync).
//     dim: its P2T code words masked in place (`w & 3 << 2(d % 4)`: 4 tokens of one
//     dim, value c * 4^(d % 4)) -> A operand of the PV MMA in TMEM.  [CTA barrier 2]
//  4. the stage is consumed: one thread refills it with the tile kStages ahead.  Tile
//     maxima and the online-softmax bookkeeping (kvcache.py:38-44) run lane-parallel
//     over the heads and are broadcast with shuffles.
//  5. token: P' = p * scale of its heads x 4 value groups in 24-bit fixed point
//     relative to the tile bound, three int8 digits by one FFMA (float magic-number
//     rounding) + one LOP3 -> the PV MMA's B operand (MN-major smem); zero-point term
//     sum p * zero on the CUDA cores.  [CTA barrier 3]
//  6. one thread: tcgen05.mma kind::i8 D[dim][(head, group, digit)] over the 128 tokens.
//  7. dim: the PV accumulators are read back at the start of the NEXT tile (after its
//     sign words are loaded), so the PV MMA overlaps the next tile's copy wait.
#include <cstdio>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace qjl {
namespace ud {

using namespace ptx;

constexpr int kThreads = 128;      // 4 warps; thread t: token t (scores) and dim t (PV)
#ifndef QJL_UD_SPLIT
#define QJL_UD_SPLIT 0             // 1: the MMA issuer waits on mbarriers the warps arrive on
#endif
constexpr bool kSplit = QJL_UD_SPLIT != 0;
constexpr int kTile = 128;         // tokens per tile
#ifndef QJL_UD_STAGES
#define QJL_UD_STAGES 3
#endif
constexpr int kStages = QJL_UD_STAGES;   // records in flight per CTA (a refill is issued kStages ahead)
constexpr int kRecF = 130;         // per (partial, query): m (log2 domain), l, out[128]
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kPMax = 8.0e6f;                  // P' fixed-point full scale (< 2^23)
constexpr float kMagic = 8388608.f;              // 2^23: fma(p, s, 2^23) leaves rint(p s) in the mantissa

// Decode-step append: the new token of every unit, quantized inside the
// query-sketch kernel (which streams S_full anyway) and written at row `row` before the
// decode kernel reads rows [0, row + 1).
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
  const uint8_t* rec;    // tile records [units][cap_tiles][rec_bytes]
  int64_t rec_bytes;
  int64_t cap_tiles;     // capacity / 128
  int64_t n;
  int G;
  int units;
  int tpu;               // tiles per unit holding rows < n
  int64_t total_tiles;
  int ctas;
  int max_seg;
  int chained;           // QJL_DECODE_CHAINED (informational here; the prep acts on it)
  int seg;               // QJL_DECODE_DETERMINISTIC: tiles per fixed segment (CTAs own whole
                         // segments; partial slot = segment index); 0: stream-K over tiles
  int spu;               // segments per unit (deterministic) -- total work units = units * spu
  const uint8_t* bsc;    // [units][NH][2048] score B operand images (SW128, K-major)
  const float4* qconst;  // [units][4 queries] {k_in, b_in, k_out, b_out} (log2 domain)
  float* part;           // [units][max_seg][G][kRecF]
  int* counters;         // [units]
  float* out;            // [units][G][128]
  float* lse;            // [units][G] or null
  float* logits;         // [units][G][n]: scores kernel (always), decode (optional, scaled by 1/T)
};

#ifndef QJL_UD_TRACE
#define QJL_UD_TRACE 0      // diagnostics only: per-CTA %globaltimer stamps (tools/trace_decode.py)
#endif
#if QJL_UD_TRACE
__device__ unsigned long long g_ud_trace[4096][4];   // [cta] {after wait, loop done, end, smid}
__device__ unsigned long long g_ud_stat[4096][4];    // [cta] {tiles, issue cycles, full-wait cycles, runs}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

__host__ __device__ __forceinline__ int64_t tile_begin(int64_t c, int64_t T, int64_t C) { return c * T / C; }
__host__ __device__ __forceinline__ int cta_of_tile(int64_t t, int64_t T, int C) {
  return (int)(((t + 1) * (int64_t)C + T - 1) / T) - 1;
}

// --------------------------------------------------------------- smem layout
template <int KCI, int KCO>
struct Layout {
  static constexpr int KC = KCI + KCO;
  static constexpr int NHI = KCI / 4, NHO = (KCO + 3) / 4, NH = NHI + NHO;   // 128-byte K halves of B
  // one stage = one tile record, fields in qjl_tile_record order
  static constexpr int oBitsIn = 0;
  static constexpr int oBitsOut = oBitsIn + kTile * KCI * 4;
  static constexpr int oNormIn = oBitsOut + kTile * KCO * 4;
  static constexpr int oNormOut = oNormIn + kTile * 2;
  static constexpr int oCodes = oNormOut + (KCO ? kTile * 2 : 0);
  static constexpr int oZero = oCodes + kTile * 32;
  static constexpr int oScale = oZero + kTile * 8;
  static constexpr int kRec = oScale + kTile * 8;
  static constexpr int kKeyRec = oCodes;                // the key fields (scores-only stages)
  static constexpr int oBsc = 0;                        // 1024-aligned
  static constexpr int oBpv = oBsc + NH * 2048;         // [4 heads][128 tokens][16 B] (MN-major chunks)
  static constexpr int oRed = oBsc;                     // flush scratch aliases Bsc/Bpv
  static constexpr int oStage = oBpv + 4 * 2048;
  static constexpr int oMax = oStage + kStages * kRec;  // [8 slots][4 warps] tile maxima
  static constexpr int oQc = oMax + 4 * 8 * 4;          // [4 queries] float4 estimator constants
  static constexpr int oBar = oQc + 4 * 16;
  static constexpr int kBars = kStages + 6;             // full[kStages], score MMA, PV MMA, B image, A ready, P ready,
                                                        // first score-MMA half (split-K decode)
  static constexpr int oTmem = oBar + kBars * 8;
  static constexpr int oFlag = oTmem + 4;
  static constexpr int kTotal = oFlag + 12 + 1024;      // + alignment slack
  // scores-only kernel: B image, key stages, constants, barriers
  static constexpr int sStage = NH * 2048;
  static constexpr int sQc = sStage + kStages * kKeyRec;
  static constexpr int sBar = sQc + 4 * 16;
  static constexpr int sTmem = sBar + (kStages + 3) * 8;
  static constexpr int sTotal = sTmem + 16 + 1024;
  // TMEM columns: A_sc [0, 8 KC); after the score MMA: A_pv [0, 32), D_pv [32, 96);
  // D_sc (in: 16, out: 16) after both
  static constexpr int cDsc = (8 * KC > 96) ? 8 * KC : 96;
  static constexpr int kCols = cDsc + (KCO ? 32 : 16);
  static constexpr int kAlloc = kCols <= 128 ? 128 : 256;
  static_assert(kRec % 16 == 0 && kKeyRec % 16 == 0, "bulk copies move multiples of 16 bytes");
  static_assert(NH * 2048 + 4 * 2048 >= (20 * kThreads + 20) * 4, "flush scratch must fit in Bsc/Bpv");
};

// Decode TMEM geometry.  m_in = 512 (KC > 12): the score MMA runs in two K halves whose
// A operands (<= 80 columns each) reuse columns [0, 96), so D_sc sits at 96 and a CTA
// needs 128 columns -- 3 CTAs per SM instead of 2 with a 256-column allocation.
template <int KCI, int KCO>
struct DecTmem {
  static constexpr int KC = KCI + KCO;
  static constexpr bool SK = KC > 12;
  static constexpr int KH = SK ? KCI / 2 : KC;          // sign words in the first half
  static constexpr int cDsc = SK ? 96 : Layout<KCI, KCO>::cDsc;
  static constexpr int kAlloc = SK ? 128 : Layout<KCI, KCO>::kAlloc;
  static_assert(!SK || 8 * (KC - KH) <= 96, "second A half must fit below D_sc");
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
//
// PDL: without `chained` the kernel waits for the stream (griddepcontrol.wait) before it
// reads anything.  With `chained` (QJL_DECODE_CHAINED: the previous kernel on the stream
// is this library's decode and every input predates it) the reads and the math overlap
// the previous decode's tail, and only the workspace writes wait for it.
template <typename TQ, typename TS, int KCI, int KCO, bool APPEND>
__global__ void __launch_bounds__(640) k_uprep(const TQ* __restrict__ q, int G, const TS* __restrict__ s_full,
                                               int64_t s_unit_stride, float inv_t, int chained,
                                               uint8_t* __restrict__ bsc, float4* __restrict__ qconst,
                                               int* __restrict__ counters, const Append A) {
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
  if (!chained) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int u = blockIdx.x;
  const TS* S = s_full + (int64_t)u * s_unit_stride;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  // 16-bit sketches: the thread's whole S row (256 B) is requested before anything else,
  // so one memory round trip covers it
  uint4 srow[F32 ? 16 : 1];
  if constexpr (F32) {
    const uint4* rp = reinterpret_cast<const uint4*>(S + (int64_t)threadIdx.x * d);
#pragma unroll
    for (int i = 0; i < 16; ++i) srow[i] = __ldg(rp + i);
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
  // grid-dependency wait when chained) already see it.  Row n is padding for the previous
  // step's decode (masked), so writing it while that decode drains is harmless.
  // Arithmetic: K1's fp64 path and the value quantizer's (kvcache.py:293-306, :140-161).
  double vzero = 0.0, vscale = 0.0;
  uint32_t vbyte = 0;                         // this lane's P2T byte (dims 4a..4a+3)
  if constexpr (APPEND) {
    __syncthreads();                          // kd / vd / outl_ch
    if (threadIdx.x < A.h) {
      const int c = A.channels[(int64_t)u * A.h + threadIdx.x];
      if (c >= 0 && c < d) outl_ch[c] = 1;
    }
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
      const double spread = mx - mn;
      vzero = mn;
      vscale = spread == 0.0 ? 0.0 : spread / 3.0;
      int code = 0;
      if (spread != 0.0) code = (int)fmin(fmax(rint((x - mn) / vscale), 0.0), 3.0);
      uint32_t b = (uint32_t)code << (2 * (lane & 3));
      b |= __shfl_xor_sync(0xffffffffu, b, 1);
      b |= __shfl_xor_sync(0xffffffffu, b, 2);
      vbyte = b;
    }
    __syncthreads();                          // an
    const int64_t cap = A.kc.capacity, ts = A.kc.tile_stride;
    if (threadIdx.x < MT / 32) {
      const int w = threadIdx.x;
      if (w < MI / 32) reinterpret_cast<uint32_t*>(A.kc.bits_in + row_off(u, A.row, MI / 8, cap, ts))[w] = aw[w];
      else reinterpret_cast<uint32_t*>(A.kc.bits_out + row_off(u, A.row, MO / 8, cap, ts))[w - MI / 32] = aw[w];
    }
    if (threadIdx.x == 0) {
      const double sin = (an[0][0] + an[1][0]) + (an[2][0] + an[3][0]);
      const double sout = (an[0][1] + an[1][1]) + (an[2][1] + an[3][1]);
      const int64_t no = row_off(u, A.row, 2, cap, ts);
      *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(A.kc.norm_in) + no) = f16_canon(f64_to_f16_bits(sqrt(sin)));
      if (MO)
        *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(A.kc.norm_out) + no) =
            f16_canon(f64_to_f16_bits(sqrt(sout)));
    }
    if (wid < 4) {
      if ((lane & 3) == 0)
        reinterpret_cast<uint8_t*>(A.vc.codes)[tile_off(u, A.row, 4096, cap, ts) + p2t_byte(A.row, threadIdx.x)] =
            (uint8_t)vbyte;
      if (lane == 0) {
        const int64_t co = row_off(u, A.row, 8, cap, ts) + 2 * wid;
        *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(A.vc.zero) + co) = f64_to_f16_bits(vzero);
        *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(A.vc.scale) + co) = f64_to_f16_bits(vscale);
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
    // j - lo = lane (mod 32), so the weight 2^-(j mod 8) is fixed per lane; scaling by a
    // power of two is exact, so this is rint(Sq_j / (sigma 2^(j mod 8))) bit for bit
    const int sh = lane & 7;
    const double inv = 1.0 / red[g][side][0] / (double)(1 << sh);
    long long acc = 0;
    for (int j = lo + lane; j < hi; j += 32) {
      int32_t x = (int32_t)rint((double)sq[g][j] * inv);
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
  // The workspace writes below must wait for the previous decode (it reads them).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) counters[u] = 0;
  {
    uint4* out = reinterpret_cast<uint4*>(bsc + (size_t)u * L::NH * 2048);
    for (int i = threadIdx.x; i < L::NH * 128; i += blockDim.x) out[i] = reinterpret_cast<const uint4*>(img)[i];
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

// ------------------------------------------------------- shared tile stages
// Score A operand: the thread's sign words (token t of the tile) expanded into TMEM.
template <int KCI, int KCO>
__device__ __forceinline__ void load_sign_words(const uint8_t* st, int tid, uint32_t* wv) {
  using L = Layout<KCI, KCO>;
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
}
template <int KC>
__device__ __forceinline__ void store_sign_operand(uint32_t tlane, const uint32_t* wv) {
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
// one elected thread: the score MMAs of a tile (exact int32 2 * sum_set(Sq) per head digit)
template <int KCI, int KCO>
__device__ __forceinline__ void issue_score_mma(uint32_t tbase, uint64_t dsc0) {
  using L = Layout<KCI, KCO>;
  constexpr uint32_t ID = idesc_i8(16, 0);
  // descriptor start address is in 16-byte units: K chunk c -> +2 per 32 B, +128 per 2 KB half
  mma_i8<0>(tbase + L::cDsc, tbase, dsc0, ID);
#pragma unroll
  for (int c = 1; c < KCI; ++c)
    mma_i8<1>(tbase + L::cDsc, tbase + 8 * c, dsc0 + (uint64_t)((c >> 2) * 128 + (c & 3) * 2), ID);
  if (KCO) {
    constexpr int h0 = L::NHI * 128;
    mma_i8<0>(tbase + L::cDsc + 16, tbase + 8 * KCI, dsc0 + (uint64_t)h0, ID);
#pragma unroll
    for (int c = 1; c < KCO; ++c)
      mma_i8<1>(tbase + L::cDsc + 16, tbase + 8 * (KCI + c), dsc0 + (uint64_t)(h0 + (c >> 2) * 128 + (c & 3) * 2), ID);
  }
}
// sign words [W0, W1) of the thread's token row (in-side words first, then out-side)
template <int KCI, int KCO, int W0, int W1>
__device__ __forceinline__ void load_sign_range(const uint8_t* st, int tid, uint32_t* wv) {
  using L = Layout<KCI, KCO>;
  static_assert(W0 % 4 == 0 && (W1 <= KCI ? W1 % 4 == 0 : (W1 - KCI) % 2 == 0), "vector-aligned ranges");
  const uint4* bi = reinterpret_cast<const uint4*>(st + L::oBitsIn + tid * KCI * 4);
#pragma unroll
  for (int c = W0 / 4; c < (W1 < KCI ? W1 : KCI) / 4; ++c) {
    const uint4 x = bi[c];
    wv[4 * c - W0] = x.x; wv[4 * c + 1 - W0] = x.y; wv[4 * c + 2 - W0] = x.z; wv[4 * c + 3 - W0] = x.w;
  }
  if (KCO && W1 > KCI) {
    const uint2* bo = reinterpret_cast<const uint2*>(st + L::oBitsOut + tid * KCO * 4);
#pragma unroll
    for (int c = 0; c < (W1 - KCI) / 2; ++c) {
      const uint2 x = bo[c];
      wv[KCI - W0 + 2 * c] = x.x; wv[KCI - W0 + 2 * c + 1] = x.y;
    }
  }
}
// split-K score MMAs: half 0 = in-side chunks [0, KH) at A columns 8 c; half 1 = in-side
// chunks [KH, KCI) and the out-side chunks, at A columns from 0 again
template <int KCI, int KCO, int HALF>
__device__ __forceinline__ void issue_score_mma_half(uint32_t tbase, uint64_t dsc0) {
  using L = Layout<KCI, KCO>;
  using T = DecTmem<KCI, KCO>;
  constexpr uint32_t ID = idesc_i8(16, 0);
  if (HALF == 0) {
    mma_i8<0>(tbase + T::cDsc, tbase, dsc0, ID);
#pragma unroll
    for (int c = 1; c < T::KH; ++c)
      mma_i8<1>(tbase + T::cDsc, tbase + 8 * c, dsc0 + (uint64_t)((c >> 2) * 128 + (c & 3) * 2), ID);
  } else {
#pragma unroll
    for (int c = T::KH; c < KCI; ++c)
      mma_i8<1>(tbase + T::cDsc, tbase + 8 * (c - T::KH), dsc0 + (uint64_t)((c >> 2) * 128 + (c & 3) * 2), ID);
    if (KCO) {
      constexpr int h0 = L::NHI * 128, a0 = 8 * (KCI - T::KH);
      mma_i8<0>(tbase + T::cDsc + 16, tbase + a0, dsc0 + (uint64_t)h0, ID);
#pragma unroll
      for (int c = 1; c < KCO; ++c)
        mma_i8<1>(tbase + T::cDsc + 16, tbase + a0 + 8 * c, dsc0 + (uint64_t)(h0 + (c >> 2) * 128 + (c & 3) * 2), ID);
    }
  }
}
// logits (log2 domain) of the NQ heads from the score accumulators (kvcache.py:311-329)
// (split in two: the accumulator read-back is issued, the caller waits (tcgen05.wait::ld),
// then the arithmetic)
template <int KCO, int NQ, int CDSC>
__device__ __forceinline__ void score_acc_load(uint32_t tlane, uint32_t* dr) {
  if (NQ == 4) {
    tmem_ld16(tlane + CDSC, dr);
    if (KCO) tmem_ld16(tlane + CDSC + 16, dr + 16);
  } else if (NQ == 2) {
    tmem_ld8(tlane + CDSC, dr);
    if (KCO) tmem_ld8(tlane + CDSC + 16, dr + 16);
  } else {
    tmem_ld4(tlane + CDSC, dr);
    if (KCO) tmem_ld4(tlane + CDSC + 16, dr + 16);
  }
}
template <int KCO, int NQ>
__device__ __forceinline__ void score_logits_of(const uint32_t* dr, const float4* qcs, float nin, float nout,
                                                float* lg) {
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
    lg[q] = l2;
  }
}
template <int KCO, int NQ, int CDSC>
__device__ __forceinline__ void score_logits(uint32_t tlane, const float4* qcs, float nin, float nout, float* lg) {
  uint32_t dr[32];
  score_acc_load<KCO, NQ, CDSC>(tlane, dr);
  tmem_wait_ld();
  score_logits_of<KCO, NQ>(dr, qcs, nin, nout, lg);
}

// ----------------------------------------------------------------- main kernel
// NQ: query heads the epilogue processes (1, 2 or 4 >= G): MHA (G = 1) skips the work of
// three padding heads
template <int KCI, int KCO, int NQ>
__global__ void __launch_bounds__(kThreads, (KCI + KCO > 12) ? 3 : 4) k_udecode(const Params P) {
  using L = Layout<KCI, KCO>;
  using TM = DecTmem<KCI, KCO>;
  constexpr int KC = KCI + KCO;
  extern __shared__ uint8_t sm_raw[];
  // align to 1024 B (SWIZZLE_128B atoms) by pointer arithmetic on the shared array, so the
  // compiler keeps shared-window loads (LDS) instead of generic ones
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  const uint32_t s_sm = smem_u32(sm);
  const uint32_t a_full = s_sm + L::oBar;                      // [kStages]
  const uint32_t a_sc = a_full + 8 * kStages, a_pv = a_sc + 8, a_bsc = a_sc + 16, a_ard = a_sc + 24,
                 a_prd = a_sc + 32, a_sk = a_sc + 40;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::oTmem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = P.ctas;
  const int64_t T = P.total_tiles;
  // contiguous ranges of the flattened (unit, tile) space; deterministic: of whole segments
  auto seg_tile = [&](int64_t g) -> int64_t {          // first flattened tile of segment g
    const int64_t u = g / P.spu, j = g - u * P.spu;
    const int64_t t = j * P.seg;
    return u * P.tpu + (t < P.tpu ? t : P.tpu);
  };
  int64_t r0, r1;
  if (P.seg) {
    const int64_t Sg = (int64_t)P.units * P.spu;
    r0 = seg_tile(tile_begin(blockIdx.x, Sg, C));
    r1 = seg_tile(tile_begin(blockIdx.x + 1, Sg, C));
  } else {
    r0 = tile_begin(blockIdx.x, T, C);
    r1 = tile_begin(blockIdx.x + 1, T, C);
  }
  const int ntiles = (int)(r1 - r0);
  const int u_first = (int)(r0 / P.tpu), lt_first = (int)(r0 - (int64_t)u_first * P.tpu);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(a_full + 8 * s, 1);
    mbar_init(a_sc, 1);
    mbar_init(a_pv, 1);
    mbar_init(a_bsc, 1);
    mbar_init(a_ard, 4);
    mbar_init(a_prd, 4);
    mbar_init(a_sk, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) reinterpret_cast<float*>(sm + L::oMax)[tid] = 0.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TM::kAlloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint64_t dsc0 = desc_sw128(s_sm + L::oBsc);
  const uint64_t dpv0 = desc_none(s_sm + L::oBpv, 128, 2048);
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);   // this warp's TMEM lanes

  // ---- record stream: thread 0 issues one bulk copy per tile, kStages ahead
  int iss_i = 0, iss_s = 0, iss_lt = lt_first;
  const uint8_t* iss_p = P.rec + ((int64_t)u_first * P.cap_tiles + lt_first) * P.rec_bytes;
  int64_t iss_unit = (int64_t)u_first * P.cap_tiles * P.rec_bytes;
  const uint64_t pol = evict_first_policy();
  auto issue_next = [&]() {
    const uint32_t fb = a_full + 8 * iss_s;
    mbar_expect_tx(fb, L::kRec);
    bulk_g2s_hint(s_sm + L::oStage + iss_s * L::kRec, iss_p, L::kRec, fb, pol);
    ++iss_i;
    if (++iss_s == kStages) iss_s = 0;
    if (++iss_lt == P.tpu) {
      iss_lt = 0;
      iss_unit += P.cap_tiles * P.rec_bytes;
      iss_p = P.rec + iss_unit;
    } else {
      iss_p += P.rec_bytes;
    }
  };
  // The first record copies are issued before the grid-dependency wait: the only PDL
  // predecessor is k_uprep, which triggers its dependents only after its own wait on the
  // stream (unless the caller vouched for the inputs with QJL_DECODE_CHAINED) and after its
  // decode-step append is written and fenced -- so every cache row this kernel reads is
  // complete before it starts.  Only the B images and constants wait for the prep.
  if (tid == 0)
    for (int i = 0; i < kStages && i < ntiles; ++i) issue_next();

  // per-thread running state: token-side partials (l, Z), dim-side output (acc); the
  // running max of head (lane & 7) lives in lane-parallel form (m_lane)
  float m_lane = -INFINITY, l_part[4], acc[4], invK[4];
  float2 Z[4][2];                      // [q][group pair]
  const float4* qcs = reinterpret_cast<const float4*>(sm + L::oQc);
  uint32_t sc_ph = 0, pv_ph = 0, bsc_par = 0, rd_ph = 0, sk_ph = 0;
  bool pv_pend = false;
  // the thread's code-chunk offsets within its dim quad's 128-byte row (p2t_byte swizzle)
  const uint32_t c_row = L::oCodes + (tid >> 2) * 128, c_sw = ((tid >> 2) & 3) << 4;

  // PV accumulators of the previous tile -> fp32 running output (thread = dim)
  auto pv_readback = [&]() {
    mbar_wait(a_pv, pv_ph);
    pv_ph ^= 1;
    tc_fence_after();
    uint32_t dd[4][4];                                    // [head q][lo, mid, hi, exponent byte]
#pragma unroll
    for (int q = 0; q < NQ; ++q) tmem_ld4(tlane + 32 + 16 * q + 4 * warp, dd[q]);   // value group = warp
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float f = fmaf((float)(int)dd[q][2], 65536.f, (float)((int)dd[q][0] + 256 * (int)dd[q][1]));
      acc[q] = fmaf(f, invK[q], acc[q]);
    }
  };

  auto load_unit = [&](int u) {
    // the unit's estimator constants -> smem; the first reader is behind the tile's first
    // CTA barrier (and the previous unit's last reader is behind flush's barriers)
    if (tid < 4) reinterpret_cast<float4*>(sm + L::oQc)[tid] = P.qconst[(int64_t)u * 4 + tid];
    // the unit's score B image: one bulk copy; only the MMA issuer waits for it
    if (tid == 0) {
      mbar_expect_tx(a_bsc, L::NH * 2048);
      bulk_g2s(s_sm + L::oBsc, P.bsc + (size_t)u * L::NH * 2048, L::NH * 2048, a_bsc);
    }
  };
  auto reset_state = [&]() {
    m_lane = -INFINITY;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      l_part[q] = 0.f;
      acc[q] = 0.f;
      Z[q][0] = Z[q][1] = make_float2(0.f, 0.f);
    }
  };

  auto flush = [&](int u, int slot, int ns) {
    if (pv_pend) {
      pv_readback();
      pv_pend = false;
    }
    const float wrow = 1.f / (float)(1 << (2 * (tid & 3)));   // code weight 4^(d % 4) of this dim
    // token-side partials -> CTA sums, transposed through smem (the Bsc/Bpv region is
    // free: the last PV MMA completed above): every thread stores its values, then warp
    // w reduces values w, w + 4, ... (4 tokens per lane, then one warp sum)
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
    float* tr = reinterpret_cast<float*>(sm + L::oRed);            // [20][128]
    float* red = tr + 20 * kThreads;                               // [20] CTA sums
    bar_sync(1, kThreads);                // everyone is done with Bsc/Bpv
#pragma unroll
    for (int i = 0; i < 20; ++i)
      if (i < NQ || (i >= 4 && (i - 4) / 4 < NQ)) tr[i * kThreads + tid] = v[i];
    bar_sync(1, kThreads);
#pragma unroll
    for (int i0 = 0; i0 < 20; i0 += 4) {
      const int i = i0 + warp;
      if (i < NQ || (i >= 4 && (i - 4) / 4 < NQ)) {
        const float* t = tr + i * kThreads + lane;
        const float x = warp_sum((t[0] + t[32]) + (t[64] + t[96]));
        if (lane == 0) red[i] = x;
      }
    }
    bar_sync(1, kThreads);
    // the running maxima of the heads, from their lanes
    float mrun[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) mrun[q] = __shfl_sync(0xffffffffu, m_lane, q);
    float* mypart = P.part + ((int64_t)u * P.max_seg + slot) * P.G * kRecF;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (q < P.G) {
        const float lq = red[q];
        const float zq = red[4 + 4 * q + warp];                      // value group of dim tid
        if (tid == 0) {
          mypart[q * kRecF + 0] = mrun[q];
          mypart[q * kRecF + 1] = lq;
        }
        mypart[q * kRecF + 2 + tid] = fmaf(acc[q], wrow, zq);
      }
    }
    int* flag = reinterpret_cast<int*>(sm + L::oFlag);
    if (ns > 1) {
      // publish: the CTA's partial writes are ordered before the counter increment by
      // one cumulative fence after the barrier (not one fence per thread)
      bar_sync(1, kThreads);
      if (tid == 0) {
        __threadfence();
        const int last = atomicAdd(&P.counters[u], 1) == ns - 1;
        if (last) P.counters[u] = 0;             // self-cleaning for the next decode
        *flag = last;
      }
      bar_sync(1, kThreads);
      if (!*flag) {
        bar_sync(1, kThreads);                 // (matches the merge's closing barrier)
        return;
      }
      __threadfence();
    } else {
      bar_sync(1, kThreads);
    }
    // last CTA of the unit: merge the ns partials.  (1) warp q turns the segments' (m, l)
    // into normalized weights w_s = 2^(m_s - M) / L in smem; (2) every thread sums its
    // (q, dim) outputs over the segments with all loads of a chunk in flight.
    const float* up = P.part + (int64_t)u * P.max_seg * P.G * kRecF;
    float* wgt = reinterpret_cast<float*>(sm + L::oRed);          // [ns][4] (Bsc/Bpv are free)
    if (warp < P.G) {
      const int qq = warp;
      float M = -INFINITY;
      for (int s0 = lane; s0 < ns; s0 += 32) M = fmaxf(M, __ldcg(up + (s0 * P.G + qq) * kRecF));
      M = redux_max(M);
      float Ls = 0.f;
      for (int s0 = lane; s0 < ns; s0 += 32) {
        const float* W = up + (s0 * P.G + qq) * kRecF;
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
    bar_sync(1, kThreads);
    {
      const int dim = tid;                                         // 128 threads = 128 dims
      float o[4] = {0.f, 0.f, 0.f, 0.f};
      for (int s0 = 0; s0 < ns; s0 += 8) {
        float av[4][8];
#pragma unroll
        for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            av[qq][k] = (qq < P.G && s0 + k < ns) ? __ldcg(up + ((s0 + k) * P.G + qq) * kRecF + 2 + dim) : 0.f;
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
    bar_sync(1, kThreads);                   // the scratch is free for the next unit's B image
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
#if QJL_UD_TRACE
  long long st_issue = 0, st_wait = 0, st_tiles = 0;
#endif
  const int n32 = (int)P.n;                            // n <= capacity < 2^30 (supported())
  int u = u_first, lt = lt_first, s = 0;
  uint32_t full_ph = 0;
  int it = 0;
  bool first = true;                                      // the MMA issuer waits for the B image
  while (it < ntiles) {
    // this piece: to the end of the unit (stream-K) or of the fixed segment (deterministic)
    const int piece_end_lt = P.seg ? min((lt / P.seg + 1) * P.seg, P.tpu) : P.tpu;
    const int seg_end = min(ntiles, it + (piece_end_lt - lt));
    int slot, ns;
    if (P.seg) {
      slot = lt / P.seg;
      ns = P.spu;
    } else {
      const int c0 = cta_of_tile((int64_t)u * P.tpu, T, C);
      const int c1 = cta_of_tile((int64_t)u * P.tpu + P.tpu - 1, T, C);
      ns = c1 - c0 + 1;
      slot = blockIdx.x - c0;
    }
    load_unit(u);             // (again after a segment flush: the flush scratch aliases the B image)
    first = true;
    reset_state();
    for (; it < seg_end; ++it, ++lt) {
#if QJL_UD_TRACE
      {
        const long long cw0 = clock64();
        mbar_wait(a_full + 8 * s, full_ph);
        st_wait += clock64() - cw0;
        ++st_tiles;
      }
#else
      mbar_wait(a_full + 8 * s, full_ph);
#endif
      const uint8_t* st = sm + L::oStage + s * L::kRec;
      auto body = [&](auto mask_tag) {
        constexpr bool MASK = decltype(mask_tag)::value;
        const bool valid = !MASK || lt * kTile + tid < n32;            // this thread's token is < n

        // ---------------- 1. score A operand: masked sign words -> TMEM ----------------
        if constexpr (TM::SK) {
          // split K (m_in = 512): first half of the in-side words, its MMAs, then the rest
          {
            uint32_t wv[TM::KH];
            load_sign_range<KCI, KCO, 0, TM::KH>(st, tid, wv);
            if (pv_pend) pv_readback();               // the PV MMA of the previous tile (aliases A_sc)
            store_sign_operand<TM::KH>(tlane, wv);
          }
          tmem_wait_st();
          tc_fence_before();
          bar_sync(1, kThreads);
          if (warp == 0) {
            if (elect_one()) {
              if (first) {
                mbar_wait(a_bsc, bsc_par);
                bsc_par ^= 1;
              }
              tc_fence_after();
              issue_score_mma_half<KCI, KCO, 0>(tbase, dsc0);
              tc_commit(a_sk);
            }
            __syncwarp();
          }
          {
            uint32_t wv[KC - TM::KH];
            load_sign_range<KCI, KCO, TM::KH, KC>(st, tid, wv);
            mbar_wait(a_sk, sk_ph);                   // the first half's A columns are free
            sk_ph ^= 1;
            tc_fence_after();
            store_sign_operand<KC - TM::KH>(tlane, wv);
          }
        } else {
          uint32_t wv[KC];
          load_sign_words<KCI, KCO>(st, tid, wv);
          if (pv_pend) pv_readback();                 // the PV MMA of the previous tile (aliases A_sc)
          store_sign_operand<KC>(tlane, wv);
        }
        tmem_wait_st();
        tc_fence_before();
        if constexpr (kSplit) {
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a_ard) : "memory");
        } else {
          bar_sync(1, kThreads);
        }
        if (warp == 0) {
          if (elect_one()) {
            if (kSplit) mbar_wait(a_ard, rd_ph);
            if (first && !TM::SK) {
              mbar_wait(a_bsc, bsc_par);
              bsc_par ^= 1;
            }
            tc_fence_after();
            if constexpr (TM::SK) issue_score_mma_half<KCI, KCO, 1>(tbase, dsc0);
            else issue_score_mma<KCI, KCO>(tbase, dsc0);
            tc_commit(a_sc);
          }
          __syncwarp();
        }

        // token-side inputs that do not depend on the MMA
        const float nin = __half2float(reinterpret_cast<const __half*>(st + L::oNormIn)[tid]);
        const float nout = KCO ? __half2float(reinterpret_cast<const __half*>(st + L::oNormOut)[tid]) : 0.f;
        uint2 zr = reinterpret_cast<const uint2*>(st + L::oZero)[tid];
        uint2 sr = reinterpret_cast<const uint2*>(st + L::oScale)[tid];
        if (MASK && !valid) zr = sr = make_uint2(0u, 0u);      // rows past n (stale padding)

        // ---------------- 3. logits, warp maxima ----------------
        mbar_wait(a_sc, sc_ph);
        sc_ph ^= 1;
        tc_fence_after();
        float lg[4];
        score_logits<KCO, NQ, TM::cDsc>(tlane, qcs, nin, nout, lg);
        if (MASK && !valid) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) lg[q] = -INFINITY;
        }
        if (P.logits != nullptr && valid) {          // optional: the logits the softmax consumes
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (q < P.G) __stcs(P.logits + ((int64_t)u * P.G + q) * P.n + (int64_t)lt * kTile + tid, lg[q] * kLn2);
        }
        {
          float* mx = reinterpret_cast<float*>(sm + L::oMax);
          const float2 hf = h2f2(hmax2u(sr.x, sr.y));
          const float smax_w = redux_max(fmaxf(hf.x, hf.y));
          float tm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int q = 0; q < NQ; ++q) tm[q] = redux_max(lg[q]);
          if (lane == 0) {                        // slot-major: slot q's 4 warp maxima are one float4
#pragma unroll
            for (int q = 0; q < NQ; ++q) mx[4 * q + warp] = tm[q];
            mx[16 + warp] = smax_w;
          }
        }
        // A_pv row of dim tid (the score MMA is done, its A columns are free): 32 columns of
        // 4 tokens, value c * 4^(tid % 4)
        {
          const uint32_t mk = 0x03030303u << (2 * (tid & 3));
          const uint8_t* crow = st + c_row;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t cw[16];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              // chunk 4h + k sits at position (4h + k) ^ (dq % 4) = 4h + (k ^ (dq % 4))
              const uint4 x = *reinterpret_cast<const uint4*>(crow + ((k << 4) ^ c_sw) + 64 * h);
              cw[4 * k] = x.x & mk; cw[4 * k + 1] = x.y & mk; cw[4 * k + 2] = x.z & mk; cw[4 * k + 3] = x.w & mk;
            }
            tmem_st16(tlane + 16 * h, cw);
          }
        }
        bar_sync(1, kThreads);                  // maxima visible; the stage is fully read
#if QJL_UD_TRACE
        if (tid == 0 && iss_i < ntiles) {
          const long long c0 = clock64();
          issue_next();
          st_issue += clock64() - c0;
        }
#else
        if (tid == 0 && iss_i < ntiles) issue_next();   // refill this stage kStages ahead
#endif

        // ---------------- 4. softmax bookkeeping, lane-parallel over the heads ----------------
        // lane l reduces slot (l & 7) over the 4 warps: heads 0..3, the scale bound at 4
        const float4 m4 = reinterpret_cast<const float4*>(sm + L::oMax)[lane & 7];
        const float mv = fmaxf(fmaxf(m4.x, m4.y), fmaxf(m4.z, m4.w));
        const float smax = __shfl_sync(0xffffffffu, mv, 4);
        // p = 2^(lg - m_new) = pt * et with pt = 2^(lg - tmax) <= 1 and the tile-uniform
        // et = 2^(tmax - m_new); P' K = pt * scale * kPMax / smax <= kPMax, and the PV sums
        // come back scaled by invK = et * smax / kPMax
        const float m_new = fmaxf(m_lane, mv);            // finite: every tile has a valid token
        const float alpha_l = ex2(m_lane - m_new);
        const float et_l = ex2(mv - m_new);
        m_lane = m_new;
        const bool moved = __any_sync(0xffffffffu, (lane & 7) < NQ && alpha_l != 1.f);   // CTA-uniform
        const float ksm = smax > 0.f ? kPMax * rcp_approx(smax) : 0.f;
        const float invk_l = et_l * smax * (1.f / kPMax);
        float p[4], pk[4];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float tmax = __shfl_sync(0xffffffffu, mv, q);
          const float et = __shfl_sync(0xffffffffu, et_l, q);
          const float pt = ex2(lg[q] - tmax);
          p[q] = pt * et;
          pk[q] = pt * ksm;
          invK[q] = __shfl_sync(0xffffffffu, invk_l, q);
        }
        if (moved) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const float a = __shfl_sync(0xffffffffu, alpha_l, q);
            const float2 a2 = make_float2(a, a), z2 = make_float2(0.f, 0.f);
            l_part[q] *= a;
            acc[q] *= a;
            Z[q][0] = fma2(Z[q][0], a2, z2);
            Z[q][1] = fma2(Z[q][1], a2, z2);
          }
        }
        // ---------------- 5. P' digits (B of the PV MMA), zero-point sums ----------------
        const float2 z01 = h2f2(zr.x), z23 = h2f2(zr.y);
        const float2 s01 = h2f2(sr.x), s23 = h2f2(sr.y);
        {
          const float2 mg = make_float2(kMagic, kMagic);
          uint4* bpv = reinterpret_cast<uint4*>(sm + L::oBpv) + tid;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            l_part[q] += p[q];
            const float2 pp = make_float2(p[q], p[q]);
            Z[q][0] = fma2(pp, z01, Z[q][0]);
            Z[q][1] = fma2(pp, z23, Z[q][1]);
            const float2 pk2 = make_float2(pk[q], pk[q]);
            const float2 w01 = fma2(pk2, s01, mg), w23 = fma2(pk2, s23, mg);
            // column n = 16 q + 4 G + digit: the fma leaves v(q, G) = rint(P' K) < 2^23 in the
            // mantissa, so the float's bytes ARE the unsigned digits {lo, mid, hi} of the u8 B
            // operand; byte 3 (the exponent, 0x4B) feeds a column nobody reads
            bpv[128 * q] = make_uint4(__float_as_uint(w01.x), __float_as_uint(w01.y), __float_as_uint(w23.x),
                                      __float_as_uint(w23.y));
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // B_pv -> tensor core
        tmem_wait_st();
        tc_fence_before();
        if constexpr (kSplit) {
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a_prd) : "memory");
        } else {
          bar_sync(1, kThreads);
        }

        // ---------------- 6. PV MMA (read back at the next tile) ----------------
        if (warp == 0) {
          if (elect_one()) {
            if (kSplit) mbar_wait(a_prd, rd_ph);
            tc_fence_after();
            constexpr uint32_t ID = idesc_i8(16 * NQ, 1, 0);        // N = (head, group, digit), B u8
            mma_i8<0>(tbase + 32, tbase, dpv0, ID);
            mma_i8<1>(tbase + 32, tbase + 8, dpv0 + 32, ID);       // + 512 B per 32 tokens
            mma_i8<1>(tbase + 32, tbase + 16, dpv0 + 64, ID);
            mma_i8<1>(tbase + 32, tbase + 24, dpv0 + 96, ID);
            tc_commit(a_pv);
          }
          __syncwarp();
        }
        pv_pend = true;
        rd_ph ^= 1;
      };
      if ((lt + 1) * kTile <= n32) body(std::false_type{});
      else body(std::true_type{});
      first = false;
      if (++s == kStages) {
        s = 0;
        full_ph ^= 1;
      }
    }
    if (it == ntiles) {
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // all tiles consumed
#if QJL_UD_TRACE
      if (tid == 0) g_ud_trace[blockIdx.x][1] = gtimer();
#endif
    }
    flush(u, slot, ns);
    if (lt == P.tpu) {
      ++u;
      lt = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
#if QJL_UD_TRACE
  if (tid == 0) {
    g_ud_stat[blockIdx.x][0] = st_tiles;
    g_ud_stat[blockIdx.x][1] = st_issue;
    g_ud_stat[blockIdx.x][2] = st_wait;
    g_ud_stat[blockIdx.x][3] = 1;
  }
  if (tid == 0) g_ud_trace[blockIdx.x][2] = gtimer();
#endif
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(TM::kAlloc));
}

// ------------------------------------------------------------ scores-only K2
#ifndef QJL_US_EARLY_TRIGGER
#define QJL_US_EARLY_TRIGGER 1
#endif
// The score stage of the decode with logits written out (kvcache.py:311-329 ->
// estimate_logits): stages hold the key fields of each record (one bulk copy), the
// score accumulators become logits (natural-log units) stored coalesced per head.
template <int KCI, int KCO, int NQ>
__global__ void __launch_bounds__(kThreads, 4) k_uscores(const Params P) {
  using L = Layout<KCI, KCO>;
  using TM = DecTmem<KCI, KCO>;                 // m_in = 512: split-K score MMA, 128 TMEM columns
  constexpr int KC = KCI + KCO;
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  const uint32_t s_sm = smem_u32(sm);
  const uint32_t a_full = s_sm + L::sBar;
  const uint32_t a_sc = a_full + 8 * kStages, a_bsc = a_sc + 8, a_sk = a_sc + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::sTmem);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t T = P.total_tiles;
  const int64_t r0 = tile_begin(blockIdx.x, T, P.ctas), r1 = tile_begin(blockIdx.x + 1, T, P.ctas);
  const int ntiles = (int)(r1 - r0);
  const int u_first = (int)(r0 / P.tpu), lt_first = (int)(r0 - (int64_t)u_first * P.tpu);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(a_full + 8 * s, 1);
    mbar_init(a_sc, 1);
    mbar_init(a_bsc, 1);
    mbar_init(a_sk, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TM::kAlloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint64_t dsc0 = desc_sw128(s_sm);
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);

  int iss_i = 0, iss_s = 0, iss_lt = lt_first;
  const uint8_t* iss_p = P.rec + ((int64_t)u_first * P.cap_tiles + lt_first) * P.rec_bytes;
  int64_t iss_unit = (int64_t)u_first * P.cap_tiles * P.rec_bytes;
  const uint64_t pol = evict_first_policy();
  auto issue_next = [&]() {
    const uint32_t fb = a_full + 8 * iss_s;
    mbar_expect_tx(fb, L::kKeyRec);
    bulk_g2s_hint(s_sm + L::sStage + iss_s * L::kKeyRec, iss_p, L::kKeyRec, fb, pol);
    ++iss_i;
    if (++iss_s == kStages) iss_s = 0;
    if (++iss_lt == P.tpu) {
      iss_lt = 0;
      iss_unit += P.cap_tiles * P.rec_bytes;
      iss_p = P.rec + iss_unit;
    } else {
      iss_p += P.rec_bytes;
    }
  };
  if (tid == 0)                                        // (early copies: see k_udecode)
    for (int i = 0; i < kStages && i < ntiles; ++i) issue_next();
  asm volatile("griddepcontrol.wait;" ::: "memory");   // Bsc / qconst come from k_uprep
#if QJL_US_EARLY_TRIGGER
  // the next step's query sketch may launch now: it takes the SMs this grid's CTAs leave,
  // and (chained) computes while this grid drains; its workspace writes wait for our exit
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  const float4* qcs = reinterpret_cast<const float4*>(sm + L::sQc);
  const int64_t n = P.n;
  uint32_t sc_ph = 0, bsc_par = 0, full_ph = 0, sk_ph = 0;
  int u = u_first, lt = lt_first, s = 0, it = 0;
  while (it < ntiles) {
    const int seg_end = min(ntiles, it + (P.tpu - lt));
    bar_sync(1, kThreads);                      // the previous unit's MMAs / constants are done
    if (tid < 4) reinterpret_cast<float4*>(sm + L::sQc)[tid] = P.qconst[(int64_t)u * 4 + tid];
    if (tid == 0) {
      mbar_expect_tx(a_bsc, L::NH * 2048);
      bulk_g2s(s_sm, P.bsc + (size_t)u * L::NH * 2048, L::NH * 2048, a_bsc);
    }
    float* const lbase = P.logits + (int64_t)u * P.G * n + tid;      // this unit's rows, this token
    if constexpr (!TM::SK) {
      // Software-pipelined over the unit's tiles: tile i+1's sign words are loaded while
      // MMA(i) runs, stored as the next A operand once MMA(i) is done (same columns), and
      // MMA(i+1) is issued before tile i's logits are computed and stored.
      float nin, nout;
      {
        mbar_wait(a_full + 8 * s, full_ph);
        const uint8_t* st = sm + L::sStage + s * L::kKeyRec;
        uint32_t wv[KC];
        load_sign_words<KCI, KCO>(st, tid, wv);
        store_sign_operand<KC>(tlane, wv);
        nin = __half2float(reinterpret_cast<const __half*>(st + L::oNormIn)[tid]);
        nout = KCO ? __half2float(reinterpret_cast<const __half*>(st + L::oNormOut)[tid]) : 0.f;
        tmem_wait_st();
        tc_fence_before();
        bar_sync(1, kThreads);                  // A operand in TMEM; the stage is fully read
        if (tid == 0 && iss_i < ntiles) issue_next();
        if (warp == 0) {
          if (elect_one()) {
            mbar_wait(a_bsc, bsc_par);
            tc_fence_after();
            issue_score_mma<KCI, KCO>(tbase, dsc0);
            tc_commit(a_sc);
          }
          __syncwarp();
        }
        bsc_par ^= 1;
        if (++s == kStages) {
          s = 0;
          full_ph ^= 1;
        }
      }
      for (; it < seg_end; ++it, ++lt) {
        const bool nxt = it + 1 < seg_end;
        uint32_t wv[KC];
        float nin_n = 0.f, nout_n = 0.f;
        if (nxt) {
          mbar_wait(a_full + 8 * s, full_ph);
          const uint8_t* st = sm + L::sStage + s * L::kKeyRec;
          load_sign_words<KCI, KCO>(st, tid, wv);
          nin_n = __half2float(reinterpret_cast<const __half*>(st + L::oNormIn)[tid]);
          nout_n = KCO ? __half2float(reinterpret_cast<const __half*>(st + L::oNormOut)[tid]) : 0.f;
        }
        mbar_wait(a_sc, sc_ph);
        sc_ph ^= 1;
        tc_fence_after();
        uint32_t dr[32];
        score_acc_load<KCO, NQ, TM::cDsc>(tlane, dr);
        if (nxt) store_sign_operand<KC>(tlane, wv);
        tmem_wait_ld();
        tmem_wait_st();
        tc_fence_before();
        bar_sync(1, kThreads);                  // D(i) read by all; A(i+1) stored; its stage read
        if (nxt) {
          if (tid == 0 && iss_i < ntiles) issue_next();
          if (warp == 0) {
            if (elect_one()) {
              tc_fence_after();
              issue_score_mma<KCI, KCO>(tbase, dsc0);
              tc_commit(a_sc);
            }
            __syncwarp();
          }
          if (++s == kStages) {
            s = 0;
            full_ph ^= 1;
          }
        }
        float lg[4];
        score_logits_of<KCO, NQ>(dr, qcs, nin, nout, lg);
        if (lt * kTile + tid < n) {
          float* lp = lbase + lt * kTile;
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (q < P.G) __stcs(lp + q * n, lg[q] * kLn2);
        }
        nin = nin_n;
        nout = nout_n;
      }
      tc_fence_before();
    } else {
      // split-K (m_in = 512): the same pipeline with the two K halves of each tile's MMA --
      // the second half's A columns overlap the first half's, so they wait for it
      float nin, nout;
      auto stage_in = [&](const uint8_t* st, bool first_tile) {
        uint32_t wv[KC - TM::KH];
        load_sign_range<KCI, KCO, TM::KH, KC>(st, tid, wv);
        mbar_wait(a_sk, sk_ph);                 // the first half's A columns are free
        sk_ph ^= 1;
        tc_fence_after();
        store_sign_operand<KC - TM::KH>(tlane, wv);
        tmem_wait_st();
        tc_fence_before();
        bar_sync(1, kThreads);                  // A (second half) in TMEM; the stage is fully read
        if (tid == 0 && iss_i < ntiles) issue_next();
        if (warp == 0) {
          if (elect_one()) {
            tc_fence_after();
            issue_score_mma_half<KCI, KCO, 1>(tbase, dsc0);
            tc_commit(a_sc);
          }
          __syncwarp();
        }
        if (++s == kStages) {
          s = 0;
          full_ph ^= 1;
        }
      };
      {
        mbar_wait(a_full + 8 * s, full_ph);
        const uint8_t* st = sm + L::sStage + s * L::kKeyRec;
        {
          uint32_t wv[TM::KH];
          load_sign_range<KCI, KCO, 0, TM::KH>(st, tid, wv);
          store_sign_operand<TM::KH>(tlane, wv);
        }
        nin = __half2float(reinterpret_cast<const __half*>(st + L::oNormIn)[tid]);
        nout = KCO ? __half2float(reinterpret_cast<const __half*>(st + L::oNormOut)[tid]) : 0.f;
        tmem_wait_st();
        tc_fence_before();
        bar_sync(1, kThreads);
        if (warp == 0) {
          if (elect_one()) {
            mbar_wait(a_bsc, bsc_par);
            tc_fence_after();
            issue_score_mma_half<KCI, KCO, 0>(tbase, dsc0);
            tc_commit(a_sk);
          }
          __syncwarp();
        }
        bsc_par ^= 1;
        stage_in(st, true);
      }
      for (; it < seg_end; ++it, ++lt) {
        const bool nxt = it + 1 < seg_end;
        uint32_t wv[TM::KH];
        float nin_n = 0.f, nout_n = 0.f;
        const uint8_t* st = sm + L::sStage + s * L::kKeyRec;
        if (nxt) {
          mbar_wait(a_full + 8 * s, full_ph);
          load_sign_range<KCI, KCO, 0, TM::KH>(st, tid, wv);
          nin_n = __half2float(reinterpret_cast<const __half*>(st + L::oNormIn)[tid]);
          nout_n = KCO ? __half2float(reinterpret_cast<const __half*>(st + L::oNormOut)[tid]) : 0.f;
        }
        mbar_wait(a_sc, sc_ph);
        sc_ph ^= 1;
        tc_fence_after();
        uint32_t dr[32];
        score_acc_load<KCO, NQ, TM::cDsc>(tlane, dr);
        if (nxt) store_sign_operand<TM::KH>(tlane, wv);
        tmem_wait_ld();
        tmem_wait_st();
        tc_fence_before();
        bar_sync(1, kThreads);                  // D(i) read by all; A(i+1) first half stored
        if (nxt) {
          if (warp == 0) {
            if (elect_one()) {
              tc_fence_after();
              issue_score_mma_half<KCI, KCO, 0>(tbase, dsc0);
              tc_commit(a_sk);
            }
            __syncwarp();
          }
          stage_in(st, false);
        }
        float lg[4];
        score_logits_of<KCO, NQ>(dr, qcs, nin, nout, lg);
        if (lt * kTile + tid < n) {
          float* lp = lbase + lt * kTile;
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (q < P.G) __stcs(lp + q * n, lg[q] * kLn2);
        }
        nin = nin_n;
        nout = nout_n;
      }
      tc_fence_before();
    }
    ++u;
    lt = 0;
  }
#if !QJL_US_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(TM::kAlloc));
}

// ------------------------------------------------------------------- host side
struct Plan {
  int tpu;
  int ctas;
  int max_seg;
  int seg, spu;
  int64_t T;
  size_t bsc_off, qconst_off, part_off, cnt_off, total;
};

// resident CTAs per SM, from the register file, shared memory and the 512 TMEM columns
// (the runtime's occupancy calculator cannot see the TMEM footprint of tcgen05 kernels)
template <typename K>
static int resident_ctas(K kern, int smem_bytes, int tmem_cols) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  int dev = 0, smem_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
  const int by_regs = 65536 / (regs_warp * (kThreads / 32));
  const int by_smem = smem_sm / (smem_bytes + 1024);
  int o = by_regs < by_smem ? by_regs : by_smem;
  const int tmem_cap = 512 / tmem_cols;
  return o < 1 ? 1 : (o > tmem_cap ? tmem_cap : o);
}

template <int KCI, int KCO, int NQ>
static int occupancy_dec() {
  static int occ = -1;
  if (occ < 0) occ = resident_ctas(k_udecode<KCI, KCO, NQ>, Layout<KCI, KCO>::kTotal, DecTmem<KCI, KCO>::kAlloc);
  return occ;
}
template <int KCI, int KCO, int NQ>
static int occupancy_sc() {
  static int occ = -1;
  if (occ < 0) occ = resident_ctas(k_uscores<KCI, KCO, NQ>, Layout<KCI, KCO>::sTotal, DecTmem<KCI, KCO>::kAlloc);
  return occ;
}

static bool kc_dispatch(int kci, int kco, int* id) {
  const int pairs[][2] = {{8, 2}, {8, 4}, {8, 0}, {16, 2}, {16, 0}, {16, 4}};
  for (int i = 0; i < 6; ++i)
    if (pairs[i][0] == kci && pairs[i][1] == kco) {
      *id = i;
      return true;
    }
  return false;
}
static int nq_of(int G) { return G <= 1 ? 1 : G <= 2 ? 2 : 4; }
static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

template <int KCI, int KCO>
static int occupancy_any(int G, bool scores) {
  switch (nq_of(G)) {
    case 1: return scores ? occupancy_sc<KCI, KCO, 1>() : occupancy_dec<KCI, KCO, 1>();
    case 2: return scores ? occupancy_sc<KCI, KCO, 2>() : occupancy_dec<KCI, KCO, 2>();
    default: return scores ? occupancy_sc<KCI, KCO, 4>() : occupancy_dec<KCI, KCO, 4>();
  }
}
static int occupancy_by_id(int id, int G, bool scores) {
  switch (id) {
    case 0: return occupancy_any<8, 2>(G, scores);
    case 1: return occupancy_any<8, 4>(G, scores);
    case 2: return occupancy_any<8, 0>(G, scores);
    case 3: return occupancy_any<16, 2>(G, scores);
    case 4: return occupancy_any<16, 0>(G, scores);
    case 5: return occupancy_any<16, 4>(G, scores);
  }
  return 1;
}
static int nh_by_id(int id) {
  const int nh[] = {3, 3, 2, 5, 4, 5};
  return nh[id];
}

constexpr int kDetSeg = 4;          // deterministic schedule: 512-token segments

static Plan make_plan(const qjl_key_cache_t& kc, int64_t n, int G, int id, bool scores, bool det = false) {
  Plan p;
  p.tpu = (int)((n + kTile - 1) / kTile);
  p.T = (int64_t)kc.units * p.tpu;
  const int64_t slots = (int64_t)device_sm_count() * occupancy_by_id(id, G, scores);
  p.seg = det && !scores ? kDetSeg : 0;
  p.spu = p.seg ? (p.tpu + p.seg - 1) / p.seg : 1;
  const int64_t work = p.seg ? (int64_t)kc.units * p.spu : p.T;
  p.ctas = (int)(work < slots ? work : slots);
  // few units (small batch): at most max(32, tiles per unit / 8) CTAs per unit -- a unit's
  // last CTA merges one partial per CTA in dependent L2 rounds, which beyond ~32 partials
  // costs more than the extra CTAs gain unless each still gets >= 8 tiles (measured: C5
  // B1 x 32k 28.4 -> 21.7 us; B1 x 128k keeps its 74 CTAs per unit)
  if (!p.seg) {
    const int64_t nsmax = p.tpu / 8 > 32 ? p.tpu / 8 : 32;
    if ((int64_t)kc.units * nsmax < p.ctas) p.ctas = (int)((int64_t)kc.units * nsmax);
  }
  int ms = 1;
  if (p.seg) {
    ms = p.spu;
  } else {
    for (int u = 0; u < kc.units; ++u) {
      const int ns = cta_of_tile((int64_t)u * p.tpu + p.tpu - 1, p.T, p.ctas) -
                     cta_of_tile((int64_t)u * p.tpu, p.T, p.ctas) + 1;
      ms = ms > ns ? ms : ns;
    }
  }
  p.max_seg = ms;
  p.bsc_off = 0;
  p.qconst_off = align256((size_t)kc.units * nh_by_id(id) * 2048);
  p.part_off = p.qconst_off + align256((size_t)kc.units * 4 * 16);
  p.cnt_off = p.part_off + (scores ? 0 : align256((size_t)kc.units * p.max_seg * G * kRecF * 4));
  p.total = p.cnt_off + align256((size_t)kc.units * 4);
  return p;
}

}  // namespace ud

// The tile-major fast path: P2T values in the same records as the keys, d = 128, G <= 4,
// (m_in/32, m_out/32) in the instantiated set.  vc == nullptr (scores): the key fields of
// either record variant (keys only, or keys + values) -- they sit at the same offsets.
static bool record_matches(const qjl_key_cache_t& kc, const qjl_value_cache_t* vc) {
  const TileRecord r = tile_record(kc.d, kc.m_in, kc.m_out, vc != nullptr);
  const bool stride_ok = vc ? kc.tile_stride == r.bytes
                            : (kc.tile_stride == r.bytes || kc.tile_stride == tile_record(kc.d, kc.m_in, kc.m_out, true).bytes);
  if (!stride_ok || kc.capacity % 128 != 0) return false;
  const uint8_t* base = kc.bits_in;
  if (kc.m_out && (kc.bits_out != base + r.off[QJL_REC_BITS_OUT] ||
                   (const uint8_t*)kc.norm_out != base + r.off[QJL_REC_NORM_OUT]))
    return false;
  if ((const uint8_t*)kc.norm_in != base + r.off[QJL_REC_NORM_IN]) return false;
  if (vc) {
    if (vc->tile_stride != r.bytes || vc->capacity != kc.capacity) return false;
    if ((const uint8_t*)vc->codes != base + r.off[QJL_REC_CODES] ||
        (const uint8_t*)vc->zero != base + r.off[QJL_REC_ZERO] || (const uint8_t*)vc->scale != base + r.off[QJL_REC_SCALE])
      return false;
  }
  return true;
}

bool tile_path_supported(const qjl_key_cache_t& kc, const qjl_value_cache_t* vc, int G) {
  int id;
  if (vc && !(vc->layout == QJL_VLAYOUT_P2T && vc->d == 128 && vc->bits == 2 && vc->group == 32)) return false;
  return kc.d == 128 && G >= 1 && G <= 4 && ud::kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id) && kc.m_in % 32 == 0 &&
         kc.m_out % 32 == 0 && kc.capacity < (int64_t(1) << 30) && record_matches(kc, vc);
}

size_t decode_tile_workspace(const qjl_key_cache_t& kc, int64_t n, int G, bool scores) {
  int id;
  if (!ud::kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id)) return 0;
  const size_t a = ud::make_plan(kc, n, G, id, scores).total;
  const size_t b = scores ? 0 : ud::make_plan(kc, n, G, id, false, true).total;   // either schedule
  return a > b ? a : b;
}

namespace ud {

struct Launch {
  const qjl_key_cache_t* kc;
  int64_t n;
  const void* q;
  int q_dtype;
  int G;
  const qjl_sketch_t* sk;
  float inv_t;
  float* out;
  float* lse;
  float* logits;
  void* ws;
  unsigned flags;
  const Append* app;
  int mode;              // 0 decode, 1 scores, 2 benchmark: prep + `reps` chained decodes
  int reps;
  float* ms;
};

template <int KCI, int KCO, int NQ>
static cudaError_t launch_main(const cudaLaunchConfig_t& cfg, const Params& P, int mode) {
  if (mode == 1) return cudaLaunchKernelEx(&cfg, k_uscores<KCI, KCO, NQ>, P);
  return cudaLaunchKernelEx(&cfg, k_udecode<KCI, KCO, NQ>, P);
}

template <int KCI, int KCO>
static int launch_impl(const Launch& a, const Plan& plan, cudaStream_t st) {
  const qjl_key_cache_t& kc = *a.kc;
  const qjl_sketch_t& sk = *a.sk;
  uint8_t* w = (uint8_t*)a.ws;
  uint8_t* bsc = w + plan.bsc_off;
  float4* qconst = (float4*)(w + plan.qconst_off);
  float* part = (float*)(w + plan.part_off);
  int* counters = (int*)(w + plan.cnt_off);
  constexpr int MT = (KCI + KCO) * 32;
  const int chained = (a.flags & QJL_DECODE_CHAINED) ? 1 : 0;
  cudaLaunchAttribute pattr[1];
  pattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pattr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t pcfg = {};
  pcfg.gridDim = dim3(kc.units);
  pcfg.blockDim = dim3(MT);                      // x threads per row, set per sketch dtype below
  pcfg.stream = st;
  pcfg.attrs = pattr;
  pcfg.numAttrs = 1;
  const Append none{};
  const Append& app = a.app ? *a.app : none;
  cudaError_t pe = cudaErrorInvalidValue;
#define QJL_UPREP(TQ, TS)                                                                                     \
  pe = app.k ? cudaLaunchKernelEx(&pcfg, k_uprep<TQ, TS, KCI, KCO, true>, (const TQ*)a.q, a.G,                 \
                                  (const TS*)sk.s_full, sk.unit_stride, a.inv_t, chained, bsc, qconst, counters, \
                                  app)                                                                        \
             : cudaLaunchKernelEx(&pcfg, k_uprep<TQ, TS, KCI, KCO, false>, (const TQ*)a.q, a.G,                \
                                  (const TS*)sk.s_full, sk.unit_stride, a.inv_t, chained, bsc, qconst, counters, \
                                  app)
#define QJL_UPREP_S(TQ)                                 \
  switch (sk.dtype) {                                   \
    case QJL_BF16: QJL_UPREP(TQ, __nv_bfloat16); break; \
    case QJL_F16: QJL_UPREP(TQ, __half); break;         \
    case QJL_F32: QJL_UPREP(TQ, float); break;          \
    default: QJL_UPREP(TQ, double); break;              \
  }
  switch (a.q_dtype) {
    case QJL_BF16: QJL_UPREP_S(__nv_bfloat16); break;
    case QJL_F16: QJL_UPREP_S(__half); break;
    case QJL_F32: QJL_UPREP_S(float); break;
    default: QJL_UPREP_S(double); break;
  }
#undef QJL_UPREP_S
#undef QJL_UPREP
  if (pe != cudaSuccess) return cuda_status(pe, "decode_prep");
  QJL_LAUNCH_CHECK("decode_prep");
  Params P;
  P.rec = kc.bits_in;
  P.rec_bytes = kc.tile_stride;
  P.cap_tiles = kc.capacity / kTile;
  P.n = a.n;
  P.G = a.G;
  P.units = kc.units;
  P.tpu = plan.tpu;
  P.total_tiles = plan.T;
  P.ctas = plan.ctas;
  P.max_seg = plan.max_seg;
  // with an append the prep writes a row the decode streams: the decode's early copies
  // rely on the prep's fence-then-trigger order, which holds only for chained launches
  P.chained = chained;
  P.seg = plan.seg;
  P.spu = plan.spu;
  P.bsc = bsc;
  P.qconst = qconst;
  P.part = part;
  P.counters = counters;
  P.out = a.out;
  P.lse = a.lse;
  P.logits = a.logits;
  const int mode = a.mode == 1 ? 1 : 0;
  using L = Layout<KCI, KCO>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = mode == 1 ? L::sTotal : L::kTotal;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  occupancy_any<KCI, KCO>(a.G, mode == 1);   // shared-memory attributes
  auto launch = [&]() -> cudaError_t {
    switch (nq_of(a.G)) {
      case 1: return launch_main<KCI, KCO, 1>(cfg, P, mode);
      case 2: return launch_main<KCI, KCO, 2>(cfg, P, mode);
      default: return launch_main<KCI, KCO, 4>(cfg, P, mode);
    }
  };
  cudaError_t e = launch();
  if (e != cudaSuccess) return cuda_status(e, mode == 1 ? "scores_tc" : "decode_tc");
  if (a.mode == 2) {
    // benchmark: reps more decode kernels chained on the first (each re-reads the cache;
    // the merging CTAs reset the unit counters), bracketed by events
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    P.chained = 1;
    e = launch();                       // untimed: the chain's first kernel follows the prep
    cudaEventRecord(e0, st);
    for (int r = 0; r < a.reps && e == cudaSuccess; ++r) e = launch();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (a.ms) *a.ms = a.reps > 0 ? ms / a.reps : 0.f;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (e != cudaSuccess) return cuda_status(e, "decode_tc (bench)");
  }
  QJL_LAUNCH_CHECK("decode_tc");
  return QJL_OK;
}

static int launch_any(const Launch& a, size_t ws_bytes, cudaStream_t st) {
  const qjl_key_cache_t& kc = *a.kc;
  int id;
  if (!kc_dispatch(kc.m_in / 32, kc.m_out / 32, &id)) return QJL_ERR_UNSUPPORTED;
  const Plan plan = make_plan(kc, a.n, a.G, id, a.mode == 1, (a.flags & QJL_DECODE_DETERMINISTIC) != 0);
  if (ws_bytes < plan.total) {
    set_error("decode workspace needs %zu bytes", plan.total);
    return QJL_ERR_WORKSPACE;
  }
  switch (id) {
    case 0: return launch_impl<8, 2>(a, plan, st);
    case 1: return launch_impl<8, 4>(a, plan, st);
    case 2: return launch_impl<8, 0>(a, plan, st);
    case 3: return launch_impl<16, 2>(a, plan, st);
    case 4: return launch_impl<16, 0>(a, plan, st);
    case 5: return launch_impl<16, 4>(a, plan, st);
  }
  return QJL_ERR_UNSUPPORTED;
}

}  // namespace ud

int launch_decode_tile(const qjl_key_cache_t& kc, int64_t n, const void* q, int q_dtype, int G,
                       const qjl_sketch_t& sk, float inv_t, float* out, float* lse, float* logits, void* ws,
                       size_t ws_bytes, unsigned flags, cudaStream_t st) {
  ud::Launch a{&kc, n, q, q_dtype, G, &sk, inv_t, out, lse, logits, ws, flags, nullptr, 0, 0, nullptr};
  return ud::launch_any(a, ws_bytes, st);
}

int launch_decode_step_tile(const qjl_key_cache_t& kc, const qjl_value_cache_t& vc, int64_t n, const void* q,
                            int q_dtype, int G, const qjl_sketch_t& sk, const int32_t* channels, int h,
                            const void* k_new, const void* v_new, float inv_t, float* out, float* lse,
                            float* logits, void* ws, size_t ws_bytes, unsigned flags, cudaStream_t st) {
  ud::Append app{};
  app.k = k_new;
  app.v = v_new;
  app.kc = kc;
  app.vc = vc;
  app.channels = channels;
  app.h = h;
  app.row = n;                                   // the new token's row; decode over n + 1
  ud::Launch a{&kc, n + 1, q, q_dtype, G, &sk, inv_t, out, lse, logits, ws, flags, &app, 0, 0, nullptr};
  return ud::launch_any(a, ws_bytes, st);
}

int launch_scores_tile(const qjl_key_cache_t& kc, int64_t n, const void* q, int q_dtype, int G,
                       const qjl_sketch_t& sk, float* logits, void* ws, size_t ws_bytes, unsigned flags,
                       cudaStream_t st) {
  ud::Launch a{&kc, n, q, q_dtype, G, &sk, 1.f, nullptr, nullptr, logits, ws, flags, nullptr, 1, 0, nullptr};
  return ud::launch_any(a, ws_bytes, st);
}

int bench_decode_tile(const qjl_key_cache_t& kc, int64_t n, const void* q, int q_dtype, int G, const qjl_sketch_t& sk,
                      float inv_t, float* out, float* lse, void* ws, size_t ws_bytes, unsigned flags, int reps,
                      float* ms, cudaStream_t st) {
  ud::Launch a{&kc, n, q, q_dtype, G, &sk, inv_t, out, lse, nullptr, ws, flags, nullptr, 2, reps, ms};
  return ud::launch_any(a, ws_bytes, st);
}

}  // namespace qjl

#if QJL_UD_TRACE
extern "C" __attribute__((visibility("default"))) int qjl_debug_ud_trace(void* host, int ctas) {
  return (int)cudaMemcpyFromSymbol(host, qjl::ud::g_ud_trace, sizeof(unsigned long long) * 4 * ctas);
}
extern "C" __attribute__((visibility("default"))) int qjl_debug_ud_stat(void* host, int ctas) {
  return (int)cudaMemcpyFromSymbol(host, qjl::ud::g_ud_stat, sizeof(unsigned long long) * 4 * ctas);
}
#endif
