// fwd_tc.cu -- Rolling Update forward (prefill) on sm_100a tensor cores.
//
// The paper's Rolling Update (Alg. 1) fuses the attention
// reduction chain of Fig. 8 into ONE loop over KV tiles; the
// tile-level loop body is Fig. 19: local max, global max,
// repair term h(t, r, r') = exp(r - r') t (Fig. 18d) applied to
// the running sum and to the PV accumulator (Eq. 7), local exp
// sum, PV, then m_old <- m_new (Alg. 1 CacheReducePrevResult);
// O / l after the loop (Fig. 9 reverse_compute_at(norm)).
//
// B200 mapping:
//   D = 128: CTA = 2 query tiles of BM = 128 rows of one (b, hq) -> 256 rows; 384 threads.
//     warps 0-3   : softmax/correction/epilogue for query tile 0 (thread = row)
//     warps 4-7   : same for query tile 1
//     warp 8      : TMA producer (Q once; K_j / V_j through a 3-slot ring of 128-key tiles)
//     warps 9-11  : tcgen05.mma issuers (warp-wide, one elected lane issues), rotating by KV
//                   step (kGridIssuers); warp 10 also allocates TMEM (512 columns)
//     The producer and MMA warps get the HIGHEST warp ids on purpose: the warp
//     arbiter is highest-id-first, so they are never starved by the softmax warps.
//     TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512) (fp32 columns).
//     P_t (bf16/fp16) goes to shared memory in the UMMA K-major layout: S_t is free as soon as
//     its softmax threads hold it in registers, so the issue order per KV step j is PV0(j),
//     QK0(j+2), PV1(j), QK1(j+2) and S_t(j+1) is computed while the softmax of step j runs; K
//     runs two tiles ahead of V in the ring.  (P aliasing S in TMEM with a TS MMA serialises
//     softmax -> PV -> QK per tile: measured 3 % (r1, with the exp token) to 10 % (r2) slower.)
//     Pure-causal problems run the persistent variant (fwd_tc_persist_kernel) of this layout; it
//     runs the MMA issuer on hardware warp 1 (the lowest id of its sub-partition) and the tile-0
//     quarter-1 softmax warp on warp 9 (role_warp_persist).
//   D = 64: CTA = ONE 128-row query tile, 64-key KV tiles, 192 threads (4 softmax warps, TMA
//     producer, MMA issuer + TMEM allocator), TMEM S [0,64) (P aliasing it) + O [64,128): four
//     CTAs per SM.  Producer and issuer alternate between the two extra warps by block parity,
//     and the issuer trades ids with its sub-partition's softmax warp so it holds the lowest id.
//   MMA issue: whole K loops as one batched asm block with one elect.sync (ptx.cuh mma_*_x4/x8)
//     in every kernel (only the ALiBi extra K = 16 step is a single MMA).
//   Repair is lazy (reading R9): the reference max r' only moves when the
//   running max exceeds it by more than kTau (log2 units); exact because h
//   tag-updates to any reference (Eq. 6).
#include <math.h>

#include <algorithm>

#include "kernels.h"
#include "ptx.cuh"

namespace attn {
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int kTileThreads = 128;                       // softmax threads per query tile (thread = row)
constexpr int kSoftmaxWarps = 2 * kTileThreads / 32;    // (the NT = 2 layout of the persistent kernel)
constexpr int kWarpLoad = kSoftmaxWarps, kWarpMma = kSoftmaxWarps + 1, kWarpAlloc = kSoftmaxWarps + 2;
constexpr int kThreads = (kSoftmaxWarps + 3) * 32;
constexpr float kTau = 8.0f;                      // lazy-repair threshold (log2 units), reading R9
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLog2e = 1.4426950408889634f;
constexpr uint32_t kBarP0 = 5;                    // 5 / 6: "P_t ready" (softmax threads of tile t + MMA warp)
constexpr uint32_t kBarS0 = 9;                    // 9 / 10: "S_t loaded into registers" (P in smem only)
// Causal block order: heaviest-first over a group of (head, batch) slices whose K/V fit in
// this much of the 126 MB L2 (see the block order in fwd_tc_kernel).
constexpr long long kCausalL2Bytes = 96LL << 20;
#ifdef ATTN_TRACE
constexpr bool kTraceBuild = true;    // the timeline trace instruments the non-persistent kernel
#else
constexpr bool kTraceBuild = false;
#endif

// D = 128 grid kernel: the MMA issue rotates over three warps (9, 10, 11 -> SM sub-partitions
// 1, 2, 3) by KV step.  A warp blocked in tcgen05.mma issue slows the softmax warps of its own
// sub-partition (the TMEM lane quarter there ran ~550 cycles/step behind, profiles/
// r2_mma_issue_study.md); rotating spreads that over three quarters.  Same-box A/B (r2): MHA
// +1.4 %, GQA window +0.6 %, ALiBi +1.0 %, ALiBi-causal +0.5 % (two issuers: +1.7 / +0.9 / +0.2 /
// -0.8 %).  Every tcgen05.commit still covers only its own issuer's MMAs, which is all each
// barrier needs (a step's K / V slots, S_t and O_t are produced within one step).
constexpr int kGridIssuers = 3;
#define WAIT_SM(bar, par) mbar_wait(bar, par)        // softmax waits: try_wait (HW sleep; test_wait polling: equal / -2.5 % at D = 64)
#define WAIT_LM(bar, par) mbar_wait_spin(bar, par)   // loader / MMA thread waits: poll (try_wait: equal)

#ifdef ATTN_TRACE
// Debug-only timeline of one CTA: clock() per (event, step), kept in shared
// memory while the kernel runs (so tracing adds no global-memory traffic
// before the mbarrier releases) and copied to g_trace at the end.
// 32-bit clock() samples (the host unwraps differences modulo 2^32).
constexpr int kTrEv = 32, kTrSteps = 16;
__device__ long long g_trace[kTrEv][kTrSteps];
// per-CTA lifetime (trace builds, tools/cta_log.py): entry / exit globaltimer, SM id, clock64 cycles
constexpr int kCtaLog = 8192;
__device__ unsigned long long g_cta[kCtaLog][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool trace_cta() { return blockIdx.x == 5 && blockIdx.y == 3 && blockIdx.z == 2; }
#define TRACE(ev, step)                                                          \
  do {                                                                           \
    if (trace_cta() && (step) < kTrSteps) s_trace[(ev) * kTrSteps + (step)] = (uint32_t)clock(); \
  } while (0)
#else
#define TRACE(ev, step) do { } while (0)
#endif

// Shipped configuration per head dim (the measured alternatives are listed there):
//   D = 128: NT = 2 query tiles per CTA (one CTA per SM, the two tiles' exponentials overlap),
//            P in shared memory (PV = SS MMA, S released early), 3-slot K/V ring of 128-key
//            tiles, packed f32x2 exponent FMA / row sum, chunk-classified masks.
//   D = 64 : NT = 1 (four 128-row CTAs per SM), 64-key tiles, P aliasing S in TMEM (PV = TS
//            MMA), 4-slot ring.
// Both: 2 of every 16 exponential pairs on the FMA pipe (ex2_poly2) except with ALiBi.
// ALiBi (without softcap) is folded into the QK contraction at both head dims (kExt).
template <int D>
__host__ __device__ constexpr int nt_of() { return D == 128 ? 2 : 1; }
// KV tile width: D = 64 uses 64-key tiles so that a CTA needs 128 TMEM columns (S 64 + O 64) and
// FOUR 128-row CTAs (16 softmax warps) share an SM: the D = 64 kernel is bound by the latency of
// each CTA's softmax <-> tensor-core chain, not by MUFU throughput, so more independent CTAs per
// SM is what raises the exponential rate.  Same-box A/B (r2, vs 128-key tiles with 2 CTAs/SM):
// scaled-dot +12 %, causal +18 %, softcap-causal +14 %, ALiBi-causal +12 %, ALiBi +11 %.
template <int D>
__host__ __device__ constexpr int bn_of() { return D == 64 ? 64 : 128; }
template <int D, bool kAlibi>
__host__ __device__ constexpr bool alibi_mma() { return kAlibi && !(D == 128 && kTraceBuild); }   // (trace: no smem left)

template <int D, bool kExt = false, int NT = 2>
struct Cfg {
  static constexpr int kBoxes = D / 64;           // 64-column (128 B) swizzle atoms per row
  static constexpr int kQTileBytes = BM * D * 2;
  static constexpr int BNk = bn_of<D>();
  static constexpr int kKVTileBytes = BNk * D * 2;
  // P in shared memory at D = 128 (else in TMEM, aliasing S: at D = 64 P in shared memory with a
  // 3-slot ring measured equal, r2)
  static constexpr bool kPS = D == 128;
  static constexpr int kPTileBytes = kPS ? BM * BNk * 2 : 0;
  static constexpr int kStages = D == 128 ? 3 : 4;   // D = 64: 4 x 8 KiB slots (4 CTAs per SM)
  // Load-group barriers (ring).  The producer can be at most kStages/2 groups
  // ahead of the issuer's wait, so kStages/2 + 1 barriers never alias a phase.
  static constexpr int kPairBars = kStages / 2 + 1;
  // ALiBi-in-contraction operands, after the K/V ring, no swizzle: A_ext(+-s) 2 x 256 B (two
  // K core matrices, all 128 rows aliased by SBO = 0) and B_ext 2 KB (16 row groups; its K 8..15
  // half aliases K 0..7 by LBO = 0 and meets zeros in A).  (The D = 128 two-tile CTA has 3 KB left.)
  static constexpr int kExt2Bytes = kExt ? 2 * 256 + 2048 : 0;
  static constexpr int kSmemQ = NT * kQTileBytes + NT * kPTileBytes;   // Q, P tiles
  static constexpr int kSmemKV = kStages * kKVTileBytes;
  static constexpr int kNumBars = 1 + 2 * kStages + 6;
#ifdef ATTN_TRACE
  static constexpr int kSmemBytes = kSmemQ + kSmemKV + kExt2Bytes + 256 + kTrEv * kTrSteps * 4;
#else
  static constexpr int kSmemBytes = kSmemQ + kSmemKV + kExt2Bytes + kNumBars * 8 + 16;
#endif
};

struct Range {
  int lo, hi;                      // active KV tiles [lo, hi)
  int jlo_first, jhi_first;        // allowed key interval of the first row
  int jlo_last, jhi_last;          // ... and of the last valid row
};

// Allowed local key interval [jlo, jhi] of a query at absolute position qp
// (mask definition in include/attn.h), clamped to [0, Skv - 1].
__device__ __forceinline__ void row_bounds(const Shape& s, const VariantParams& v, long long qp, int& jlo,
                                           int& jhi) {
  long long lo = 0, hi = s.Skv - 1;
  if (v.window_left >= 0) lo = max(lo, qp - v.window_left - v.kv_off);
  const long long kInf = 0x3fffffffffffffffLL;
  long long h = kInf;
  if (v.causal) h = qp;
  if (v.window_right >= 0) h = min(h, qp + (long long)v.window_right);
  if (h != kInf) hi = min(hi, h - v.kv_off);
  jlo = (int)min(lo, (long long)s.Skv);
  jhi = (int)max(hi, -1LL);
}

template <int BNt = BN>
__device__ __forceinline__ Range tile_range(const Shape& s, const VariantParams& v, int i0) {
  Range r{0, 0, 0, -1, 0, -1};
  if (i0 >= s.Sq) return r;
  const int il = min(i0 + BM, s.Sq) - 1;
  row_bounds(s, v, v.q_off + i0, r.jlo_first, r.jhi_first);
  row_bounds(s, v, v.q_off + il, r.jlo_last, r.jhi_last);
  if (r.jlo_first <= r.jhi_last) {
    r.lo = r.jlo_first / BNt;
    r.hi = r.jhi_last / BNt + 1;
  }
  return r;
}

__device__ __forceinline__ bool active(const Range& r, int j) { return j >= r.lo && j < r.hi; }

// MUFU offload: pair e (of the 16 pairs of a 32-column chunk) takes the FMA-pipe exp2
// (ex2_poly2) for kPolyPairs evenly spread pairs, MUFU ex2.approx for the rest.  Same-box A/B
// (r2, pairs of 16 on the polynomial): persistent causal D = 128 2/16 +4 %, 4/16 +1 %, 6/16 -4 %
// (vs none); D = 64 (4 CTAs/SM) 2/16: scaled-dot +3 %, softcap +4 %; grid kernel D = 128 2/16
// +1 % (MHA), 4/16 -1 … -2 %,
// 6/16 -8 % (the MUFU is not the binding unit there: the exp phase is paced by synchronisation,
// DESIGN.md §4.1); ALiBi kernels keep MUFU only (2/16 -2 %, 4/16 -4 … -8 %).
// (r2, 4 CTAs/SM at D = 64: ALiBi 2/16 +0.4 … +0.9 % vs MUFU only; softcap 4/16 +1.4 %, the
// others 4/16 -3 … -4 %, 1/16 -2 … -4 %.)
constexpr int kPolyGrid128 = 2, kPolyGrid64 = 2, kPolyGrid64Cap = 4, kPolyPersist = 2;   // (D = 128 ALiBi: 0)
template <int kPolyPairs>
__device__ __forceinline__ constexpr bool poly_pair(int e) {
  return kPolyPairs > 0 && ((e * kPolyPairs) % 16) + kPolyPairs >= 16;
}
template <int kPolyPairs>
__device__ __forceinline__ void exp2_pair(float a0, float a1, float& p0, float& p1, int e) {
  if (poly_pair<kPolyPairs>(e)) {
    ex2_poly2(a0, a1, p0, p1);
  } else {
    p0 = ex2_approx(a0);
    p1 = ex2_approx(a1);
  }
}

// ALiBi-in-MMA class of (query tile starting at row i0, KV tile j): +1 if every key is at or
// before every query of the tile (bias = -slope (qpos - kpos) = slope*c + a row constant:
// A_ext(+s)), -1 if every key is at or after every query (A_ext(-s)), 0 mixed (A_ext(+s) and
// a per-element fix-up).  The issuer and the softmax threads classify identically.
template <int BNt = BN>
__device__ __forceinline__ int ext_class(const Shape& s, const VariantParams& v, int i0, int j) {
  // Causal: every ALLOWED key of any tile is at or before its query, so the linear form holds
  // for the allowed elements of a diagonal tile too (the rest are masked to -inf).
  if (v.causal) return 1;
  const long long qf = v.q_off + i0, ql = v.q_off + min(i0 + BM, s.Sq) - 1;
  const long long k0 = v.kv_off + (long long)j * BNt, k1 = k0 + BNt - 1;
  if (k1 <= qf) return 1;
  if (k0 >= ql) return -1;
  return 0;
}

__device__ __forceinline__ float u2f(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// Max-pass over one S row held in registers, in chunks of 32 columns: `xf(xv, c)` applies
// score_mod; on mask tiles each chunk is classified warp-uniformly (all 32 rows of the warp
// see it wholly allowed / wholly masked / partial) so only partial chunks pay the per-element
// compare-and-select (on a causal diagonal tile that is one chunk in four per warp).
// (kChunked = false: every element of a mask tile is compared; measured better at D = 64,
// where the chunk branches cost registers in the MUFU-bound kernels.)
template <bool kMask, bool kChunked, int N, class XF>
__device__ __forceinline__ float row_max_pass(float (&x)[N], int rel_lo, int rel_hi, XF xf) {
  constexpr int kCh = 4;
  float mx[kCh];   // independent chains for ILP
#pragma unroll
  for (int q = 0; q < kCh; ++q) mx[q] = -INFINITY;
  if constexpr (!kChunked) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      float xv = xf(x[c], c);
      if constexpr (kMask) xv = (c >= rel_lo && c <= rel_hi) ? xv : -INFINITY;
      x[c] = xv;
      mx[c % kCh] = fmaxf(mx[c % kCh], xv);
    }
  } else {
#pragma unroll
  for (int q = 0; q < N / 32; ++q) {
    bool part = false;   // some row of the warp has a masked column in this chunk
    if constexpr (kMask) part = !__all_sync(0xffffffffu, rel_lo <= q * 32 && rel_hi >= q * 32 + 31);
    if (!part) {
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int c = q * 32 + e;
        const float xv = xf(x[c], c);
        x[c] = xv;
        mx[c % kCh] = fmaxf(mx[c % kCh], xv);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int c = q * 32 + e;
        const float xv = (c >= rel_lo && c <= rel_hi) ? xf(x[c], c) : -INFINITY;
        x[c] = xv;
        mx[c % kCh] = fmaxf(mx[c % kCh], xv);
      }
    }
  }
  }
#pragma unroll
  for (int w = kCh / 2; w > 0; w /= 2)
#pragma unroll
    for (int q = 0; q < w; ++q) mx[q] = fmaxf(mx[q], mx[q + w]);
  return mx[0];
}

// score_mod + mask of one S row (BN raw fp32 dots in `x`), in place, into the
// log2 domain used by the exponentials; returns the row max of the tile.
// Plain variant: x stays raw (scale folded into the exp FFMA) and the max is
// rescaled afterwards (scale > 0 so max commutes with it).
template <bool kAlibi, bool kSoftcap, bool kMask, bool kChunked = true, int N>
__device__ __forceinline__ float score_tile(float (&x)[N], const VariantParams& v, float nslope2, float dq0,
                                            int rel_lo, int rel_hi) {
  float mt = row_max_pass<kMask, kChunked>(x, rel_lo, rel_hi, [&](float xv, int c) {
    if constexpr (kSoftcap) {
      xv = v.softcap_log2 * tanh_approx(xv * v.scale_over_cap);   // R3: cap * tanh(x / cap)
    } else if constexpr (kAlibi) {
      xv = xv * v.scale_log2;
    }
    if constexpr (kAlibi) xv = fmaf(nslope2, fabsf(dq0 - (float)c), xv);  // R4: -slope |qpos - kpos|
    return xv;
  });
  if constexpr (!kAlibi && !kSoftcap) mt *= v.scale_log2;
  return mt;
}

// Mixed ALiBi-in-MMA tile (ext_class 0, built with A_ext(+s)): S = q.k + s c, so
// x = scale S - slope (c + |qpos - kpos|) = scale S - slope max(dq0, 2c - dq0) (log2 units).
template <bool kMask, int N>
__device__ __forceinline__ float score_tile_ext_mixed(float (&x)[N], const VariantParams& v, float nslope2, float dq0,
                                                      int rel_lo, int rel_hi) {
  return row_max_pass<kMask, false>(x, rel_lo, rel_hi, [&](float xv, int c) {
    return fmaf(nslope2, fmaxf(dq0, 2.f * (float)c - dq0), xv * v.scale_log2);
  });
}

// One accumulator's whole K loop as ONE batched issue (ptx.cuh mma_*_x4/x8: a single elect.sync
// for the batch, so the issuing warp keeps the tensor rate and leaves its sub-partition's issue
// slots to the softmax warps).  SW128 K-major A / B: k-step kk starts (kk >> 2) atoms of
// kAtomA / kAtomB bytes and (kk & 3) * 32 bytes into the tile; V (MN-major B of PV) advances
// 2048 bytes (16 keys) per k-step.  Descriptor start addresses are in 16-byte units.
template <int NK>
__device__ __forceinline__ void mma_ss_kloop(uint32_t d, uint64_t da, uint32_t atom_a, uint64_t db, uint32_t atom_b,
                                             bool b_mn16, uint32_t idesc, uint32_t acc) {
  uint64_t a[NK], b[NK];
#pragma unroll
  for (int kk = 0; kk < NK; ++kk) {
    a[kk] = da + (uint64_t)(((kk >> 2) * atom_a + (kk & 3) * 32) >> 4);
    b[kk] = db + (uint64_t)((b_mn16 ? kk * 2048 : (kk >> 2) * atom_b + (kk & 3) * 32) >> 4);
  }
  if constexpr (NK == 8) mma_ss_x8(d, a, b, idesc, acc);
  else mma_ss_x4(d, a, b, idesc, acc);
}
template <int NK>
__device__ __forceinline__ void mma_ts_kloop(uint32_t d, uint32_t ta, uint64_t db, uint32_t idesc, uint32_t acc) {
  uint32_t a[NK];
  uint64_t b[NK];
#pragma unroll
  for (int kk = 0; kk < NK; ++kk) {
    a[kk] = ta + kk * 8;                              // 16 keys of 16-bit P = 8 TMEM columns
    b[kk] = db + (uint64_t)((kk * 2048) >> 4);
  }
  if constexpr (NK == 8) mma_ts_x8(d, a, b, idesc, acc);
  else mma_ts_x4(d, a, b, idesc, acc);
}

// Role id of a hardware warp in the persistent kernel: the MMA issuer (role 9) runs on hardware
// warp 1 and the tile-0 quarter-1 softmax warp on hardware warp 9 -- the same SM sub-partition
// (id % 4), but the issuer now has the lowest arbitration priority there (the warp arbiter is
// highest-id-first).  Same-box A/B (r2): persistent causal +1.3 %; the grid kernel -0.4 % (kept
// as is), issuer on warp 5: grid -1 … -2 %.
__device__ __forceinline__ uint32_t role_warp_persist(uint32_t w) { return w == 9 ? 1 : (w == 1 ? 9 : w); }

template <int NT, int BNt = BN>
struct Roles {   // warp roles of fwd_tc_kernel
  static constexpr int kSoftmaxWarps = NT * kTileThreads / 32;
  static constexpr int kWarpLoad = kSoftmaxWarps, kWarpMma = kSoftmaxWarps + 1;
  static constexpr int kWarpAlloc = NT == 2 ? kSoftmaxWarps + 2 : kWarpMma;   // NT = 1: the MMA warp allocates
  static constexpr int kThreads = (NT == 2 ? kSoftmaxWarps + (kGridIssuers > 2 ? 4 : 3) : kSoftmaxWarps + 2) * 32;
  // NT = 1: 2 CTAs per SM at 128-key tiles (256 TMEM columns each), 4 at 64-key tiles (128 each)
  static constexpr int kMinBlocks = NT == 2 ? 1 : (BNt == 64 ? 4 : 2);
  static constexpr int kTmemCols = NT == 2 ? 512 : (BNt == 64 ? 128 : 256);
  static constexpr uint32_t kOBase = NT == 2 ? 256 : BNt;   // TMEM column of O_0 (S_t at t * 128)
};

template <int D, bool kAlibi, bool kSoftcap, bool kF16, int NT>
__global__ void __launch_bounds__(Roles<NT, bn_of<D>()>::kThreads, Roles<NT, bn_of<D>()>::kMinBlocks)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o, const Shape s,
                  const VariantParams v, float* __restrict__ lse) {
  constexpr bool kExt = alibi_mma<D, kAlibi && !kSoftcap>();   // softcap: the bias follows the tanh
  constexpr bool kChunkMask = D == 128;   // chunk-classified masking (measured: + at D = 128, - at D = 64)
  using C = Cfg<D, kExt, NT>;
  using Ro = Roles<NT, C::BNk>;
  constexpr int BN = C::BNk;   // KV tile width of this kernel (shadows the file constant)
  constexpr int kSoftmaxWarps = Ro::kSoftmaxWarps;
  // NT = 1 (several CTAs per SM): alternate the TMA-producer and MMA-issuer warps between the two
  // extra warp ids by block parity, so co-resident CTAs spread their issuers over SM
  // sub-partitions 0 and 1 (the issuer's sub-partition slows its softmax warps).
  const bool swap_roles = NT == 1 &&
                          ((blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) & 1);
  const int kWarpLoad = swap_roles ? Ro::kWarpMma : Ro::kWarpLoad;
  const int kWarpMma = swap_roles ? Ro::kWarpLoad : Ro::kWarpMma;
  const int kWarpAlloc = NT == 1 ? kWarpMma : Ro::kWarpAlloc;
  constexpr bool kPSmem = C::kPS;
  constexpr bool kF32x2 = D == 128;   // packed FFMA2 / FADD2 (measured: +1.5-2 % at D = 128, -4 % at D = 64)
  // (r1 alternated the two tiles' exp phases through a named-barrier token; r2 same-box A/B
  // without it: MHA +2.2 %, GQA window +1 %)
  constexpr bool kPlain = !kAlibi && !kSoftcap;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // The 128-byte swizzle needs 1024-byte aligned tiles; dynamic shared memory
  // starts at offset 0 of the CTA's window (no static shared memory here).
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem;
  uint8_t* sP = smem + NT * C::kQTileBytes;   // kPSmem: P_t, K-major SW128 [key atom][row][128 B]
  uint8_t* sExt = smem + C::kSmemQ + C::kSmemKV;   // kExt: A_ext(+s), A_ext(-s), B_ext
  uint8_t* sKV = smem + C::kSmemQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::kSmemKV + C::kExt2Bytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;
  uint64_t* p_ready = s_full + 2;
  uint64_t* o_done = p_ready + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
#ifdef ATTN_TRACE
  uint32_t* s_trace = reinterpret_cast<uint32_t*>(smem + C::kSmemQ + C::kSmemKV + C::kExt2Bytes + 256);
  if (trace_cta())
    for (int i = threadIdx.x; i < kTrEv * kTrSteps; i += blockDim.x) s_trace[i] = 0;
#endif

  // NT = 1: the MMA issuer also takes the LOWEST hardware warp id of its sub-partition (it trades
  // ids with the softmax warp there), so the arbiter (highest id first) favours the softmax warp
  // (same-box A/B, r2: scaled-dot +1.4 %, causal +2 %, ALiBi-causal +0.8 %, softcap equal).
  const uint32_t hw_warp = warp_id();
  const uint32_t warp = NT == 1
                            ? (swap_roles ? (hw_warp == 0 ? 4u : hw_warp == 4 ? 0u : hw_warp)
                                          : (hw_warp == 1 ? 5u : hw_warp == 5 ? 1u : hw_warp))
                            : hw_warp;
  const uint32_t lane = lane_id();
#ifdef ATTN_TRACE
  const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (threadIdx.x == 0 && cta_lin < kCtaLog) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_cta[cta_lin][0] = gtimer();
    g_cta[cta_lin][2] = smid;
    g_cta[cta_lin][3] = clock64();
  }
#endif
  // Block order.  Causal: heaviest q-blocks first -- across a GROUP of (head, batch) slices
  // whose K/V fit in kCausalL2Bytes of L2 (longest-processing-time order over the group),
  // not head by head: the hardware dispatches blocks in linear order, so a group's light
  // blocks fill in behind all of its heavy ones.  (A/B vs head by head, 96 MB: D = 64 causal
  // 426 -> 477, ALiBi-causal 389 -> 441, softcap-causal 294 -> 337; D = 128 ALiBi-causal +2 %.)
  int qblk = (int)blockIdx.x, hq = (int)blockIdx.y, zb = (int)blockIdx.z;   // zb: output batch (split * B + b)
  if (v.causal) {
    const int nqb = gridDim.x, nh = gridDim.y * gridDim.z;
    const long long kv_bytes = 4LL * s.Skv * D / (s.Hq / s.Hkv);       // K + V of one q head's group, / G
    const int gh = (int)max(1LL, min((long long)nh, kCausalL2Bytes / max(kv_bytes, 1LL)));
    const int lin = blockIdx.x + nqb * (blockIdx.y + gridDim.y * blockIdx.z);
    const int grp = lin / (nqb * gh), idx = lin - grp * nqb * gh;
    const int ghe = min(gh, nh - grp * gh);                          // heads in this (maybe partial) group
    qblk = nqb - 1 - idx / ghe;
    const int head = grp * gh + idx % ghe;
    hq = head % gridDim.y;
    zb = head / gridDim.y;
  }
  const int b = s.kv_splits > 1 ? zb % s.B : zb;              // input batch index
  const int hkv = hq / (s.Hq / s.Hkv);                       // R6: contiguous GQA groups
  const int row0 = qblk * NT * BM;
  Range rng0 = tile_range<BN>(s, v, row0), rng1 = NT == 2 ? tile_range<BN>(s, v, row0 + BM) : Range{0, 0, 0, -1, 0, -1};
  if (s.kv_splits > 1) {   // this CTA's KV split: a contiguous run of whole tiles
    // (kv_split_tiles counts 128-key tiles, the host's unit)
    const int t_lo = (zb / s.B) * s.kv_split_tiles * (128 / BN), t_hi = t_lo + s.kv_split_tiles * (128 / BN);
    for (Range* r : {&rng0, &rng1}) {
      r->lo = max(r->lo, t_lo);
      r->hi = min(r->hi, t_hi);
      if (r->lo >= r->hi) r->lo = r->hi = 0;
    }
  }
  const bool has_rows1 = NT == 2 && row0 + BM < s.Sq;
  int ulo = 0, uhi = 0;
  if (rng0.hi > rng0.lo && rng1.hi > rng1.lo) {
    ulo = min(rng0.lo, rng1.lo);
    uhi = max(rng0.hi, rng1.hi);
  } else if (rng0.hi > rng0.lo) {
    ulo = rng0.lo; uhi = rng0.hi;
  } else if (rng1.hi > rng1.lo) {
    ulo = rng1.lo; uhi = rng1.hi;
  }
  // KV order.  Rolling Update is exact in any order (Thm. 3-4); with ALiBi and keys only at or
  // before the queries the bias grows toward the diagonal, so the ascending order raises the
  // running max by slope * 128 per tile and repairs O every step.  Those problems walk the KV
  // tiles from the diagonal down (the first tile holds the max): step k visits tile J(k).  The
  // loops below count steps k in [ulo, uhi); rng0/rng1 lo/hi are mapped to step space.
  // Without a mask edge inside [ulo, uhi) (both tiles span it) the walk starts at the CTA's
  // diagonal tile d, goes down to ulo, then up from d + 1: J(k) = d - (k - ulo) for the first
  // d - ulo + 1 steps, else k (the reflection above is the case d = uhi - 1).
  const bool full = (rng0.lo == ulo && rng0.hi == uhi) && (!has_rows1 || (rng1.lo == ulo && rng1.hi == uhi));
  const bool rev = kAlibi && (v.causal || v.window_right == 0);
  int d_walk = ulo - 1;   // identity
  if (rev) {
    d_walk = uhi - 1;
  } else if (kAlibi && full && uhi > ulo) {
    const long long ql = v.q_off + min(row0 + NT * BM, s.Sq) - 1;
    d_walk = (int)max((long long)ulo, min((long long)uhi - 1, (ql - v.kv_off) / BN));
  }
  auto J = [=](int k) {
    if constexpr (kAlibi) return k - ulo <= d_walk - ulo ? d_walk - (k - ulo) : k;
    else return k;
  };
  if (rev)
    for (Range* r : {&rng0, &rng1})
      if (r->hi > r->lo) {
        const int lo = ulo + uhi - r->hi, hi = ulo + uhi - r->lo;
        r->lo = lo;
        r->hi = hi;
      }

  if (warp == kWarpLoad && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    prefetch_tmap(&tm_o);
    mbar_init(q_full, 1);
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&o_done[t], 1);
    }
    fence_mbarrier_init();
  }
  if (warp == kWarpAlloc) tmem_alloc<Ro::kTmemCols>(tmem_slot);
  // ALiBi in the contraction (kExt): is it usable for this head?  (fp16 parts must not overflow.)
  bool ext_on = false;
  if constexpr (kExt) {
    const float sx = v.alibi[hq] / v.scale;
    ext_on = kF16 ? fabsf(sx) < 256.f : fabsf(sx) < 1e30f;
    {
      // B_ext row c = (c, c, c, 0, 0, 0, 0, 0) (c <= 127: exact), A_ext(+-s) rows = (s_hi, s_mid,
      // s_lo, 0, ...) with s = slope / scale split into three 16-bit parts.
      const float hi = round16<kF16>(sx), mid = round16<kF16>(sx - hi), lo = round16<kF16>(sx - hi - mid);
      for (int ti = threadIdx.x; ext_on && ti < BM + 32; ti += blockDim.x) {
        if (ti < BM) {   // B_ext: group c / 8, row c % 8 of its core matrix
          const float c = (float)ti;
          *reinterpret_cast<uint4*>(sExt + 512 + (ti >> 3) * 128 + (ti & 7) * 16) =
              make_uint4(pack2<kF16>(c, c), pack2<kF16>(c, 0.f), 0u, 0u);
        } else {         // A_ext(+-s): core matrix K 0..7 = 8 identical rows, K 8..15 = 0
          const int u = (ti - BM) >> 4, k = (ti - BM) & 15;
          const float sg = u ? -1.f : 1.f;
          *reinterpret_cast<uint4*>(sExt + u * 256 + k * 16) =
              k < 8 ? make_uint4(pack2<kF16>(sg * hi, sg * mid), pack2<kF16>(sg * lo, 0.f), 0u, 0u)
                    : make_uint4(0u, 0u, 0u, 0u);
        }
      }
    }
    fence_proxy_async_smem();   // generic-proxy stores -> tensor core reads
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRACE(3, 0);

  if (warp == kWarpLoad) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();   // K/V are re-read by the other q-blocks of this head
      const int nq = has_rows1 ? 2 : 1;
      mbar_arrive_expect_tx(q_full, nq * C::kQTileBytes);
      for (int t = 0; t < nq; ++t)
        for (int bx = 0; bx < C::kBoxes; ++bx)
          tma_load_4d(&tm_q, q_full, sQ + t * C::kQTileBytes + bx * BM * 128, bx * 64, row0 + t * BM, hq, b, pol_q);
      if constexpr (kPSmem) {
        // One barrier per ring slot; ring order = the issuer's consumption order:
        // K_ulo, K_ulo+1, then (V_j, K_j+2) for every step j.
        int it = 0;
        auto load = [&](bool is_k, int jj) {
          WAIT_LM(&kv_empty[it % C::kStages], ((it / C::kStages) & 1) ^ 1);
          TRACE(24 + (is_k ? 0 : 1), jj);   // slot free: the load is issued now (trace builds)
          uint64_t* bar = &kv_full[it % C::kStages];
          mbar_arrive_expect_tx(bar, C::kKVTileBytes);
          uint8_t* dst = sKV + (it % C::kStages) * C::kKVTileBytes;
          for (int bx = 0; bx < C::kBoxes; ++bx)
            tma_load_4d(is_k ? &tm_k : &tm_v, bar, dst + bx * BN * 128, bx * 64, J(jj) * BN, hkv, b, pol_kv);
          ++it;
        };
        if (uhi > ulo) {
          load(true, ulo);
          if (ulo + 1 < uhi) load(true, ulo + 1);
          for (int j = ulo; j < uhi; ++j) {
            load(false, j);
            if (j + 2 < uhi) load(true, j + 2);
          }
        }
      } else {
      // Load groups: g = 0 is K_ulo; g >= 1 is the pair (V_{ulo+g-1}, K_{ulo+g}) (the last
      // group has no K).  A group signals ONE "pair" barrier (kv_full[g % C::kPairBars]), so
      // the MMA issuer waits once per KV step for both tiles it needs next.
      const int n = uhi - ulo;
      for (int g = 0; g <= n; ++g) {
        const int j = ulo + g;
        const int it0 = g == 0 ? 0 : 2 * g - 1;          // ring index of the group's first tile
        const int it1 = g < n ? 2 * g : 2 * g - 1;       // ... and of its last tile
        for (int it = it0; it <= it1; ++it) WAIT_LM(&kv_empty[it % C::kStages], ((it / C::kStages) & 1) ^ 1);
        uint64_t* bar = &kv_full[g % C::kPairBars];
        mbar_arrive_expect_tx(bar, (it1 - it0 + 1) * C::kKVTileBytes);
        for (int it = it0; it <= it1; ++it) {
          const bool is_k = (it % 2) == 0;              // even ring index: K_{ulo + it/2}; odd: V_{ulo + it/2}
          const int jj = ulo + it / 2;
          TRACE(24 + (is_k ? 0 : 1), jj);
          uint8_t* dst = sKV + (it % C::kStages) * C::kKVTileBytes;
          for (int bx = 0; bx < C::kBoxes; ++bx)
            tma_load_4d(is_k ? &tm_k : &tm_v, bar, dst + bx * BN * 128, bx * 64, J(jj) * BN, hkv, b, pol_kv);
        }
      }
      }
    }
  } else if (warp == kWarpMma || (NT == 2 && kGridIssuers > 1 && warp > kWarpMma &&
                                   warp < kWarpMma + kGridIssuers)) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs this role with warp-uniform values; one elected lane
    // issues each tcgen05 instruction (see mma_*_warp).
    if (uhi > ulo) {
      constexpr uint32_t idesc_qk = idesc_f16_f32(BM, BN, 0, 0, !kF16);  // Q K-major, K K-major
      constexpr uint32_t idesc_pv = idesc_f16_f32(BM, D, 0, 1, !kF16);   // P (TMEM), V MN-major
      const uint32_t tS[2] = {tmem, tmem + 128};
      const uint32_t tO[2] = {tmem + Ro::kOBase, tmem + Ro::kOBase + 128};
      const Range rg[2] = {rng0, rng1};
      WAIT_LM(q_full, 0);

      auto wait_group = [&](int g) {   // load group g (see the producer)
        WAIT_LM(&kv_full[g % C::kPairBars], (g / C::kPairBars) & 1);
        tc_fence_after();
      };
      auto qk = [&](int t, int it, int j) {   // S_t = Q_t K_j^T (+ s*c, ALiBi in the contraction)
        const uint32_t sq = smem_u32(sQ + t * C::kQTileBytes);
        const uint32_t sk = smem_u32(sKV + (it % C::kStages) * C::kKVTileBytes);
        // batched issue (one elect.sync per K loop; with the rotating issuers +1.1 … +1.5 % vs per-MMA
        // issue, which had measured better with a single issuer)
        mma_ss_kloop<D / 16>(tS[t], smem_desc_sw128(sq, 16, 1024), BM * 128, smem_desc_sw128(sk, 16, 1024), BN * 128,
                             false, idesc_qk, 0u);
        if constexpr (kExt) {
          if (ext_on) {
            const int cls = ext_class<BN>(s, v, row0 + t * BM, J(j));
            const uint32_t sa = smem_u32(sExt + (cls < 0 ? 256 : 0));
            mma_ss_warp(tS[t], smem_desc_nosw(sa, 128, 0), smem_desc_nosw(smem_u32(sExt + 512), 0, 128), idesc_qk, 1u);
          }
        }
        mma_commit_warp(&s_full[t]);
      };
      auto pv = [&](int t, int it, bool acc) {   // O_t += P_t V (P straight from TMEM)
        named_bar_sync(kBarP0 + t, kTileThreads + 32);   // the softmax threads of tile t arrived
        tc_fence_after();
        if (lane == 0) TRACE(13 + t, it / 2);
        const uint32_t sv = smem_u32(sKV + (it % C::kStages) * C::kKVTileBytes);
        mma_ts_kloop<BN / 16>(tO[t], tS[t], smem_desc_sw128(sv, BN * 128, 1024), idesc_pv, acc ? 1u : 0u);
        mma_commit_warp(&o_done[t]);
      };

      if constexpr (kPSmem) {
        // Order per step j: PV0(j), QK0(j+2), PV1(j), QK1(j+2).  QK_t(i) overwrites
        // S_t once the tile's softmax threads have loaded S_t(i-1) (barrier kBarS0+t).
        auto wait_tile = [&](int it) {
          WAIT_LM(&kv_full[it % C::kStages], (it / C::kStages) & 1);
          tc_fence_after();
        };
        auto qk_p = [&](int t, int it, int i) {
          if (i > rg[t].lo) {
            named_bar_sync(kBarS0 + t, kTileThreads + 32);
            tc_fence_after();
          }
          qk(t, it, i);
        };
        auto pv_p = [&](int t, int it, bool acc) {   // O_t += P_t V (P from shared memory)
          named_bar_sync(kBarP0 + t, kTileThreads + 32);
          tc_fence_after();
          if (lane == 0) TRACE(13 + t, it / 2);
          const uint32_t sp = smem_u32(sP + t * C::kPTileBytes);
          const uint32_t sv = smem_u32(sKV + (it % C::kStages) * C::kKVTileBytes);
          mma_ss_kloop<BN / 16>(tO[t], smem_desc_sw128(sp, 16, 1024), BM * 128, smem_desc_sw128(sv, BN * 128, 1024), 0,
                                true, idesc_pv, acc ? 1u : 0u);
          mma_commit_warp(&o_done[t]);
        };
        // KV step j is issued by issuer (j - ulo) % kNI, after the previous step's issuer has
        // issued its last MMA (named barrier 12 + next issuer).
        constexpr int kNI = NT == 2 ? kGridIssuers : 1;   // issuer warps (kWarpMma, +1, +2)
        constexpr bool k2I = kNI > 1;
        const int my = (int)warp - kWarpMma;
        int it = 0;
        if (my == 0) {
          wait_tile(it);
          if (active(rg[0], ulo)) qk_p(0, it, ulo);
          if (active(rg[1], ulo)) qk_p(1, it, ulo);
          mma_commit_warp(&kv_empty[it % C::kStages]);
        }
        ++it;
        if (ulo + 1 < uhi) {
          if (my == 0) {
            wait_tile(it);
            if (active(rg[0], ulo + 1)) qk_p(0, it, ulo + 1);
            if (active(rg[1], ulo + 1)) qk_p(1, it, ulo + 1);
            mma_commit_warp(&kv_empty[it % C::kStages]);
          }
          ++it;
        }
        for (int j = ulo; j < uhi; ++j) {
          const int itV = it++;
          const bool k2 = j + 2 < uhi;
          const int itK = k2 ? it++ : 0;
          if (k2I && ((j - ulo) % kNI) != my) continue;
          if (k2I && j > ulo) named_bar_sync(12 + my, 64);   // step j-1 is issued
          wait_tile(itV);
          if (lane == 0) TRACE(12, j);
          if (active(rg[0], j)) pv_p(0, itV, j > rg[0].lo);
          if (lane == 0) TRACE(0, j);
          if (k2) {
            wait_tile(itK);
            if (active(rg[0], j + 2)) qk_p(0, itK, j + 2);
          }
          if (lane == 0) TRACE(1, j);
          if (active(rg[1], j)) pv_p(1, itV, j > rg[1].lo);
          if (lane == 0) TRACE(2, j);
          mma_commit_warp(&kv_empty[itV % C::kStages]);
          if (k2) {
            if (active(rg[1], j + 2)) qk_p(1, itK, j + 2);
            mma_commit_warp(&kv_empty[itK % C::kStages]);
          }
          if (k2I && j + 1 < uhi) named_bar_arrive(12 + ((j + 1 - ulo) % kNI), 64);
        }
      } else {
      wait_group(0);
      if (active(rg[0], ulo)) qk(0, 0, ulo);
      if (active(rg[1], ulo)) qk(1, 0, ulo);
      mma_commit_warp(&kv_empty[0]);
      for (int j = ulo; j < uhi; ++j) {
        const int itV = 2 * (j - ulo) + 1, itK1 = itV + 1;
        const bool more = j + 1 < uhi;
        wait_group(j - ulo + 1);                         // V_j and K_{j+1}
        if (lane == 0) TRACE(12, j);
        if (active(rg[0], j)) pv(0, itV, j > rg[0].lo);
        if (lane == 0) TRACE(0, j);
        if (more && active(rg[0], j + 1)) qk(0, itK1, j + 1);
        if (lane == 0) TRACE(1, j);
        if (active(rg[1], j)) pv(1, itV, j > rg[1].lo);
        if (lane == 0) TRACE(2, j);
        mma_commit_warp(&kv_empty[itV % C::kStages]);
        if (more) {
          if (active(rg[1], j + 1)) qk(1, itK1, j + 1);
          mma_commit_warp(&kv_empty[itK1 % C::kStages]);
        }
      }
      }
    }
  } else if (warp < kSoftmaxWarps) {
    // ------------------------------------------------------------ softmax / correction / epilogue
    // Thread (tile t, row r) owns row r of S_t / O_t (TMEM lane r).
    const int t = (int)warp / (kSoftmaxWarps / NT);
    const int wt = (int)warp % (kSoftmaxWarps / NT);      // warp within the tile
    const int wq = warp & 3;                               // TMEM lane quarter
    const int r = wq * 32 + lane;
    const int tid_t = wt * 32 + lane;                      // thread index within the tile
    const Range R = t == 0 ? rng0 : rng1;
    const int i = row0 + t * BM + r;
    const long long qpos = v.q_off + i;
    int jlo_row, jhi_row;
    row_bounds(s, v, qpos, jlo_row, jhi_row);
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tS = tmem + t * 128 + lane_off;
    const uint32_t tP = tmem + t * 128 + lane_off;         // 16-bit pairs, aliasing S (D = 64)
    const uint32_t tO = tmem + Ro::kOBase + t * 128 + lane_off;
    const float nslope2 = kAlibi ? -v.alibi[hq] * kLog2e : 0.f;
    float m_ref = -INFINITY;  // stale reference max (log2 units), R9
    float l = 0.f;            // running denominator over this thread's columns (un-rounded fp32 p, R10)

    for (int j = ulo; j < uhi; ++j) {
      if (!active(R, j)) continue;
      const int it = j - R.lo;
      if (tid_t == 0) TRACE(4 + 4 * t, j);
      WAIT_SM(&s_full[t], it & 1);
      tc_fence_after();
      if (tid_t == 0) TRACE(5 + 4 * t, j);
      if (t == 0 && tid_t == 32) TRACE(20, j);   // warp quarter 1: S ready
      float x[BN];
      {
        uint32_t u[BN];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS + c * 32, reinterpret_cast<uint32_t(&)[32]>(u[c * 32]));
        tmem_ld_wait();
        if constexpr (kPSmem) {
          if (j + 1 < R.hi) {   // S_t is in registers: the issuer may compute S_t(j+1) into it
            tc_fence_before();
            named_bar_arrive(kBarS0 + t, kTileThreads + 32);
          }
        }
#pragma unroll
        for (int c = 0; c < BN; ++c) x[c] = u2f(u[c]);
      }
      if (tid_t == 0) TRACE(26 + 3 * t, j);   // S in registers
      if (t == 0 && tid_t == 32) TRACE(21, j);
      // Fig. 19 max_local (+ score_mod, mask) -> max_global
      const int jt = J(j);   // the KV tile of step j
      const bool need_mask = !(jt * BN >= R.jlo_last && (jt + 1) * BN - 1 <= R.jhi_first);
      const int rel_lo = jlo_row - jt * BN, rel_hi = jhi_row - jt * BN;
      const float dq0 = (float)(qpos - v.kv_off - (long long)jt * BN);
      // exponent argument a = x * e_mul + e_off' (e_off' = e_off - m, set after the max)
      float e_mul = kPlain ? v.scale_log2 : 1.f, e_off = 0.f;
      float mt;
      if (kExt && ext_on) {
        // ALiBi in the contraction: S already holds q.k + (+-s) c (see ext_class)
        const int cls = ext_class<BN>(s, v, row0 + t * BM, jt);
        if (cls != 0) {   // bias = row constant: the plain path with an offset
          e_mul = v.scale_log2;
          e_off = (cls > 0 ? nslope2 : -nslope2) * dq0;
          mt = (need_mask ? score_tile<false, false, true, kChunkMask>(x, v, nslope2, dq0, rel_lo, rel_hi)
                          : score_tile<false, false, false, kChunkMask>(x, v, nslope2, dq0, rel_lo, rel_hi)) + e_off;
        } else {
          mt = need_mask ? score_tile_ext_mixed<true>(x, v, nslope2, dq0, rel_lo, rel_hi)
                         : score_tile_ext_mixed<false>(x, v, nslope2, dq0, rel_lo, rel_hi);
        }
      } else {
        mt = need_mask ? score_tile<kAlibi, kSoftcap, true, kChunkMask>(x, v, nslope2, dq0, rel_lo, rel_hi)
                       : score_tile<kAlibi, kSoftcap, false, kChunkMask>(x, v, nslope2, dq0, rel_lo, rel_hi);
      }
      const float m_run = fmaxf(m_ref, mt);
      bool move, need_o;
      if (m_ref == -INFINITY) {
        move = m_run != -INFINITY;
        need_o = false;          // nothing accumulated yet for this row
      } else {
        move = m_run - m_ref > kTau;
        need_o = move;
      }
      float alpha = 1.f;
      if (need_o) alpha = ex2_approx(m_ref - m_run);   // repair term h = exp(r - r') (Fig. 18d)
      if (move) m_ref = m_run;
      l *= alpha;                                       // xsum = h(xsum) + ...
      if (tid_t == 0) TRACE(27 + 3 * t, j);   // max and repair factor done
      if (t == 0 && tid_t == 32) TRACE(22, j);
      // exp(x - m), local sum, P -> bf16 into TMEM (aliasing S)
      const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
      if constexpr (kPSmem) {
        // PV_t(j-1) must be complete before P_t(j) overwrites sP_t
        // (the rare O rescale stays after the exponentials, where the S registers are dead)
        if (it > 0) {
          WAIT_SM(&o_done[t], (it - 1) & 1);
          tc_fence_after();
        }
      }
      if (tid_t == 0) TRACE(28 + 3 * t, j);   // PV_t(j-1) done
      float e_add = e_off - m_use;
#ifdef ATTN_TRACE
      asm volatile("" : "+f"(e_add));   // trace builds: the exponentials are not hoisted above this point
#endif
      if (tid_t == 0) TRACE(6 + 4 * t, j);
      if (t == 0 && tid_t == 32) TRACE(23, j);
      float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          float a0, a1;   // exponent argument (log2 units): x * e_mul + e_off - m
          if constexpr (kF32x2) {
            fma2_bc(a0, a1, x[c0 + 2 * e], x[c0 + 2 * e + 1], e_mul, e_add);
          } else {
            a0 = fmaf(x[c0 + 2 * e], e_mul, e_add);
            a1 = fmaf(x[c0 + 2 * e + 1], e_mul, e_add);
          }
          float p0, p1;
          exp2_pair<D == 64 ? (kSoftcap ? kPolyGrid64Cap : kPolyGrid64) : (kAlibi ? 0 : kPolyGrid128)>(a0, a1, p0, p1, e);
          if constexpr (kF32x2) {
            add2_acc(sum0, sum1, p0, p1);
          } else {
            sum0 += p0;
            sum1 += p1;
          }
          pk[e] = pack2<kF16>(p0, p1);
        }
        if constexpr (kPSmem) {   // row r of P_t: K-major, 128-B swizzle (the UMMA A layout)
          const int cc = c0;                               // S / P column of pk[0]
          uint8_t* rowp = sP + t * C::kPTileBytes + (cc >> 6) * (BM * 128) + r * 128;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int ch = ((cc & 63) >> 3) + q4;
            *reinterpret_cast<uint4*>(rowp + ((ch ^ (r & 7)) << 4)) =
                make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
          }
        } else {
          tmem_st16(tP + c0 / 2, pk);
        }
      }
      const float sum = sum0 + sum1;
      if (tid_t == 0) TRACE(7 + 4 * t, j);
      if (t == 0 && lane == 0 && wt < 4) TRACE(16 + wq, j);
      // (done after P so the S registers are dead; PV(j) cannot start before P is ready)
      if (__any_sync(0xffffffffu, need_o)) {
        // O = h(O): wait for PV of the previous tile, then rescale this thread's O columns.
        if (v.repair_events != nullptr && lane == 0) atomicAdd(v.repair_events + (D == 64 ? 1 : 0), 1u);
        mbar_wait(&o_done[t], (it - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(tO + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = f2u(u2f(o[e]) * alpha);
          tmem_st32(tO + c * 32, o);
        }
        tmem_st_wait();
      }
      tmem_st_wait();
      l += sum;
#ifdef ATTN_STRICT_WAITS
      // Checking build: the TMEM-aliased-P path (D = 64) waits on o_done only when it rescales O.
      // Skipping the other phases is safe because S_t(j) is produced by the QK MMA the issuer
      // enqueued AFTER PV_t(j-1), and the tcgen05.commit behind s_full tracks every earlier MMA of
      // that thread: s_full(j) complete => PV_t(j-1) complete.  Assert it (trap if the phase is not
      // complete), which also observes every phase for compute-sanitizer's synccheck.
      if (!kPSmem && it > 0 && !__any_sync(0xffffffffu, need_o)) {
        if (!mbar_test_wait(&o_done[t], (it - 1) & 1)) __trap();
        tc_fence_after();
      }
#endif
      if constexpr (kPSmem) fence_proxy_async_smem();   // generic-proxy P stores -> tensor core reads
      tc_fence_before();

      named_bar_arrive(kBarP0 + t, kTileThreads + 32);   // P_t(j) in TMEM / smem -> MMA issuer
    }

    // ------------------------------------------------------------ epilogue: O / l -> 16-bit -> TMA store
    // (s.o_part: fp32 O / l straight to global instead -- the KV-split and context-parallel
    // partials, so the Eq. 8 merge sees un-rounded partials)
    const int n_it = R.hi - R.lo;
    const bool tile_rows = (row0 + t * BM) < s.Sq;
    if (tile_rows) {
      if (n_it > 0) {
        mbar_wait(&o_done[t], (n_it - 1) & 1);
        tc_fence_after();
      } else {
        mbar_wait(q_full, 0);   // the Q tile we overwrite must have landed
      }
      const float inv_l = l > 0.f ? 1.f / l : 0.f;
      if (s.o_part != nullptr) {
        float* dst = s.o_part + (((size_t)zb * s.Hq + hq) * s.Sq + i) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          if (n_it > 0) {
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = 0u;
          }
          if (i < s.Sq) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(dst + c * 32 + e) =
                  make_float4(u2f(o[e]) * inv_l, u2f(o[e + 1]) * inv_l, u2f(o[e + 2]) * inv_l, u2f(o[e + 3]) * inv_l);
          }
        }
      } else {
        uint8_t* sOut = sQ + t * C::kQTileBytes;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          if (n_it > 0) {
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = 0u;
          }
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[e] = pack2<kF16>(u2f(o[2 * e]) * inv_l, u2f(o[2 * e + 1]) * inv_l);
          uint8_t* rowp = sOut + (c >> 1) * (BM * 128) + r * 128;   // 32-column chunk c of the O row
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int ch = (c & 1) * 4 + q4;
            *reinterpret_cast<uint4*>(rowp + ((ch ^ (r & 7)) << 4)) =
                make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1 + t, kTileThreads);
        if (tid_t == 0) {
          for (int bx = 0; bx < C::kBoxes; ++bx) tma_store_4d(&tm_o, sOut + bx * BM * 128, bx * 64, row0 + t * BM, hq, zb);
          bulk_commit();
          bulk_wait_read0();
        }
      }
      if (lse != nullptr && i < s.Sq)
        lse[((size_t)zb * s.Hq + hq) * s.Sq + i] = l > 0.f ? m_ref * kLn2 + logf(l) : -INFINITY;
    }
  }

  tc_fence_before();
  __syncthreads();
#ifdef ATTN_TRACE
  if (trace_cta())
    for (int i = threadIdx.x; i < kTrEv * kTrSteps; i += blockDim.x)
      g_trace[i / kTrSteps][i % kTrSteps] = s_trace[i];
  if (threadIdx.x == 0 && cta_lin < kCtaLog) {
    g_cta[cta_lin][1] = gtimer();
    g_cta[cta_lin][3] = clock64() - g_cta[cta_lin][3];
  }
#endif
  if (warp == kWarpAlloc) {
    tc_fence_after();
    tmem_dealloc<Ro::kTmemCols>(tmem);
  }
}

// ============================================================================
// Persistent variant (D = 128, P in shared memory): one CTA per SM walks a
// static snake schedule of work units (q-block, hq, b[, split]) -- head-major
// with the heaviest causal q-blocks first, so the 148 concurrent units share a
// few heads' K/V in L2 and the snake balances causal work like a dynamic
// scheduler would.  Across units nothing drains: the K/V ring, the S/O TMEM
// buffers and all barrier phases run on, the next unit's K tiles load while the
// previous unit's last PV runs, and its first QK is issued as soon as its Q has
// landed and S is free -- hiding the per-CTA prologue/epilogue a grid of
// short-lived CTAs pays once per unit.  Shared memory holds two 64 KiB regions
// that swap roles each unit: unit u keeps Q in region u&1 and P in region
// (u+1)&1; the epilogue of unit u stages O in its Q region.  Q(u+1) therefore
// loads into P(u)'s region once unit u's PVs are done (pv_done) and unit
// u-1's O store has left it (epi_done).
// ============================================================================
// Used for pure-causal (no window), non-ALiBi problems.  Measured (r1g): causal MHA 996 ->
// 1022 TFLOP/s (short, uneven units: the hidden boundaries matter); non-causal MHA 1229 ->
// 1218 and the GQA window 1120 -> 1102 (long units, and the persistent loop carries more
// live registers), so those stay on the grid kernel; ALiBi needs the grid kernel's
// diagonal-first KV walk.

struct Unit {
  int qblk, hq, zb, b, valid;
};
__device__ __forceinline__ Unit unit_of(const Shape& s, const VariantParams& v, int idx) {
  const int nqb = (s.Sq + 2 * BM - 1) / (2 * BM);
  const int nz = s.B * (s.kv_splits > 1 ? s.kv_splits : 1);
  Unit u;
  u.valid = idx < nqb * s.Hq * nz;
  const int head_lin = idx / nqb, qi = idx % nqb;
  u.qblk = v.causal ? nqb - 1 - qi : qi;          // heaviest causal q-block first
  u.hq = head_lin % s.Hq;
  u.zb = head_lin / s.Hq;
  u.b = s.kv_splits > 1 ? u.zb % s.B : u.zb;
  return u;
}
// k-th unit of CTA c (snake order over rounds of gridDim.x units)
__device__ __forceinline__ int unit_index(int k) {
  const int G = gridDim.x, c = blockIdx.x;
  return G * k + ((k & 1) ? G - 1 - c : c);
}
struct UnitRanges {
  Range r0, r1;
  int ulo, uhi, row0;
  bool has_rows1;
};
__device__ __forceinline__ UnitRanges ranges_of(const Shape& s, const VariantParams& v, const Unit& u) {
  UnitRanges q;
  q.row0 = u.qblk * 2 * BM;
  q.r0 = tile_range(s, v, q.row0);
  q.r1 = tile_range(s, v, q.row0 + BM);
  if (s.kv_splits > 1) {
    const int t_lo = (u.zb / s.B) * s.kv_split_tiles, t_hi = t_lo + s.kv_split_tiles;
    for (Range* r : {&q.r0, &q.r1}) {
      r->lo = max(r->lo, t_lo);
      r->hi = min(r->hi, t_hi);
      if (r->lo >= r->hi) r->lo = r->hi = 0;
    }
  }
  q.has_rows1 = q.row0 + BM < s.Sq;
  q.ulo = q.uhi = 0;
  const bool a0 = q.r0.hi > q.r0.lo, a1 = q.r1.hi > q.r1.lo;
  if (a0 && a1) {
    q.ulo = min(q.r0.lo, q.r1.lo);
    q.uhi = max(q.r0.hi, q.r1.hi);
  } else if (a0) {
    q.ulo = q.r0.lo; q.uhi = q.r0.hi;
  } else if (a1) {
    q.ulo = q.r1.lo; q.uhi = q.r1.hi;
  }
  return q;
}

template <bool kSoftcap, bool kF16>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_tc_persist_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                          const Shape s, const VariantParams v, float* __restrict__ lse) {
  constexpr int D = 128;
  constexpr int kRegion = 2 * BM * D * 2;                    // 64 KiB: two 128 x 128 16-bit tiles
  constexpr int kTile = BM * D * 2;                          // 32 KiB
  constexpr int kStages = 3;
  constexpr int kKV = BN * D * 2;
  constexpr bool kPlain = !kSoftcap;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint8_t* sKV = smem + 2 * kRegion;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * kKV);
  uint64_t* q_full = bars;                 // [2] per region
  uint64_t* kv_full = bars + 2;            // [3]
  uint64_t* kv_empty = kv_full + kStages;  // [3]
  uint64_t* s_full = kv_empty + kStages;   // [2] per tile
  uint64_t* o_done = s_full + 2;           // [2] per tile
  uint64_t* pv_done = o_done + 2;          // [1] all PVs of a unit done
  uint64_t* epi_done = pv_done + 1;        // [2] per region: the O store staged in it has been read
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(epi_done + 2);
  auto region = [&](int r) { return smem + r * kRegion; };

  const uint32_t warp = role_warp_persist(warp_id()), lane = lane_id();
  if (warp == kWarpLoad && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    prefetch_tmap(&tm_o);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&o_done[i], 1);
      mbar_init(&epi_done[i], 2);
    }
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(pv_done, 1);
    fence_mbarrier_init();
  }
  if (warp == kWarpAlloc) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWarpLoad) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      int it = 0;
      auto load_kv = [&](bool is_k, int jj, int hkv, int b) {
        WAIT_LM(&kv_empty[it % kStages], ((it / kStages) & 1) ^ 1);
        uint64_t* bar = &kv_full[it % kStages];
        mbar_arrive_expect_tx(bar, kKV);
        uint8_t* dst = sKV + (it % kStages) * kKV;
        for (int bx = 0; bx < 2; ++bx)
          tma_load_4d(is_k ? &tm_k : &tm_v, bar, dst + bx * BN * 128, bx * 64, jj * BN, hkv, b, pol_kv);
        ++it;
      };
      for (int k = 0;; ++k) {
        const Unit un = unit_of(s, v, unit_index(k));
        if (!un.valid) break;
        const UnitRanges ur = ranges_of(s, v, un);
        const int hkv = un.hq / (s.Hq / s.Hkv);
        if (ur.uhi > ur.ulo) {            // K tiles of this unit go first: they need no region
          load_kv(true, ur.ulo, hkv, un.b);
          if (ur.ulo + 1 < ur.uhi) load_kv(true, ur.ulo + 1, hkv, un.b);
        }
        // Q(k) -> region k&1, which held P(k-1) and the O staging of unit k-2
        if (k >= 1) WAIT_LM(pv_done, (k - 1) & 1);
        if (k >= 2) WAIT_LM(&epi_done[k & 1], ((k - 2) >> 1) & 1);
        const int nq = ur.has_rows1 ? 2 : 1;
        mbar_arrive_expect_tx(&q_full[k & 1], nq * kTile);
        for (int t = 0; t < nq; ++t)
          for (int bx = 0; bx < 2; ++bx)
            tma_load_4d(&tm_q, &q_full[k & 1], region(k & 1) + t * kTile + bx * BM * 128, bx * 64, ur.row0 + t * BM,
                        un.hq, un.b, pol_q);
        for (int j = ur.ulo; j < ur.uhi; ++j) {
          load_kv(false, j, hkv, un.b);
          if (j + 2 < ur.uhi) load_kv(true, j + 2, hkv, un.b);
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ------------------------------------------------------------ MMA issuer (warp-wide)
    constexpr uint32_t idesc_qk = idesc_f16_f32(BM, BN, 0, 0, !kF16);
    constexpr uint32_t idesc_pv = idesc_f16_f32(BM, D, 0, 1, !kF16);
    const uint32_t tS[2] = {tmem, tmem + 128};
    const uint32_t tO[2] = {tmem + 256, tmem + 384};
    int it = 0;
    bool qk_any[2] = {false, false};
    auto wait_tile = [&](int i) {
      WAIT_LM(&kv_full[i % kStages], (i / kStages) & 1);
      tc_fence_after();
    };
    for (int k = 0;; ++k) {
      const Unit un = unit_of(s, v, unit_index(k));
      if (!un.valid) break;
      const UnitRanges ur = ranges_of(s, v, un);
      const Range rg[2] = {ur.r0, ur.r1};
      uint8_t* sQ = region(k & 1);
      uint8_t* sP = region((k + 1) & 1);
      auto qk = [&](int t, int i) {   // S_t = Q_t K^T (K tile in ring slot i)
        if (qk_any[t]) {              // S_t free: its softmax threads hold the previous S_t
          named_bar_sync(kBarS0 + t, kTileThreads + 32);
          tc_fence_after();
        }
        qk_any[t] = true;
        const uint32_t sq = smem_u32(sQ + t * kTile);
        const uint32_t sk = smem_u32(sKV + (i % kStages) * kKV);
        mma_ss_kloop<D / 16>(tS[t], smem_desc_sw128(sq, 16, 1024), BM * 128, smem_desc_sw128(sk, 16, 1024), BN * 128,
                             false, idesc_qk, 0u);
        mma_commit_warp(&s_full[t]);
      };
      auto pv = [&](int t, int i, bool acc) {   // O_t += P_t V (P from this unit's P region)
        named_bar_sync(kBarP0 + t, kTileThreads + 32);
        tc_fence_after();
        const uint32_t sp = smem_u32(sP + t * kTile);
        const uint32_t sv = smem_u32(sKV + (i % kStages) * kKV);
        mma_ss_kloop<BN / 16>(tO[t], smem_desc_sw128(sp, 16, 1024), BM * 128, smem_desc_sw128(sv, BN * 128, 1024), 0,
                              true, idesc_pv, acc ? 1u : 0u);
        mma_commit_warp(&o_done[t]);
      };
      // Q(k) must have landed even for a unit without KV work: pv_done #k may only
      // complete after the producer has waited for #(k-1) (else its parity wait aliases).
      WAIT_LM(&q_full[k & 1], (k >> 1) & 1);
      tc_fence_after();
      if (ur.uhi > ur.ulo) {
        const int itK0 = it++;
        const int itK1 = ur.ulo + 1 < ur.uhi ? it++ : -1;
        wait_tile(itK0);
        if (active(rg[0], ur.ulo)) qk(0, itK0);
        if (active(rg[1], ur.ulo)) qk(1, itK0);
        mma_commit_warp(&kv_empty[itK0 % kStages]);
        if (itK1 >= 0) {
          wait_tile(itK1);
          if (active(rg[0], ur.ulo + 1)) qk(0, itK1);
          if (active(rg[1], ur.ulo + 1)) qk(1, itK1);
          mma_commit_warp(&kv_empty[itK1 % kStages]);
        }
        for (int j = ur.ulo; j < ur.uhi; ++j) {
          const int itV = it++;
          const bool k2 = j + 2 < ur.uhi;
          const int itK = k2 ? it++ : 0;
          wait_tile(itV);
          if (active(rg[0], j)) pv(0, itV, j > rg[0].lo);
          if (k2) {
            wait_tile(itK);
            if (active(rg[0], j + 2)) qk(0, itK);
          }
          if (active(rg[1], j)) pv(1, itV, j > rg[1].lo);
          mma_commit_warp(&kv_empty[itV % kStages]);
          if (k2) {
            if (active(rg[1], j + 2)) qk(1, itK);
            mma_commit_warp(&kv_empty[itK % kStages]);
          }
        }
      }
      mma_commit_warp(pv_done);       // every MMA of unit k (its P region is free once this lands)
    }
    for (int t = 0; t < 2; ++t)      // the softmax's arrival for its last S load
      if (qk_any[t]) named_bar_sync(kBarS0 + t, kTileThreads + 32);
  } else if (warp < kSoftmaxWarps) {
    // ------------------------------------------------------------ softmax / correction / epilogue
    const int t = (int)warp / 4;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const int tid_t = (warp & 3) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tS = tmem + t * 128 + lane_off;
    const uint32_t tO = tmem + 256 + t * 128 + lane_off;
    uint32_t n_s = 0, n_pv = 0;            // S loads / PVs of this tile so far (barrier phases)
    for (int k = 0;; ++k) {
      const Unit un = unit_of(s, v, unit_index(k));
      if (!un.valid) break;
      const UnitRanges ur = ranges_of(s, v, un);
      const Range R = t == 0 ? ur.r0 : ur.r1;
      const int row0 = ur.row0;
      const int hq = un.hq;
      const int i = row0 + t * BM + r;
      const long long qpos = v.q_off + i;
      int jlo_row, jhi_row;
      row_bounds(s, v, qpos, jlo_row, jhi_row);
      uint8_t* sP = region((k + 1) & 1) + t * kTile;
      float m_ref = -INFINITY, l = 0.f;
      for (int j = R.lo; j < R.hi; ++j) {
        WAIT_SM(&s_full[t], n_s & 1);
        ++n_s;
        tc_fence_after();
        float x[BN];
        {
          uint32_t u[BN];
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS + c * 32, reinterpret_cast<uint32_t(&)[32]>(u[c * 32]));
          tmem_ld_wait();
          tc_fence_before();
          named_bar_arrive(kBarS0 + t, kTileThreads + 32);   // S_t may be overwritten
#pragma unroll
          for (int c = 0; c < BN; ++c) x[c] = u2f(u[c]);
        }
        const bool need_mask = !(j * BN >= R.jlo_last && (j + 1) * BN - 1 <= R.jhi_first);
        const int rel_lo = jlo_row - j * BN, rel_hi = jhi_row - j * BN;
        const float dq0 = (float)(qpos - v.kv_off - (long long)j * BN);
        const float mt = need_mask ? score_tile<false, kSoftcap, true, true>(x, v, 0.f, dq0, rel_lo, rel_hi)
                                   : score_tile<false, kSoftcap, false, true>(x, v, 0.f, dq0, rel_lo, rel_hi);
        const float m_run = fmaxf(m_ref, mt);
        bool move, need_o;
        if (m_ref == -INFINITY) {
          move = m_run != -INFINITY;
          need_o = false;
        } else {
          move = m_run - m_ref > kTau;
          need_o = move;
        }
        float alpha = 1.f;
        if (need_o) alpha = ex2_approx(m_ref - m_run);   // repair term h = exp(r - r') (Fig. 18d)
        if (move) m_ref = m_run;
        l *= alpha;
        const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
        const float e_add = -m_use;
        if (n_pv > 0) {                 // PV_t of the previous step (maybe of the previous unit) is done
          WAIT_SM(&o_done[t], (n_pv - 1) & 1);
          tc_fence_after();
        }
        float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float a0, a1;   // exponent argument (log2 units), packed FFMA2
            fma2_bc(a0, a1, x[c0 + 2 * e], x[c0 + 2 * e + 1], kPlain ? v.scale_log2 : 1.f, e_add);
            float p0, p1;
            exp2_pair<kPolyPersist>(a0, a1, p0, p1, e);
            add2_acc(sum0, sum1, p0, p1);
            pk[e] = pack2<kF16>(p0, p1);
          }
          uint8_t* rowp = sP + (c0 >> 6) * (BM * 128) + r * 128;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int ch = ((c0 & 63) >> 3) + q4;
            *reinterpret_cast<uint4*>(rowp + ((ch ^ (r & 7)) << 4)) =
                make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
          }
        }
        if (__any_sync(0xffffffffu, need_o)) {   // O = h(O) (rare: lazy repair, R9)
          if (v.repair_events != nullptr && lane == 0) atomicAdd(v.repair_events + 2, 1u);
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = f2u(u2f(o[e]) * alpha);
            tmem_st32(tO + c * 32, o);
          }
          tmem_st_wait();
        }
        l += sum0 + sum1;
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_arrive(kBarP0 + t, kTileThreads + 32);   // P_t(j) -> MMA issuer
        ++n_pv;
      }
      // ---------------------------------------------------------- epilogue of unit k, tile t
      const int n_it = R.hi - R.lo;
      uint8_t* sOut = region(k & 1) + t * kTile;
      const bool tile_rows = (row0 + t * BM) < s.Sq;
      if (tile_rows) {
        if (n_it > 0) {
          mbar_wait(&o_done[t], (n_pv - 1) & 1);
          tc_fence_after();
        } else {
          mbar_wait(&q_full[k & 1], (k >> 1) & 1);   // the Q tile we overwrite must have landed
        }
        const float inv_l = l > 0.f ? 1.f / l : 0.f;
        if (s.o_part != nullptr) {   // fp32 normalised partial straight to global (no staging)
          float* dst = s.o_part + (((size_t)un.zb * s.Hq + hq) * s.Sq + i) * D;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            if (n_it > 0) {
              tmem_ld32(tO + c * 32, o);
              tmem_ld_wait();
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = 0u;
            }
            if (i < s.Sq) {
#pragma unroll
              for (int e = 0; e < 32; e += 4)
                *reinterpret_cast<float4*>(dst + c * 32 + e) = make_float4(
                    u2f(o[e]) * inv_l, u2f(o[e + 1]) * inv_l, u2f(o[e + 2]) * inv_l, u2f(o[e + 3]) * inv_l);
            }
          }
          tc_fence_before();
          if (tid_t == 0) mbar_arrive(&epi_done[k & 1]);
        } else {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            if (n_it > 0) {
              tmem_ld32(tO + c * 32, o);
              tmem_ld_wait();
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = 0u;
            }
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[e] = pack2<kF16>(u2f(o[2 * e]) * inv_l, u2f(o[2 * e + 1]) * inv_l);
            uint8_t* rowp = sOut + (c >> 1) * (BM * 128) + r * 128;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int ch = (c & 1) * 4 + q4;
              *reinterpret_cast<uint4*>(rowp + ((ch ^ (r & 7)) << 4)) =
                  make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
            }
          }
          tc_fence_before();
          fence_proxy_async_smem();
          named_bar_sync(1 + t, kTileThreads);
          if (tid_t == 0) {
            for (int bx = 0; bx < 2; ++bx) tma_store_4d(&tm_o, sOut + bx * BM * 128, bx * 64, row0 + t * BM, hq, un.zb);
            bulk_commit();
            bulk_wait_read0();
            mbar_arrive(&epi_done[k & 1]);
          }
        }
        if (lse != nullptr && i < s.Sq)
          lse[((size_t)un.zb * s.Hq + hq) * s.Sq + i] = l > 0.f ? m_ref * kLn2 + logf(l) : -INFINITY;
        if (s.o_part == nullptr) named_bar_sync(1 + t, kTileThreads);   // the staging tile is free again (P of unit k+1 goes there)
      } else if (tid_t == 0) {
        mbar_arrive(&epi_done[k & 1]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpAlloc) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int sm_count_of_current_device() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  int& c = cache[dev & 63];
  if (c == 0 && cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) c = 148;
  return c;
}

template <bool kSoftcap, bool kF16>
cudaError_t launch_persist(const FwdTcArgs& a, cudaStream_t stream) {
  constexpr int kSmem = 4 * (2 * BM * 128 * 2) / 2 + 3 * (BN * 128 * 2) + 16 * 8 + 16;   // 2 regions + ring + bars
  cudaError_t e = set_smem_once<fwd_tc_persist_kernel<kSoftcap, kF16>>(kSmem);
  if (e != cudaSuccess) return e;
  const long long nqb = (a.s.Sq + 2 * BM - 1) / (2 * BM);
  const long long units = nqb * a.s.Hq * a.s.B * (a.s.kv_splits > 1 ? a.s.kv_splits : 1);
  const int grid = (int)std::min<long long>(units, sm_count_of_current_device());
  fwd_tc_persist_kernel<kSoftcap, kF16>
      <<<grid, kThreads, kSmem, stream>>>(a.tm_q, a.tm_k, a.tm_v, a.tm_o, a.s, a.v, a.lse);
  return cudaGetLastError();
}

template <int D, bool kAlibi, bool kSoftcap, bool kF16>
cudaError_t launch_t(const FwdTcArgs& a, cudaStream_t stream) {
  constexpr int NT = nt_of<D>();
  using C = Cfg<D, alibi_mma<D, kAlibi && !kSoftcap>(), NT>;
  static_assert(C::kSmemBytes <= 232448, "shared memory");
  if constexpr (D == 128 && !kAlibi && !kTraceBuild) {
    // pure causal -> the persistent kernel (ALiBi stays on the grid kernel: it walks the KV
    // tiles diagonal-first, see J in fwd_tc_kernel)
    if (a.v.causal && a.v.window_left < 0 && a.v.window_right < 0) return launch_persist<kSoftcap, kF16>(a, stream);
  }
  auto kern = fwd_tc_kernel<D, kAlibi, kSoftcap, kF16, NT>;
  cudaError_t e = set_smem_once<fwd_tc_kernel<D, kAlibi, kSoftcap, kF16, NT>>(C::kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid((a.s.Sq + NT * BM - 1) / (NT * BM), a.s.Hq, a.s.B * (a.s.kv_splits > 1 ? a.s.kv_splits : 1));
  kern<<<grid, Roles<NT>::kThreads, C::kSmemBytes, stream>>>(a.tm_q, a.tm_k, a.tm_v, a.tm_o, a.s, a.v, a.lse);
  return cudaGetLastError();
}

template <int D, bool kF16>
cudaError_t launch_d(const FwdTcArgs& a, cudaStream_t stream) {
  const bool alibi = a.v.alibi != nullptr, cap = a.v.softcap > 0.f;
  if (alibi && cap) return launch_t<D, true, true, kF16>(a, stream);
  if (alibi) return launch_t<D, true, false, kF16>(a, stream);
  if (cap) return launch_t<D, false, true, kF16>(a, stream);
  return launch_t<D, false, false, kF16>(a, stream);
}

}  // namespace

#ifdef ATTN_TRACE
extern "C" __attribute__((visibility("default"))) int attn_debug_cta_log(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_cta, sizeof(g_cta));
}
extern "C" __attribute__((visibility("default"))) int attn_debug_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace));
}
#endif

int fwd_kv_tile_keys(int D) { return D == 64 ? bn_of<64>() : bn_of<128>(); }

cudaError_t launch_fwd_tc(const FwdTcArgs& a, cudaStream_t stream, int* launches) {
  cudaError_t e = a.f16 ? (a.s.D == 128 ? launch_d<128, true>(a, stream) : launch_d<64, true>(a, stream))
                        : (a.s.D == 128 ? launch_d<128, false>(a, stream) : launch_d<64, false>(a, stream));
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

}  // namespace attn
