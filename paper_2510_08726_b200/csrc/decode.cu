// decode.cu -- Split-K Update for decoding (Alg. 2; Fig. 5,
// P:706-722) and its global repair-combine (Eq. 8).
//
// Local section (decode_split_kernel): one CTA per (split, hkv, b).  The KV
// axis of (b, hkv) is privatised into contiguous splits (FuseAndPrivatize,
// P:673-677); the CTA streams its split of K and V from HBM exactly once
// through a TMA ring (128-byte swizzled [keys x 64] boxes) and computes, for
// all G = Hq / Hkv query heads of the group at once, the local max m_s, the
// local sum l_s = sum exp(x - m_s) and the un-normalised PV_s.  Inside a split
// each warp runs a rolling update over 16-key sub-tiles (Fig. 19), and the
// four warps' states are merged with the Eq. 8 algebra at the end.
//
// Decode is HBM-bound (4 flop per K/V byte at G = 4).  The G query heads are
// packed as rows of a 16-row mma.sync tile with the unused rows zero ("uses
// masks to apply TensorCore ... too few input matrix rows"), so
// the CUDA cores only do the softmax and the instruction budget per streamed
// byte stays far below the issue rate.
//
// Global section (combine_kernel): per (b, h): M = max_s m_s, w_s =
// exp(m_s - M), L = sum w_s l_s, O = sum w_s O_s; output O / L and
// lse = M + ln L, or the un-normalised merged triple for hierarchical merges.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>

#include "kernels.h"
#include "ptx.cuh"

namespace attn {
namespace {

constexpr int kConsumerWarps = 4;
constexpr int kKeysPerWarp = 16;
constexpr int NK = kConsumerWarps * kKeysPerWarp;  // keys per stage
#ifndef DEC_STAGES
#define DEC_STAGES 3
#endif
constexpr int kStages = DEC_STAGES;   // K+V ring stages (32 KiB each at D = 128)
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct DCfg {
  static constexpr int kBoxes = D / 64;
  static constexpr int kTileBytes = NK * D * 2;               // one K (or V) stage tile
  static constexpr int kStageBytes = 2 * kTileBytes;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + 2 * kStages * 8 + 64;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
template <bool kF16>
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (kF16)
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Byte offset of 16-byte chunk `ch` (0 .. D/8-1) of row `key` in a stage tile
// made of D/64 TMA boxes of [NK rows x 128 B] with the 128-byte swizzle.
__device__ __forceinline__ uint32_t tile_off(int key, int ch) {
  return (ch >> 3) * (NK * 128) + key * 128 + (((ch & 7) ^ (key & 7)) << 4);
}

// kHi: the packed (head, query) rows reach past 8 (G * Sq in 9..16): rows g + 8 of the
// m16n8k16 tiles carry data too (multi-token decode, NEXT-2).
template <int D, bool kAlibi, bool kSoftcap, bool kF16, bool kHi>
__global__ void __launch_bounds__(kThreads) decode_split_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                                const __grid_constant__ CUtensorMap tm_v,
                                                                const DecodeArgs a) {
  using C = DCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes);
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, hkv = blockIdx.y, b = blockIdx.z;
  const int G = a.s.Hq / a.s.Hkv;
  const int ks = split * a.split_len;
  const int ke = min(ks + a.split_len, a.s.Skv);
  const int nstage = ke > ks ? (ke - ks + NK - 1) / NK : 0;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumerWarps);
    }
    fence_mbarrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();   // K/V are streamed exactly once
      for (int st = 0; st < nstage; ++st) {
        const int slot = st % kStages;
        mbar_wait(&empty[slot], ((st / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[slot], C::kStageBytes);
        uint8_t* dst = smem + slot * C::kStageBytes;
        for (int bx = 0; bx < C::kBoxes; ++bx) {
          tma_load_4d(&tm_k, &full[slot], dst + bx * NK * 128, bx * 64, ks + st * NK, hkv, b, pol);
          tma_load_4d(&tm_v, &full[slot], dst + C::kTileBytes + bx * NK * 128, bx * 64, ks + st * NK, hkv, b, pol);
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  // Packed mma rows: rho = h * Sq + i (query head h of the group, query i); thread-quad
  // group g owns rows g (fragment halves 0/1) and g + 8 (halves 2/3, only with kHi).
  const VariantParams& v = a.v;
  const int Sq = a.s.Sq;
  const int nrows = G * Sq;
  const int quad = lane & 3;
  const int r_lo = lane >> 2, r_hi = r_lo + 8;
  const bool ok_lo = r_lo < nrows, ok_hi = kHi && r_hi < nrows;
  const int h_lo = ok_lo ? r_lo / Sq : 0, i_lo = ok_lo ? r_lo % Sq : 0;
  const int h_hi = ok_hi ? r_hi / Sq : 0, i_hi = ok_hi ? r_hi % Sq : 0;
  const int hq_lo = hkv * G + h_lo, hq_hi = hkv * G + h_hi;
  const long long qpos_lo = v.q_off + i_lo, qpos_hi = v.q_off + i_hi;
  // Q as the A operand: rows = packed (head, query) pairs (zero beyond nrows); loaded once.
  uint32_t qa[D / 16][4];
  {
    const uint16_t* q_lo = a.q + (long long)b * a.q_sb + (long long)hq_lo * a.q_sh + (long long)i_lo * a.q_ss;
    const uint16_t* q_hi = a.q + (long long)b * a.q_sb + (long long)hq_hi * a.q_sh + (long long)i_hi * a.q_ss;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int d0 = kk * 16 + quad * 2;
      qa[kk][0] = ok_lo ? *reinterpret_cast<const uint32_t*>(q_lo + d0) : 0u;
      qa[kk][1] = ok_hi ? *reinterpret_cast<const uint32_t*>(q_hi + d0) : 0u;
      qa[kk][2] = ok_lo ? *reinterpret_cast<const uint32_t*>(q_lo + d0 + 8) : 0u;
      qa[kk][3] = ok_hi ? *reinterpret_cast<const uint32_t*>(q_hi + d0 + 8) : 0u;
    }
  }
  // allowed key interval of each row's query (local indices), intersected with the split
  auto bounds = [&](long long qpos, long long& jlo, long long& jhi) {
    jlo = ks;
    jhi = ke - 1;
    if (v.window_left >= 0) jlo = max(jlo, qpos - v.window_left - v.kv_off);
    if (v.causal) jhi = min(jhi, qpos - v.kv_off);
    if (v.window_right >= 0) jhi = min(jhi, qpos + v.window_right - v.kv_off);
  };
  long long jlo_lo, jhi_lo, jlo_hi = 0, jhi_hi = -1;
  bounds(qpos_lo, jlo_lo, jhi_lo);
  if (kHi) bounds(qpos_hi, jlo_hi, jhi_hi);
  const float ns_lo = (kAlibi && ok_lo) ? -v.alibi[hq_lo] * kLog2e : 0.f;
  const float ns_hi = (kAlibi && ok_hi) ? -v.alibi[hq_hi] * kLog2e : 0.f;

  float m_lo = -INFINITY, m_hi = -INFINITY;   // running max of this warp's keys per row (log2 units)
  float l_lo = 0.f, l_hi = 0.f;               // per-thread partials of the running denominators
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;

  // one row half: score_mod + mask (log2 units), quad-max, repair, p = exp(x - m)
  auto row_step = [&](const float (&sv)[2][4], int hoff, long long qpos, long long jlo, long long jhi, float nsl,
                      bool ok, int key0, float& m, float& l, float (&p)[4]) -> float {
    float x[4];
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = key0 + n * 8 + quad * 2 + e;
        float xv = sv[n][hoff + e];
        if constexpr (kSoftcap) {
          xv = v.softcap_log2 * tanh_approx(xv * v.scale_over_cap);
        } else {
          xv *= v.scale_log2;
        }
        if constexpr (kAlibi) xv = fmaf(nsl, fabsf((float)(qpos - v.kv_off - j)), xv);
        x[n * 2 + e] = (j >= jlo && j <= jhi && ok) ? xv : -INFINITY;
      }
    float mt = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
    mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
    mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
    const float m_new = fmaxf(m, mt);
    // repair term exp(m_old - m_new) (Fig. 18d); guards for rows still empty
    const float alpha = (m == -INFINITY) ? 0.f : ex2_approx(m - m_new);
    const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = ex2_approx(x[e] - m_use);
    l = l * alpha + (p[0] + p[1] + p[2] + p[3]);
    m = m_new;
    return alpha;
  };

  for (int st = 0; st < nstage; ++st) {
    const int slot = st % kStages;
    mbar_wait(&full[slot], (st / kStages) & 1);
    const uint32_t sk = smem_u32(smem + slot * C::kStageBytes);
    const uint32_t sv = sk + C::kTileBytes;
    const int kb = warp * kKeysPerWarp;   // this warp's 16 keys of the stage

    // S (16 rows x 16 keys) = Q K^T
    float s4[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    {
      const int key = kb + (lane & 7) + ((lane >> 4) << 3);
      const int sub = (lane >> 3) & 1;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sk + tile_off(key, kk * 2 + sub), b0, b1, b2, b3);
        mma16816<kF16>(s4[0], qa[kk], b0, b1);
        mma16816<kF16>(s4[1], qa[kk], b2, b3);
      }
    }
    const int key0 = ks + st * NK + kb;
    float p_lo[4], p_hi[4] = {0.f, 0.f, 0.f, 0.f};
    const float a_lo = row_step(s4, 0, qpos_lo, jlo_lo, jhi_lo, ns_lo, ok_lo, key0, m_lo, l_lo, p_lo);
    float a_hi = 1.f;
    if constexpr (kHi) a_hi = row_step(s4, 2, qpos_hi, jlo_hi, jhi_hi, ns_hi, ok_hi, key0, m_hi, l_hi, p_hi);
    if (v.repair_events != nullptr &&   // test instrumentation: a live O accumulator rescaled by < 1
        __any_sync(0xffffffffu, (a_lo > 0.f && a_lo < 1.f) || (a_hi > 0.f && a_hi < 1.f)) && lane == 0)
      atomicAdd(v.repair_events + 3, 1u);
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      o[n][0] *= a_lo;
      o[n][1] *= a_lo;
      if constexpr (kHi) {
        o[n][2] *= a_hi;
        o[n][3] *= a_hi;
      }
    }
    // P as the A operand: rows g (keys 2t.., 2t+8..) and g + 8
    uint32_t pa[4];
    pa[0] = pack2<kF16>(p_lo[0], p_lo[1]);
    pa[1] = kHi ? pack2<kF16>(p_hi[0], p_hi[1]) : 0u;
    pa[2] = pack2<kF16>(p_lo[2], p_lo[3]);
    pa[3] = kHi ? pack2<kF16>(p_hi[2], p_hi[3]) : 0u;
    // O (16 x D) += P V
    {
      const int key = kb + (lane & 7) + (((lane >> 3) & 1) << 3);
      const int sub = lane >> 4;
#pragma unroll
      for (int nd = 0; nd < D / 8; nd += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sv + tile_off(key, nd + sub), b0, b1, b2, b3);
        mma16816<kF16>(o[nd], pa, b0, b1);
        mma16816<kF16>(o[nd + 1], pa, b2, b3);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }

  // ------------------------------------------------------------ merge the 4 warps (Eq. 8) and emit
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  if constexpr (kHi) {
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
  }
  // every stage's smem is free now: reuse it for the reduction
  named_bar_sync(1, kConsumerWarps * 32);
  float* red = reinterpret_cast<float*>(smem);   // [warp][16 rows][D + 2]
  {
    float* rw = red + (warp * 16 + r_lo) * (D + 2);
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      rw[n * 8 + quad * 2] = o[n][0];
      rw[n * 8 + quad * 2 + 1] = o[n][1];
    }
    if (quad == 0) {
      rw[D] = m_lo;
      rw[D + 1] = l_lo;
    }
    if constexpr (kHi) {
      float* rh = red + (warp * 16 + r_hi) * (D + 2);
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        rh[n * 8 + quad * 2] = o[n][2];
        rh[n * 8 + quad * 2 + 1] = o[n][3];
      }
      if (quad == 0) {
        rh[D] = m_hi;
        rh[D + 1] = l_hi;
      }
    }
  }
  named_bar_sync(1, kConsumerWarps * 32);
  for (int e = threadIdx.x; e < nrows * D; e += kConsumerWarps * 32) {
    const int rho = e / D, d = e % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, red[(w * 16 + rho) * (D + 2) + D]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        const float* r = red + (w * 16 + rho) * (D + 2);
        const float mw = r[D];
        const float wgt = (mw == -INFINITY) ? 0.f : ex2_approx(mw - M);
        L = fmaf(wgt, r[D + 1], L);
        O = fmaf(wgt, r[d], O);
      }
    }
    const int hh = hkv * G + rho / Sq, qi = rho % Sq;
    float* po = a.parts.o + split * a.parts.o_sp + (long long)b * a.parts.o_sb + (long long)hh * a.parts.o_sh +
                (long long)qi * D;
    po[d] = O;
    if (d == 0) {
      const long long mi = split * a.parts.m_sp + (long long)b * a.parts.m_sb + (long long)hh * a.parts.m_sh + qi;
      a.parts.m[mi] = M * kLn2;   // natural-log units (ABI)
      a.parts.l[mi] = L;
    }
  }
  if (a.tickets == nullptr) return;

  // ------------------------------------------------------------ fused global section (Eq. 8)
  // Every CTA publishes its triples (fence, then one ticket per CTA); the last of the
  // (b, hkv) group reads all splits back from L2 and combines them: no second launch.
  __shared__ int s_last;
  __threadfence();
  named_bar_sync(1, kConsumerWarps * 32);
  unsigned* ticket = a.tickets + (long long)b * a.s.Hkv + hkv;
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == (unsigned)a.num_splits - 1;
  named_bar_sync(1, kConsumerWarps * 32);
  if (!s_last) return;
  __threadfence();
  const int S = a.num_splits;
  float* wts = red;                       // [nrows][S] weights exp(m_s - M) (smem reused)
  float* stat = red + nrows * S;          // [nrows][2]: M (natural log), L
  for (int rho = warp; rho < nrows; rho += kConsumerWarps) {   // warp reduces row rho over the splits
    const int hh = hkv * G + rho / Sq, qi = rho % Sq;
    const long long mb = (long long)b * a.parts.m_sb + (long long)hh * a.parts.m_sh + qi;
    // one round trip: every lane loads its splits' (m, l) pairs before any reduction
    constexpr int kMaxPer = 8;            // splits per lane held in registers (S <= 256 here)
    float ms[kMaxPer], ls[kMaxPer];
#pragma unroll
    for (int i = 0; i < kMaxPer; ++i) {
      const int sp = lane + 32 * i;
      ms[i] = sp < S ? __ldcg(a.parts.m + sp * a.parts.m_sp + mb) : -INFINITY;
      ls[i] = sp < S ? __ldcg(a.parts.l + sp * a.parts.m_sp + mb) : 0.f;
    }
    float M = -INFINITY;
#pragma unroll
    for (int i = 0; i < kMaxPer; ++i) M = fmaxf(M, ms[i]);
    for (int sp = lane + 32 * kMaxPer; sp < S; sp += 32) M = fmaxf(M, __ldcg(a.parts.m + sp * a.parts.m_sp + mb));
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o2));
    float L = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxPer; ++i) {
      const int sp = lane + 32 * i;
      if (sp < S) {
        const float w = (ms[i] == -INFINITY) ? 0.f : expf(ms[i] - M);   // repair term exp(max_s - max_g)
        wts[rho * S + sp] = w;
        L = fmaf(w, ls[i], L);
      }
    }
    for (int sp = lane + 32 * kMaxPer; sp < S; sp += 32) {
      const float m_s = __ldcg(a.parts.m + sp * a.parts.m_sp + mb);
      const float w = (m_s == -INFINITY) ? 0.f : expf(m_s - M);
      wts[rho * S + sp] = w;
      L = fmaf(w, __ldcg(a.parts.l + sp * a.parts.m_sp + mb), L);
    }
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o2);
    if (lane == 0) {
      stat[rho * 2] = M;
      stat[rho * 2 + 1] = L;
    }
  }
  named_bar_sync(1, kConsumerWarps * 32);
  // O = sum_s w_s O_s: one float4 of one row per thread, the splits' loads issued in batches of 8
  for (int e4 = threadIdx.x; e4 < nrows * (D / 4); e4 += kConsumerWarps * 32) {
    const int rho = e4 / (D / 4), d = (e4 % (D / 4)) * 4;
    const int hh = hkv * G + rho / Sq, qi = rho % Sq;
    const float L = stat[rho * 2 + 1];
    const float* po = a.parts.o + (long long)b * a.parts.o_sb + (long long)hh * a.parts.o_sh + (long long)qi * D + d;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (L > 0.f) {
      for (int s0 = 0; s0 < S; s0 += 8) {
        float4 ov[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          ov[i] = s0 + i < S ? __ldcg(reinterpret_cast<const float4*>(po + (long long)(s0 + i) * a.parts.o_sp))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float w = s0 + i < S ? wts[rho * S + s0 + i] : 0.f;
          acc.x = fmaf(w, ov[i].x, acc.x);
          acc.y = fmaf(w, ov[i].y, acc.y);
          acc.z = fmaf(w, ov[i].z, acc.z);
          acc.w = fmaf(w, ov[i].w, acc.w);
        }
      }
    }
    if (a.packed != nullptr) {   // un-normalised triple for a further Eq. 8 merge (KV-sharded decode)
      float* row = a.packed + ((long long)b * a.s.Hq + hh) * (D + 2);
      row[d] = acc.x;
      row[d + 1] = acc.y;
      row[d + 2] = acc.z;
      row[d + 3] = acc.w;
      if (d == 0) {
        row[D] = L > 0.f ? stat[rho * 2] : -INFINITY;
        row[D + 1] = L;
      }
      continue;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    const float out[4] = {acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv};
    const long long oi = (long long)b * a.o_sb + (long long)hh * a.o_sh + (long long)qi * a.o_ss + d;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (a.out_f16) reinterpret_cast<__half*>(a.o)[oi + c] = __float2half_rn(out[c]);
      else reinterpret_cast<__nv_bfloat16*>(a.o)[oi + c] = __float2bfloat16_rn(out[c]);
    }
    if (d == 0 && a.lse) a.lse[((long long)b * a.s.Hq + hh) * Sq + qi] = L > 0.f ? stat[rho * 2] + logf(L) : -INFINITY;
  }
  if (threadIdx.x == 0) *ticket = 0u;     // ready for the next call
}

// ---------------------------------------------------------------- Eq. 8 combine
__global__ void __launch_bounds__(128) combine_kernel(const CombineArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * 4 + warp;   // (b, h)
  if (idx >= a.B * a.H) return;
  const int b = idx / a.H, h = idx % a.H;
  const PartsView& in = a.in;
  const long long mb = (long long)b * in.m_sb + (long long)h * in.m_sh;
  const long long ob = (long long)b * in.o_sb + (long long)h * in.o_sh;
  float M = -INFINITY;
  for (int p = lane; p < in.num_parts; p += 32) M = fmaxf(M, in.m[p * in.m_sp + mb]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float L = 0.f;
  constexpr int kMaxDL = 8;   // D <= 256
  float acc[kMaxDL];
#pragma unroll
  for (int r = 0; r < kMaxDL; ++r) acc[r] = 0.f;
  if (M != -INFINITY) {
    for (int p = 0; p < in.num_parts; ++p) {
      const float mp = in.m[p * in.m_sp + mb];
      if (mp == -INFINITY) continue;            // w_p = 0 for empty parts
      const float w = expf(mp - M);              // repair term exp(max_l - max_g)
      L = fmaf(w, in.l[p * in.m_sp + mb], L);
      const float* op = in.o + p * in.o_sp + ob;
#pragma unroll
      for (int r = 0; r < kMaxDL; ++r) {
        const int d = lane + 32 * r;
        if (d < a.D) acc[r] = fmaf(w, op[d], acc[r]);
      }
    }
  }
  if (a.o) {
    const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int r = 0; r < kMaxDL; ++r) {
      const int d = lane + 32 * r;
      if (d >= a.D) continue;
      const long long oi = (long long)b * a.o_sb + (long long)h * a.o_sh + d;
      if (a.out_bf16 == 1)
        reinterpret_cast<__nv_bfloat16*>(a.o)[oi] = __float2bfloat16_rn(acc[r] * inv);
      else if (a.out_bf16 == 2)
        reinterpret_cast<__half*>(a.o)[oi] = __float2half_rn(acc[r] * inv);
      else
        reinterpret_cast<float*>(a.o)[oi] = acc[r] * inv;
    }
  }
  if (a.lse && lane == 0) a.lse[(long long)b * a.H + h] = L > 0.f ? M + logf(L) : -INFINITY;
  if (a.acc.m) {
    const long long mi = (long long)b * a.acc.m_sb + (long long)h * a.acc.m_sh;
    if (lane == 0) {
      a.acc.m[mi] = L > 0.f ? M : -INFINITY;
      a.acc.l[mi] = L;
    }
    float* po = a.acc.o + (long long)b * a.acc.o_sb + (long long)h * a.acc.o_sh;
#pragma unroll
    for (int r = 0; r < kMaxDL; ++r) {
      const int d = lane + 32 * r;
      if (d < a.D) po[d] = acc[r];
    }
  }
}

// ---------------------------------------------------------------- Eq. 8 over normalised partials
__device__ __forceinline__ float load_elem(const void* p, long long i, int dt) {
  if (dt == 1) return static_cast<const float*>(p)[i];
  if (dt == 2) return __half2float(static_cast<const __half*>(p)[i]);
  return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}
__device__ __forceinline__ void store_elem(void* p, long long i, int dt, float x) {
  if (dt == 1) static_cast<float*>(p)[i] = x;
  else if (dt == 2) static_cast<__half*>(p)[i] = __float2half_rn(x);
  else static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(x);
}

__global__ void __launch_bounds__(128) merge_kernel(const MergeArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * 4 + warp;
  if (row >= a.rows) return;
  float M = -INFINITY;
  for (int p = lane; p < a.P; p += 32) M = fmaxf(M, a.lse_in[p * a.l_sp + row]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  constexpr int kMaxDL = 8;   // D <= 256
  float acc[kMaxDL];
#pragma unroll
  for (int r = 0; r < kMaxDL; ++r) acc[r] = 0.f;
  float L = 0.f;
  if (M != -INFINITY) {
    for (int p = 0; p < a.P; ++p) {
      const float lp = a.lse_in[p * a.l_sp + row];
      if (lp == -INFINITY) continue;                  // empty part: weight 0
      const float w = expf(lp - M);                    // repair term exp(lse_p - M), l_p = 1
      L += w;
      const long long base = p * a.o_sp + row * a.o_sr;
#pragma unroll
      for (int r = 0; r < kMaxDL; ++r) {
        const int d = lane + 32 * r;
        if (d < a.D) acc[r] = fmaf(w, load_elem(a.o_in, base + d, a.in_dtype), acc[r]);
      }
    }
  }
  if (a.o_out) {
    const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int r = 0; r < kMaxDL; ++r) {
      const int d = lane + 32 * r;
      if (d >= a.D) continue;
      long long oi = row * a.o_out_sr + d;
      if (a.out_Sq > 0) {
        const long long bh = row / a.out_Sq, i = row % a.out_Sq;
        oi = (bh / a.out_H) * a.o_out_sb + (bh % a.out_H) * a.o_out_sh + i * a.o_out_sr + d;
      }
      store_elem(a.o_out, oi, a.out_dtype, acc[r] * inv);
    }
  }
  if (a.lse_out && lane == 0) a.lse_out[row] = L > 0.f ? M + logf(L) : -INFINITY;
}

template <int D, bool kAlibi, bool kSoftcap, bool kF16, bool kHi>
cudaError_t launch_dec_h(const DecodeArgs& a, cudaStream_t stream) {
  using C = DCfg<D>;
  auto kern = decode_split_kernel<D, kAlibi, kSoftcap, kF16, kHi>;
  cudaError_t e = set_smem_once<decode_split_kernel<D, kAlibi, kSoftcap, kF16, kHi>>(C::kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid(a.num_splits, a.s.Hkv, a.s.B);
  kern<<<grid, kThreads, C::kSmemBytes, stream>>>(a.tm_k, a.tm_v, a);
  return cudaGetLastError();
}

template <int D, bool kAlibi, bool kSoftcap, bool kF16>
cudaError_t launch_dec_t(const DecodeArgs& a, cudaStream_t stream) {
  return (a.s.Hq / a.s.Hkv) * a.s.Sq > 8 ? launch_dec_h<D, kAlibi, kSoftcap, kF16, true>(a, stream)
                                         : launch_dec_h<D, kAlibi, kSoftcap, kF16, false>(a, stream);
}

template <int D, bool kF16>
cudaError_t launch_dec_d(const DecodeArgs& a, cudaStream_t stream) {
  const bool alibi = a.v.alibi != nullptr, cap = a.v.softcap > 0.f;
  if (alibi && cap) return launch_dec_t<D, true, true, kF16>(a, stream);
  if (alibi) return launch_dec_t<D, true, false, kF16>(a, stream);
  if (cap) return launch_dec_t<D, false, true, kF16>(a, stream);
  return launch_dec_t<D, false, false, kF16>(a, stream);
}

}  // namespace

int decode_stage_keys(int, int) { return NK; }
int decode_fused_max_splits(int rows, int D) {
  // the fused combine stages [rows][S] weights + [rows][2] stats in the (then idle) stage ring
  const int bytes = kStages * 2 * NK * D * 2;
  return bytes / (4 * rows) - 2;
}

cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t stream, int* launches) {
  cudaError_t e = a.f16 ? (a.s.D == 128 ? launch_dec_d<128, true>(a, stream) : launch_dec_d<64, true>(a, stream))
                        : (a.s.D == 128 ? launch_dec_d<128, false>(a, stream) : launch_dec_d<64, false>(a, stream));
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

cudaError_t launch_merge(const MergeArgs& a, cudaStream_t stream, int* launches) {
  const long long blocks = (a.rows + 3) / 4;
  merge_kernel<<<(unsigned)blocks, 128, 0, stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream, int* launches) {
  const int n = a.B * a.H;
  combine_kernel<<<(n + 3) / 4, 128, 0, stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

}  // namespace attn
