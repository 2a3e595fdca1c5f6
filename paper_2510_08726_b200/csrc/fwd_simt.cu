// fwd_simt.cu -- Rolling Update forward for fp32 inputs on CUDA cores.
//
// Same single-pass loop as the tensor-core kernel (Alg. 1; Fig. 2c
// P:205-215 at the element level): for each 32-key tile, score_mod + mask,
// m_new = max(m_old, tile max), repair alpha = exp(m_old - m_new) applied to
// l and to the output accumulator (Eq. 7), l += sum exp(x - m_new),
// O += p V, m_old = m_new; O / l at the end.
//
// fp32 has no tensor-core path that meets the 1e-4 parity bar (tf32 rounds
// the inputs), so this kernel uses FFMA and accurate expf.  One warp owns one
// query row; lane j scores key j of the tile; lane d accumulates output
// dimensions d, d + 32, ...  K/V tiles are staged in shared memory once per
// CTA (4 rows) with a +1 padding to avoid bank conflicts.
#include <math.h>

#include "kernels.h"

namespace attn {
namespace {

constexpr int kRows = 4;     // query rows (warps) per CTA
constexpr int kTile = 32;    // keys per tile
constexpr int kMaxD = 256;

__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__global__ void __launch_bounds__(kRows * 32) fwd_simt_kernel(const FwdSimtArgs a) {
  extern __shared__ float sm[];
  const int D = a.s.D, Dp = D + 1;
  float* sK = sm;                       // [kTile][D + 1]
  float* sV = sK + kTile * Dp;          // [kTile][D + 1]
  float* sQ = sV + kTile * Dp;          // [kRows][D]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hq = blockIdx.y, b = blockIdx.z, hkv = hq / (a.s.Hq / a.s.Hkv);
  const int i = blockIdx.x * kRows + warp;
  const bool row_ok = i < a.s.Sq;
  const VariantParams& v = a.v;

  const float* qrow = a.q + b * a.q_sb + hq * a.q_sh + (long long)i * a.q_ss;
  for (int d = lane; d < D; d += 32) sQ[warp * D + d] = row_ok ? qrow[d] : 0.f;

  const long long qpos = v.q_off + i;
  const float slope = v.alibi ? v.alibi[hq] : 0.f;
  constexpr int kAcc = kMaxD / 32;
  float acc[kAcc];
#pragma unroll
  for (int r = 0; r < kAcc; ++r) acc[r] = 0.f;
  float m_old = -INFINITY, l = 0.f;

  const float* kbase = a.k + b * a.k_sb + hkv * a.k_sh;
  const float* vbase = a.v_ + b * a.v_sb + hkv * a.v_sh;
  for (int j0 = 0; j0 < a.s.Skv; j0 += kTile) {
    __syncthreads();
    for (int e = threadIdx.x; e < kTile * D; e += blockDim.x) {
      const int jj = e / D, d = e % D, j = j0 + jj;
      sK[jj * Dp + d] = j < a.s.Skv ? kbase[(long long)j * a.k_ss + d] : 0.f;
      sV[jj * Dp + d] = j < a.s.Skv ? vbase[(long long)j * a.v_ss + d] : 0.f;
    }
    __syncthreads();
    // score of key j0 + lane (Fig. 8 batch_matmul + score_mod + mask)
    const int j = j0 + lane;
    float dot = 0.f;
    for (int d = 0; d < D; ++d) dot = fmaf(sQ[warp * D + d], sK[lane * Dp + d], dot);
    float x = v.scale * dot;
    if (v.softcap > 0.f) x = v.softcap * tanhf(x / v.softcap);
    const long long kpos = v.kv_off + j;
    if (v.alibi) x -= slope * fabsf((float)(qpos - kpos));
    bool ok = j < a.s.Skv;
    if (v.causal) ok = ok && kpos <= qpos;
    if (v.window_left >= 0) ok = ok && qpos - kpos <= v.window_left;
    if (v.window_right >= 0) ok = ok && kpos - qpos <= v.window_right;
    x = ok ? x : -INFINITY;
    // rolling update with repair (Fig. 2c)
    const float m_new = fmaxf(m_old, warp_max(x));
    const float alpha = (m_new == -INFINITY || m_old == -INFINITY) ? (m_old == -INFINITY ? 0.f : 1.f)
                                                                   : expf(m_old - m_new);
    const float p = (m_new == -INFINITY) ? 0.f : expf(x - m_new);
    l = alpha * l + warp_sum(p);
#pragma unroll
    for (int r = 0; r < kAcc; ++r) acc[r] *= alpha;
    for (int jj = 0; jj < kTile; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, p, jj);
#pragma unroll
      for (int r = 0; r < kAcc; ++r) {
        const int d = lane + 32 * r;
        if (d < D) acc[r] = fmaf(pj, sV[jj * Dp + d], acc[r]);
      }
    }
    m_old = m_new;
  }
  if (!row_ok) return;
  const float inv_l = l > 0.f ? 1.f / l : 0.f;
  float* orow = a.o + b * a.o_sb + hq * a.o_sh + (long long)i * a.o_ss;
#pragma unroll
  for (int r = 0; r < kAcc; ++r) {
    const int d = lane + 32 * r;
    if (d < D) orow[d] = acc[r] * inv_l;
  }
  if (a.lse && lane == 0)
    a.lse[((size_t)b * a.s.Hq + hq) * a.s.Sq + i] = l > 0.f ? m_old + logf(l) : -INFINITY;
}

}  // namespace

cudaError_t launch_fwd_simt(const FwdSimtArgs& a, cudaStream_t stream, int* launches) {
  const int D = a.s.D;
  const size_t smem = sizeof(float) * (2 * kTile * (D + 1) + kRows * D);
  cudaError_t e = cudaFuncSetAttribute(fwd_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.s.Sq + kRows - 1) / kRows, a.s.Hq, a.s.B);
  fwd_simt_kernel<<<grid, kRows * 32, smem, stream>>>(a);
  e = cudaGetLastError();
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

}  // namespace attn
