// softmax_rows.cu -- NEXT-4: the paper's motivating reduction chain (Fig. 2,
// P:164-215) as a second workload: per row, xmax = max_j x, xsum =
// sum_j exp(x - xmax) (Fig. 2a's result) and the normalised softmax
// y = exp(x - xmax) / xsum, in ONE pass over HBM.
//
// Both of the paper's repairs appear: each thread reduces its register-resident
// elements locally (privatisation, Fig. 19) and rolls its (m, l)
// across row chunks with h(t, r, r') = exp(r - r') t (Rolling Update, Fig. 2c,
// P:205-215); the row's 32-256 threads then merge their partial (m, l) with
// the Split-K global repair (Eq. 8).  Rows that fit in registers
// (<= 8192 16-bit or 4096 fp32 elements) are read once and y is written from
// registers; longer rows are re-read (from L2) for y.  HBM-bound: one read of
// x and one write of y.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>

#include "kernels.h"
#include "ptx.cuh"

namespace attn {
namespace {

constexpr int kVecPerThread = 4;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// 16-byte vector of T as floats
template <typename T> struct Vec;
template <> struct Vec<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void load(const float* p, float (&f)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
  static __device__ __forceinline__ void store(float* p, const float (&f)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  }
  static __device__ __forceinline__ float one(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ void put(float* p, float x) { *p = x; }
};
template <typename H, bool kBf16> struct Vec16 {
  static constexpr int N = 8;
  static __device__ __forceinline__ float cvt(uint16_t u) {
    if constexpr (kBf16) return __uint_as_float((uint32_t)u << 16);
    else return __half2float(__ushort_as_half(u));
  }
  static __device__ __forceinline__ uint16_t back(float x) {
    if constexpr (kBf16) return __bfloat16_as_ushort(__float2bfloat16_rn(x));
    else return __half_as_ushort(__float2half_rn(x));
  }
  static __device__ __forceinline__ void load(const H* p, float (&f)[8]) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = cvt((uint16_t)(w[i] & 0xFFFF));
      f[2 * i + 1] = cvt((uint16_t)(w[i] >> 16));
    }
  }
  static __device__ __forceinline__ void store(H* p, const float (&f)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = (uint32_t)back(f[2 * i]) | ((uint32_t)back(f[2 * i + 1]) << 16);
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  static __device__ __forceinline__ float one(const H* p) { return cvt(*reinterpret_cast<const uint16_t*>(p)); }
  static __device__ __forceinline__ void put(H* p, float x) { *reinterpret_cast<uint16_t*>(p) = back(x); }
};
template <> struct Vec<__nv_bfloat16> : Vec16<__nv_bfloat16, true> {};
template <> struct Vec<__half> : Vec16<__half, false> {};

// Eq. 8 merge of two (m, l) partials in log2 units: the repair term
// exp2(m_i - M) tag-updates each partial sum to the common reference M.
__device__ __forceinline__ void merge_ml(float& m, float& l, float m2, float l2) {
  const float M = fmaxf(m, m2);
  if (M == -INFINITY) return;                    // both empty
  l = (m == -INFINITY ? 0.f : l * ex2_approx(m - M)) + (m2 == -INFINITY ? 0.f : l2 * ex2_approx(m2 - M));
  m = M;
}

template <typename T, int kT>
__global__ void __launch_bounds__(kT) softmax_rows_kernel(const SoftmaxRowsArgs a) {
  using V = Vec<T>;
  constexpr int E = V::N * kVecPerThread;                   // elements per thread per chunk
  constexpr int kChunk = E * kT;                            // elements per chunk
  const long long row = blockIdx.x;
  const T* x = static_cast<const T*>(a.x) + row * a.x_stride;
  T* y = a.y ? static_cast<T*>(a.y) + row * a.y_stride : nullptr;
  const int tid = threadIdx.x;

  float v[E];
  auto load_chunk = [&](int c0) {                           // x * log2(e), -inf outside the row
#pragma unroll
    for (int q = 0; q < kVecPerThread; ++q) {
      const int col = c0 + (q * kT + tid) * V::N;
      float f[V::N];
      if (col + V::N <= a.cols) {
        V::load(x + col, f);
      } else {
#pragma unroll
        for (int e = 0; e < V::N; ++e) f[e] = col + e < a.cols ? V::one(x + col + e) : -INFINITY;
      }
#pragma unroll
      for (int e = 0; e < V::N; ++e) v[q * V::N + e] = f[e] * kLog2e;
    }
  };

  // ---- local (privatised) reductions, rolled across chunks (Fig. 2c repair).
  // v[] keeps exp2(x - mx) of the last chunk so a one-chunk row needs no
  // second exponential for y.
  float m = -INFINITY, l = 0.f, mx = -INFINITY;
  const int nchunk = (a.cols + kChunk - 1) / kChunk;
  for (int ch = 0; ch < nchunk; ++ch) {
    load_chunk(ch * kChunk);
    mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < E; ++e) mx = fmaxf(mx, v[e]);        // max_local
    if (mx != -INFINITY) {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int e = 0; e < E; e += 2) {                       // sum_local
        v[e] = ex2_approx(v[e] - mx);
        v[e + 1] = ex2_approx(v[e + 1] - mx);
        s0 += v[e];
        s1 += v[e + 1];
      }
      merge_ml(m, l, mx, s0 + s1);                           // xsum = h(xsum) + xsump
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = 0.f;
    }
  }
  // ---- global section across the row's threads (Eq. 8)
  float M = m, L = l;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, M, o), l2 = __shfl_xor_sync(0xffffffffu, L, o);
    merge_ml(M, L, m2, l2);
  }
  if constexpr (kT > 32) {
    __shared__ float sm[kT / 32], sl[kT / 32];
    if ((tid & 31) == 0) {
      sm[tid >> 5] = M;
      sl[tid >> 5] = L;
    }
    __syncthreads();
    M = -INFINITY;
    L = 0.f;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) merge_ml(M, L, sm[w], sl[w]);
  }
  if (tid == 0) {
    if (a.row_max) a.row_max[row] = M == -INFINITY ? -INFINITY : M * kLn2;
    if (a.row_sum) a.row_sum[row] = L;
  }
  if (y == nullptr) return;
  // ---- y = exp(x - M) / L
  const float inv = L > 0.f ? 1.f / L : 0.f;
  const float Mu = M == -INFINITY ? 0.f : M;
  for (int ch = 0; ch < nchunk; ++ch) {
    float scale;
    if (nchunk > 1) {
      load_chunk(ch * kChunk);
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = ex2_approx(v[e] - Mu);
      scale = inv;
    } else {
      scale = mx == -INFINITY ? 0.f : ex2_approx(mx - Mu) * inv;   // tag-update exp2(x - mx) to M
    }
#pragma unroll
    for (int q = 0; q < kVecPerThread; ++q) {
      const int col = ch * kChunk + (q * kT + tid) * V::N;
      float f[V::N];
#pragma unroll
      for (int e = 0; e < V::N; ++e) f[e] = v[q * V::N + e] * scale;
      if (col + V::N <= a.cols) {
        V::store(y + col, f);
      } else {
#pragma unroll
        for (int e = 0; e < V::N; ++e)
          if (col + e < a.cols) V::put(y + col + e, f[e]);
      }
    }
  }
}

// 16-bit inputs: the chunk stays in registers as the raw 16-byte vectors
// (16 registers for 32 elements); the row max is taken on packed pairs and the
// exp2 values overwrite the raw words as f16 pairs (values in (0, 1], 11-bit
// significand, below the bf16 output rounding), so the kernel needs half the
// registers of the float copy and twice the resident rows per SM (the HBM
// stream needs bytes in flight, Little's law).
template <bool kBf16> struct Raw16;
template <> struct Raw16<true> {
  static constexpr uint16_t kNegInf = 0xFF80u;
  static __device__ __forceinline__ uint32_t hmax2(uint32_t a, uint32_t b) {
    __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  static __device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
  static __device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
  static __device__ __forceinline__ uint32_t back2(float x0, float x1) {
    __nv_bfloat162 r = __floats2bfloat162_rn(x0, x1);
    return *reinterpret_cast<uint32_t*>(&r);
  }
};
template <> struct Raw16<false> {
  static constexpr uint16_t kNegInf = 0xFC00u;
  static __device__ __forceinline__ uint32_t hmax2(uint32_t a, uint32_t b) {
    __half2 r = __hmax2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  static __device__ __forceinline__ float lo(uint32_t w) { return __half2float(__ushort_as_half((uint16_t)(w & 0xFFFF))); }
  static __device__ __forceinline__ float hi(uint32_t w) { return __half2float(__ushort_as_half((uint16_t)(w >> 16))); }
  static __device__ __forceinline__ uint32_t back2(float x0, float x1) {
    __half2 r = __floats2half2_rn(x0, x1);
    return *reinterpret_cast<uint32_t*>(&r);
  }
};
__device__ __forceinline__ float f16lo(uint32_t w) { return __half2float(__ushort_as_half((uint16_t)(w & 0xFFFF))); }
__device__ __forceinline__ float f16hi(uint32_t w) { return __half2float(__ushort_as_half((uint16_t)(w >> 16))); }

#ifndef SMR_MINB
#define SMR_MINB 1536   // resident threads per SM to fit (caps registers at 40: 12 x 128-thread rows)
#endif
template <bool kBf16, int kT>
__global__ void __launch_bounds__(kT, SMR_MINB ? SMR_MINB / kT : 1) softmax_rows16_kernel(const SoftmaxRowsArgs a) {
  using R = Raw16<kBf16>;
  constexpr int kChunk = 8 * kVecPerThread * kT;
  const long long row = blockIdx.x;
  const uint16_t* x = static_cast<const uint16_t*>(a.x) + row * a.x_stride;
  uint16_t* y = a.y ? static_cast<uint16_t*>(a.y) + row * a.y_stride : nullptr;
  const int tid = threadIdx.x;

  uint32_t r[kVecPerThread][4];
  auto load_chunk = [&](int c0) {
#pragma unroll
    for (int q = 0; q < kVecPerThread; ++q) {
      const int col = c0 + (q * kT + tid) * 8;
      if (col + 8 <= a.cols) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + col));
        r[q][0] = v.x; r[q][1] = v.y; r[q][2] = v.z; r[q][3] = v.w;
      } else {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t l0 = col + 2 * w < a.cols ? x[col + 2 * w] : R::kNegInf;
          const uint32_t h0 = col + 2 * w + 1 < a.cols ? x[col + 2 * w + 1] : R::kNegInf;
          r[q][w] = l0 | (h0 << 16);
        }
      }
    }
  };

  float m = -INFINITY, l = 0.f, mx = -INFINITY;             // log2 units
  const int nchunk = (a.cols + kChunk - 1) / kChunk;
  for (int ch = 0; ch < nchunk; ++ch) {
    load_chunk(ch * kChunk);
    uint32_t pm = r[0][0];                                   // max_local on packed pairs
#pragma unroll
    for (int q = 0; q < kVecPerThread; ++q)
#pragma unroll
      for (int w = 0; w < 4; ++w) pm = R::hmax2(pm, r[q][w]);
    mx = fmaxf(R::lo(pm), R::hi(pm)) * kLog2e;
    if (mx != -INFINITY) {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int q = 0; q < kVecPerThread; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w) {                        // sum_local
          const float e0 = ex2_approx(fmaf(R::lo(r[q][w]), kLog2e, -mx));
          const float e1 = ex2_approx(fmaf(R::hi(r[q][w]), kLog2e, -mx));
          s0 += e0;
          s1 += e1;
          const __half2 h = __floats2half2_rn(e0, e1);
          r[q][w] = *reinterpret_cast<const uint32_t*>(&h);
        }
      merge_ml(m, l, mx, s0 + s1);                           // xsum = h(xsum) + xsump
    } else {
#pragma unroll
      for (int q = 0; q < kVecPerThread; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w) r[q][w] = 0u;
    }
  }
  float M = m, L = l;                                        // global section (Eq. 8)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, M, o), l2 = __shfl_xor_sync(0xffffffffu, L, o);
    merge_ml(M, L, m2, l2);
  }
  if constexpr (kT > 32) {
    __shared__ float sm[kT / 32], sl[kT / 32];
    if ((tid & 31) == 0) {
      sm[tid >> 5] = M;
      sl[tid >> 5] = L;
    }
    __syncthreads();
    M = -INFINITY;
    L = 0.f;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) merge_ml(M, L, sm[w], sl[w]);
  }
  if (tid == 0) {
    if (a.row_max) a.row_max[row] = M == -INFINITY ? -INFINITY : M * kLn2;
    if (a.row_sum) a.row_sum[row] = L;
  }
  if (y == nullptr) return;
  const float inv = L > 0.f ? 1.f / L : 0.f;                 // y = exp(x - M) / L
  const float Mu = M == -INFINITY ? 0.f : M;
#ifndef SMR_REV
#define SMR_REV 1
#endif
  for (int c = 0; c < nchunk; ++c) {
    const int ch = SMR_REV ? nchunk - 1 - c : c;   // reverse: the re-read starts with the L2-hottest chunk
    uint32_t o[kVecPerThread][4];
    if (nchunk > 1) {
      load_chunk(ch * kChunk);
#pragma unroll
      for (int q = 0; q < kVecPerThread; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w)
          o[q][w] = R::back2(ex2_approx(fmaf(R::lo(r[q][w]), kLog2e, -Mu)) * inv,
                             ex2_approx(fmaf(R::hi(r[q][w]), kLog2e, -Mu)) * inv);
    } else {
      const float scale = mx == -INFINITY ? 0.f : ex2_approx(mx - Mu) * inv;   // tag-update to M
#pragma unroll
      for (int q = 0; q < kVecPerThread; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w) o[q][w] = R::back2(f16lo(r[q][w]) * scale, f16hi(r[q][w]) * scale);
    }
#pragma unroll
    for (int q = 0; q < kVecPerThread; ++q) {
      const int col = ch * kChunk + (q * kT + tid) * 8;
      if (col + 8 <= a.cols) {
        *reinterpret_cast<uint4*>(y + col) = make_uint4(o[q][0], o[q][1], o[q][2], o[q][3]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (col + e < a.cols) y[col + e] = (uint16_t)(o[q][e >> 1] >> (16 * (e & 1)));
      }
    }
  }
}

#ifndef SMR_T512
#define SMR_T512 0      // 1: rows of 8193..16384 16-bit elements as one 512-thread chunk (measured slower: 3 resident rows)
#endif
template <bool kBf16>
cudaError_t launch_rows16(const SoftmaxRowsArgs& a, cudaStream_t stream) {
  const int need = (a.cols + 8 * kVecPerThread - 1) / (8 * kVecPerThread);
  const unsigned grid = (unsigned)a.rows;
  if (need <= 32) softmax_rows16_kernel<kBf16, 32><<<grid, 32, 0, stream>>>(a);
  else if (need <= 64) softmax_rows16_kernel<kBf16, 64><<<grid, 64, 0, stream>>>(a);
  else if (need <= 128) softmax_rows16_kernel<kBf16, 128><<<grid, 128, 0, stream>>>(a);
  else if (need <= 256 || !SMR_T512) softmax_rows16_kernel<kBf16, 256><<<grid, 256, 0, stream>>>(a);
  else softmax_rows16_kernel<kBf16, 512><<<grid, 512, 0, stream>>>(a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_rows_t(const SoftmaxRowsArgs& a, cudaStream_t stream) {
  // threads per row: enough for the row to be one chunk of kVecPerThread vectors per thread
  const int per_thread = Vec<T>::N * kVecPerThread;
  const int need = (a.cols + per_thread - 1) / per_thread;
  const unsigned grid = (unsigned)a.rows;
  if (need <= 32) softmax_rows_kernel<T, 32><<<grid, 32, 0, stream>>>(a);
  else if (need <= 64) softmax_rows_kernel<T, 64><<<grid, 64, 0, stream>>>(a);
  else if (need <= 128) softmax_rows_kernel<T, 128><<<grid, 128, 0, stream>>>(a);
  else softmax_rows_kernel<T, 256><<<grid, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_softmax_rows(const SoftmaxRowsArgs& a, cudaStream_t stream, int* launches) {
#ifndef SMR_FLOAT16
#define SMR_FLOAT16 0   // 1: 16-bit rows through the float-register kernel (A/B)
#endif
  cudaError_t e;
  if (a.dtype == 1) e = launch_rows_t<float>(a, stream);
  else if (SMR_FLOAT16) e = a.dtype == 2 ? launch_rows_t<__half>(a, stream) : launch_rows_t<__nv_bfloat16>(a, stream);
  else e = a.dtype == 2 ? launch_rows16<false>(a, stream) : launch_rows16<true>(a, stream);
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

}  // namespace attn
